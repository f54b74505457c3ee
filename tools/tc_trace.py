"""Timeline of the tcgen05 verify kernel (trace build, CTA 0): per-tile clock64
at each wait / issue point, printed relative to the first event."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from tools.microbench import attn_at
from paper_2511_12031_b200 import bmc
L = bmc.load()
cfg = sys.argv[1] if len(sys.argv) > 1 else "8"
if cfg == "8":
    attn_at(8, 8, 64, 128, 8192, t=1, path=2, reps=2, layers=1)
else:
    attn_at(64, 8, 32, 128, 4096, t=1, path=2, reps=2, layers=1)
buf = (ctypes.c_longlong * (16 * 256 + 2 * 256 * 9 + 8 * 256 * 4 + 160 * 4))()
L.bmc_tc_trace.argtypes = [ctypes.c_void_p]
assert L.bmc_tc_trace(buf) == 0
allv = np.array(buf[:])
t = allv[:16 * 256].reshape(16, 256)
mm = allv[16 * 256:16 * 256 + 2 * 256 * 9].reshape(2, 256, 9)
o = 16 * 256 + 2 * 256 * 9
sm = allv[o:o + 8 * 256 * 4].reshape(8, 256, 4)
cta = allv[o + 8 * 256 * 4:].reshape(160, 4)[:148]
base = t[t > 0].min()
names = ["K issue", "V issue", "QK fullK", "QK issued", "PV pfull", "PV fullV", "sm pre-S",
         "sm S ready", "sm pair", "sm Pempty", "sm Pfull"]
print("tile " + " ".join(f"{n:>10s}" for n in names))
for i in range(0, 40):
    print(f"{i:4d} " + " ".join(f"{(t[e][i]-base) if t[e][i] else -1:10d}" for e in range(11)))

print("MMA issue times (QK: 8 MMAs + after; PV: 8 MMAs + after), tiles 16..23, merged timeline")
ev = []
for tile in range(16, 24):
    for j in range(9):
        ev.append((mm[0, tile, j] - base, f"QK{tile}.{j}"))
        ev.append((mm[1, tile, j] - base, f"PV{tile}.{j}"))
ev.sort()
prev = None
for tm_, name in ev:
    print(f"{tm_:8d} {'+%d' % (tm_ - prev) if prev is not None else '':>7s} {name}")
    prev = tm_

print("per softmax warp (2..9): S ready / pair / Pempty / Pfull, tiles 18..21")
for tile in range(18, 22):
    for w in range(8):
        print(f"tile {tile} warp {w+2}: " + " ".join(f"{sm[w, tile, e] - base:8d}" for e in range(4)))

cyc = cta[:, 2] - cta[:, 0]; ns = cta[:, 3] - cta[:, 1]
t0 = cta[:, 1].min()
print(f"CTA cycles: min {cyc.min()} med {np.median(cyc):.0f} max {cyc.max()}; ns: min {ns.min()} med {np.median(ns):.0f} max {ns.max()}; clock {np.median(cyc / ns):.3f} GHz")
print(f"start skew {cta[:, 1].max() - t0} ns; end spread: first {cta[:, 3].min() - t0} last {cta[:, 3].max() - t0} ns")
