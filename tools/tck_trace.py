"""Timeline of the keys-on-lanes tcgen05 kernel (trace build, CTA 0): per-tile
clock64 at each wait / issue point, and per-CTA run time / SM clock.
usage: BMC_LIB=<trace build> python tools/tck_trace.py B H_kv H_q cap t"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from tools.microbench import attn_at
from paper_2511_12031_b200 import bmc
L = bmc.load()
B, Hk, Hq, cap, t = (int(x) for x in sys.argv[1:6])
tcta = int(sys.argv[6]) if len(sys.argv) > 6 else 0
L.bmc_tck_trace_cta(tcta)
print(attn_at(B, Hk, Hq, 128, cap, t=t, path=4, reps=2, layers=1))
buf = (ctypes.c_longlong * (16 * 256 + 160 * 4))()
L.bmc_tck_trace.argtypes = [ctypes.c_void_p]
assert L.bmc_tck_trace(buf) == 0
a = np.array(buf[:])
tr = a[:16 * 256].reshape(16, 256)
cta = a[16 * 256:].reshape(160, 4)[:148]
base = cta[tcta, 0]
names = ["K issue", "V issue", "QK fullK", "QK Sempty", "QK issued", "PV pfull", "PV fullV",
         "PV issued", "sm pre-S", "sm S", "sm any", "sm preP", "sm Pempty", "sm Pfull",
         "pre-ODONE", "ODONE"]
print("tile " + " ".join(f"{n:>9s}" for n in names))
for i in range(0, 32):
    print(f"{i:4d} " + " ".join(f"{(tr[e][i] - base) if tr[e][i] else -1:9d}" for e in range(16)))
print("CTA end (cycles from its start):", cta[tcta, 2] - cta[tcta, 0])
cyc = cta[:, 2] - cta[:, 0]; ns = cta[:, 3] - cta[:, 1]
t0 = cta[:, 1].min()
ok = ns > 0
print(f"CTA cycles: min {cyc[ok].min()} med {np.median(cyc[ok]):.0f} max {cyc[ok].max()}; "
      f"ns: min {ns[ok].min()} med {np.median(ns[ok]):.0f} max {ns[ok].max()}; "
      f"clock {np.median(cyc[ok] / ns[ok]):.3f} GHz")
print(f"start skew {cta[ok, 1].max() - t0} ns; end: first {cta[ok, 3].min() - t0} last {cta[ok, 3].max() - t0} ns")
order = np.argsort(ns)
print("slowest CTAs (id, ns, start offset ns):", [(int(c), int(ns[c]), int(cta[c, 1] - t0)) for c in order[-12:]])
print("fastest CTAs:", [(int(c), int(ns[c])) for c in order[:8]])
print("ns by CTA id:", " ".join(str(int(x) // 1000) for x in ns))
