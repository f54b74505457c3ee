"""A/B of the keys-on-lanes kernel's L2 prefetch distance on single-layer launches."""
import os, sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at
from paper_2511_12031_b200 import bmc
bmc.load()
shapes = [("70B M=72", dict(B=8, H_kv=8, H_q=64, t=9), (8192, 32768)),
          ("70B M=8", dict(B=8, H_kv=8, H_q=64, t=1), (8192, 32768)),
          ("L3 M=4", dict(B=64, H_kv=8, H_q=32, t=1), (2048, 8192)),
          ("7B M=1", dict(B=16, H_kv=32, H_q=32, t=1), (1024, 4096))]
for name, sh, caps in shapes:
    for cap in caps:
        row = []
        for pf in (0, 2, 3, 4, 6):
            r = attn_at(sh["B"], sh["H_kv"], sh["H_q"], 128, cap, t=sh["t"], path=4, reps=12,
                        layers=4, prefetch=pf)
            row.append(f"pf{pf} {r['GBps']:.0f}")
        print(name, cap, " | ".join(row), flush=True)
