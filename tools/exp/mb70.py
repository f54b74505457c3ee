"""70B-shaped verify attention at small and large caches: queries-on-lanes
(path 3) vs keys-on-lanes (path 4) tcgen05 kernels."""
import os
import sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402
bmc.load()
caps = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8192, 32768]
for cap in caps:
    for t in (1, 5, 9):
        for pa in (3, 4):
            r = attn_at(8, 8, 64, 128, cap, t=t, path=pa, reps=20, layers=4)
            print(cap, t, r["M"], pa, round(r["us"], 1), round(r["GBps"]))
