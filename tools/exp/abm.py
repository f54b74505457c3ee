"""70B-shaped verify launches at M = 8t (t = 5, 7, 8, 9) across builds
(BMC_LIB): GB/s of algorithmic bytes, single layer, 4 handles round-robin."""
import json
import os
import sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402
bmc.load()
tag = sys.argv[1]
for cap in (8192, 32768):
    for t in (5, 7, 8, 9):
        r = attn_at(8, 8, 64, 128, cap, t=t, path=4, reps=20, layers=4)
        print(json.dumps({"lib": tag, "cap": cap, "M": 8 * t, "us": round(r["us"], 1),
                          "GBps": round(r["GBps"])}), flush=True)
