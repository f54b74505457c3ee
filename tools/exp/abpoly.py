"""A/B of the 70B verify (M = 72) single launches across experiment builds
(BMC_LIB): GB/s at 8K and 32K context."""
import json
import os
import sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402
bmc.load()
tag = sys.argv[1]
for cap in (8192, 32768):
    r = attn_at(8, 8, 64, 128, cap, t=9, path=4, reps=20, layers=4)
    print(json.dumps({"lib": tag, "cap": cap, "M": r["M"], "us": round(r["us"], 1),
                      "GBps": round(r["GBps"])}), flush=True)
