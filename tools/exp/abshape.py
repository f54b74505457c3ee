"""A/B of single attention launches across experiment builds (BMC_LIB):
70B verify (M = 72) at 8K / 32K, L3-8B decode (M = 4) at 8K, 7B decode
(M = 1) at 4K; GB/s of algorithmic bytes."""
import json
import os
import sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402
bmc.load()
tag = sys.argv[1]
for name, B, hkv, hq, cap, t in (("70B M=72", 8, 8, 64, 8192, 9), ("70B M=72", 8, 8, 64, 32768, 9),
                                 ("L3 M=4", 64, 8, 32, 8192, 1), ("7B M=1", 16, 32, 32, 4096, 1)):
    r = attn_at(B, hkv, hq, 128, cap, t=t, path=4, reps=20, layers=4)
    print(json.dumps({"lib": tag, "shape": name, "cap": cap, "us": round(r["us"], 1),
                      "GBps": round(r["GBps"])}), flush=True)
