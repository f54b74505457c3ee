"""A/B of the M = 72 keys-on-lanes variant: 3 (default) vs 2 softmax column groups."""
import os, sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at
from paper_2511_12031_b200 import bmc
bmc.load()
for cap in (4096, 8192, 16384, 32768):
    for g in (3, 2):
        r = attn_at(8, 8, 64, 128, cap, t=9, path=4, reps=12, layers=4, groups=g)
        print(cap, g, round(r["us"], 1), round(r["GBps"]))
