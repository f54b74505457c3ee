"""Quick check of the tcgen05 verify kernel against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from harness import Pair
from paper_2511_12031_b200 import bmc
for (H_kv, H_q, n, r) in [(1, 1, 10, 16), (1, 8, 70, 16), (2, 16, 200, 24)]:
    p = Pair(2, H_kv, H_q, 128, r, 400, dtype="bf16", seed=1)
    p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, 2)
    worst = 0
    for i in range(n):
        p.append()
        try:
            p.sdpa()
        except AssertionError as e:
            print("FAIL", H_kv, H_q, i, e); break
    print("M=", H_q // H_kv, "worst(tol units)", p.worst, flush=True)
    p.close()
