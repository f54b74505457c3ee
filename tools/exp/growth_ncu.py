"""ncu targets for the growth copy (7B shape: B=16, 32 heads, d=128, r=64).
  decode : 32 layers through bmc_decode_step; launch index 4032 of attn_tck is the
           copy-on-read growth step cap 4032 -> 4096 (n = 4033)
  realloc: one layer through the per-layer API with copy-on-read off; launch
           index 62 of realloc_copy_zero_kernel is the growth 4032 -> 4096."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "decode"
B, H, D, N, r = 16, 32, 128, 4096, 64
k = torch.randn(B, H, D, device="cuda").to(torch.bfloat16)
q = torch.randn(B, H, 1, D, device="cuda").to(torch.bfloat16)
if mode == "decode":
    L = 32
    hs = [bmc.KVCache(B, H, H, D, r, N, dtype="bf16") for _ in range(L)]
    plan = bmc.StepPlan(hs)
    o = [torch.empty(B, H, 1, D, device="cuda") for _ in range(L)]
    K, Q, O = plan.ptrs([k] * L), plan.ptrs([q] * L), plan.ptrs(o)
    for n in range(1, 4036):
        bmc.bmc_decode_step(plan, K, K, Q, O, n)
else:
    h = bmc.KVCache(B, H, H, D, r, N, dtype="bf16")
    h.set_option(bmc.BMC_OPT_COPY_ON_READ, 0)
    for n in range(1, 4036):
        h.append(k, k)
torch.cuda.synchronize()
print("done", mode)
