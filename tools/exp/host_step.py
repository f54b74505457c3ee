"""Host cost of one bmc_decode_step call (7B shape, 32 layers, B=16) with a
small cache so the GPU never backs up the queue: per-call host time from
Python (ctypes) and the GPU time of the same steps."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2511_12031_b200 import bmc
L, B, H, D, N = 32, 16, 32, 128, 512
hs = [bmc.KVCache(B, H, H, D, 128, N, dtype="bf16") for _ in range(L)]
plan = bmc.StepPlan(hs)
k = [torch.randn(B, H, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
q = [torch.randn(B, H, 1, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
o = [torch.empty(B, H, 1, D, device="cuda") for _ in range(L)]
K, Q, O = plan.ptrs(k), plan.ptrs(q), plan.ptrs(o)
for n in range(1, 65):
    bmc.bmc_decode_step(plan, K, K, Q, O, n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for n in range(65, 65 + 400):
    bmc.bmc_decode_step(plan, K, K, Q, O, n)
t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
print(f"host us/step {1e6*(t1-t0)/400:.1f}  gpu us/step {1e3*e0.elapsed_time(e1)/400:.1f}")
for h in hs:
    h.close()
