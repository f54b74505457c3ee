"""One 70B-shaped verify launch shape (B=8, 8 kv / 64 q heads, d=128, t=9 ->
M=72) at a given cache size through the keys-on-lanes tcgen05 path, for ncu
captures (the first launches are warm-up; capture with -s)."""
import os
import sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402
bmc.load()
cap = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
t = int(sys.argv[2]) if len(sys.argv) > 2 else 9
r = attn_at(8, 8, 64, 128, cap, t=t, path=4, reps=int(os.environ.get("REPS", "4")), layers=2)
print(r)
