cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/ab.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from tools.microbench import attn_at
from paper_2511_12031_b200 import bmc
bmc.load()
for cap in (4096, 8192, 16384, 32768):
    r = attn_at(8, 8, 64, 128, cap, t=9, path=4, reps=12, layers=4)
    print(os.environ.get("BMC_LIB", "head"), cap, round(r["us"], 1), round(r["GBps"]), flush=True)
PY
for i in 1 2; do
timeout 300 python /tmp/ab.py
BMC_LIB=tools/exp/libbmc_ks3.so timeout 300 python /tmp/ab.py
done > $O/abks3.log 2>&1
BMC_LIB=tools/exp/libbmc_trace.so timeout 300 python tools/tck_trace.py 64 8 32 8192 1 0 > $O/trace_l3_8192.txt 2>&1
cat $O/abks3.log; tail -7 $O/trace_l3_8192.txt | cut -c1-400
