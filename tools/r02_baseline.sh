#!/bin/bash
# Round-2 first GPU call: HEAD's GPU tests, default bench, 70B verify single
# launches, and an ncu --set full capture of the M=72 keys-on-lanes launch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 300 python tools/exp/mb70.py 8192,32768 > $O/mb70.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tck -s 4 -c 1 \
  -o $O/ncu_tck72 python tools/exp/one70.py 32768 9 > $O/ncu_tck72.log 2>&1
ncu -i $O/ncu_tck72.ncu-rep --page raw --csv > $O/ncu_tck72.raw.csv 2>/dev/null
ncu -i $O/ncu_tck72.ncu-rep --page details --csv > $O/ncu_tck72.details.csv 2>/dev/null
ncu -i $O/ncu_tck72.ncu-rep --page source --csv > $O/ncu_tck72.source.csv 2>/dev/null
cat $O/pytest_gpu.log; tail -1 $O/bench_default.log | cut -c1-600; cat $O/mb70.log
