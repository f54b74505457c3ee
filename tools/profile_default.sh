#!/bin/bash
# Default bench line + its launch list + an ncu --set full capture of the
# default path's attention kernel (for `traffic`), under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_7b.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu \
  > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tck -s 3000 -c 1 \
  -o $O/ncu_attn_tck_7b python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
tail -1 $O/bench_default.log | cut -c1-300
