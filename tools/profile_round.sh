#!/bin/bash
# One GPU call that refreshes the round's evidence under gpurun_out/:
# GPU tests, smoke, the default bench line (as the driver runs it), the
# launch list of the same command, and ncu --set full captures of the two
# attention kernels inside the fused multi-layer steps (for `traffic`).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_7b.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu \
  > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_step -s 3000 -c 1 \
  -o $O/ncu_attn_step python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tck -s 3000 -c 1 \
  -o $O/ncu_attn_tck_l3 python bench.py --config l3-8b --steps 1 --warmup 0 --no-e2e --no-cpu \
  > /dev/null 2>&1
for r in $O/ncu_attn_step $O/ncu_attn_tck_l3; do
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details --csv > $r.details.csv 2>/dev/null
done
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log; tail -1 $O/bench_default.log | cut -c1-400
