#!/bin/bash
# What the driver runs at round end, on one B200: GPU tests, smoke, the default
# bench line, the reference arm, and the multi-rank code path (2 ranks sharing
# the GPU: gloo reductions, timings not meaningful).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 > $O/dc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/dc_smoke.log 2>&1
timeout 900 python bench.py > $O/dc_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/dc_ref.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --layers 2 --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $O/dc_multi.log 2>&1
cat $O/dc_pytest.log; tail -1 $O/dc_smoke.log; tail -1 $O/dc_bench.log | cut -c1-200
tail -1 $O/dc_ref.log | cut -c1-200; tail -1 $O/dc_multi.log | cut -c1-200
