#!/bin/bash
# Same-box A/B of the 7B decode attention kernel: auto (CUDA cores at M=1) vs
# forced keys-on-lanes tcgen05 (BMC_OPT_ATTN_PATH=4), alternating runs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
i=0
for pa in 0 4 0 4; do
  timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --attn-path $pa 2>&1 | tail -1 \
    > gpurun_out/ab_path_${i}_${pa}.json
  i=$((i+1))
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ab_path_*.json")):
    d = json.loads(open(f).read())
    print(f, round(d["value"]), round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"], d["gpu_launches"])
PY
