#!/bin/bash
# Same-box A/B on the default bench: auto (softmax over 8 of 16 columns at
# M <= 8) vs forced 2 groups over all 16 columns (BMC_OPT_TCK_GROUPS via
# --tck-groups 2), alternating.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
i=0
for g in 0 2 0 2; do
  timeout 400 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --tck-groups $g 2>&1 | tail -1 \
    > gpurun_out/ab_ns_${i}_${g}.json
  i=$((i+1))
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ab_ns_*.json")):
    d = json.loads(open(f).read())
    print(f, round(d["value"]), round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"])
PY
