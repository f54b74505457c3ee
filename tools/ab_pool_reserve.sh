#!/bin/bash
# Same-box A/B of bmc_pool_reserve on the default bench (alternating runs).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
i=0
for flag in "--pool-reserve" "" "--pool-reserve" ""; do
  timeout 400 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu $flag 2>&1 | tail -1 \
    > gpurun_out/ab_reserve_${i}.json
  i=$((i+1))
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ab_reserve_*.json")):
    d = json.loads(open(f).read())
    print(f, d["growth_memory"]["bytes"], round(d["value"]), round(d["ms_per_step"]),
          round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"])
PY
