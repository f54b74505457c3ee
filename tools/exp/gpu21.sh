cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build21.log 2>&1 || tail -5 $O/build21.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest21.log 2>&1; tail -5 $O/pytest21.log
timeout 400 python tools/exp/growth_cost.py --l3 --region > $O/growth21_l3_region.txt 2>&1; cat $O/growth21_l3_region.txt
timeout 300 python tools/exp/growth_cost.py --region > $O/growth21_7b_region.txt 2>&1; grep -v 'host ms' $O/growth21_7b_region.txt
for a in region pool region pool; do
  timeout 600 python bench.py --config l3-8b --arena $a --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/b21.log 2>&1
  tail -1 $O/b21.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'arena': '$a', 'value': d['value'], 'frac': d['roofline']['frac'], 'growth_frac': d['roofline'].get('growth', {}).get('frac'), 'sm_mhz': d['clocks']['sm_mhz'], 'gm': d['growth_memory']}))" | tee -a $O/arena21.jsonl
done
