cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build24.log 2>&1 || tail -5 $O/build24.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest24.log 2>&1; tail -5 $O/pytest24.log
for a in region pool; do
  timeout 900 python bench.py --config 70b-long --arena $a --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/b24.log 2>&1
  tail -1 $O/b24.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'config': '70b-long', 'arena': '$a', 'value': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz'], 'gm': d['growth_memory']}))" | tee -a $O/arena24.jsonl || tail -3 $O/b24.log
done
timeout 600 python bench.py --config l3-8b --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/b24l3.log 2>&1; tail -1 $O/b24l3.log | cut -c1-200
