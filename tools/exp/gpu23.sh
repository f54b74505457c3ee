cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build23.log 2>&1 || tail -5 $O/build23.log
for c in 7b-tree 7b-tree-b32 opt13b-tree; do
  timeout 900 python tools/tree_sweep.py --config $c > $O/tree23_$c.json 2> $O/tree23_$c.err
  tail -1 $O/tree23_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['best_T'], d['norm_latency_row'], d['paper']['norm'])" || tail -3 $O/tree23_$c.err
done
timeout 1500 python tools/advisor_validate.py > $O/advisor23.json 2> $O/advisor23.err || tail -3 $O/advisor23.err
tail -1 $O/advisor23.json | cut -c1-200
timeout 900 python tools/sweep.py --config 70b-long --n-max 8192 --rs 64,128,256,1024 > $O/sweep23_70b.json 2> $O/sweep23_70b.err || tail -3 $O/sweep23_70b.err
tail -1 $O/sweep23_70b.json | cut -c1-300
timeout 900 python tools/sweep.py --config 7b-sd --rs 32,64,128,256 > $O/sweep23_7bsd.json 2> $O/sweep23_7bsd.err || tail -3 $O/sweep23_7bsd.err
tail -1 $O/sweep23_7bsd.json | cut -c1-200
for a in region pool region pool; do
  timeout 600 python bench.py --config 7b --arena $a --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/b23.log 2>&1
  tail -1 $O/b23.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'config': '7b', 'arena': '$a', 'value': d['value'], 'frac': d['roofline']['frac'], 'growth_frac': d['roofline'].get('growth', {}).get('frac'), 'sm_mhz': d['clocks']['sm_mhz']}))" | tee -a $O/arena23.jsonl
done
