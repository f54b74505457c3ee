cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build16.log 2>&1 || tail -5 $O/build16.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest16.log 2>&1; tail -3 $O/pytest16.log
timeout 900 python bench.py > $O/bench16_default.log 2>&1; tail -1 $O/bench16_default.log | cut -c1-300
timeout 1800 python tools/sweep.py --config 7b-sd --rs 16,32,64,128,256 > $O/sweep16_7bsd.json 2> $O/sweep16_7bsd.err || tail -3 $O/sweep16_7bsd.err
tail -1 $O/sweep16_7bsd.json | cut -c1-300
for c in 7b-tree 7b-tree-b32 opt13b-tree; do
  timeout 1500 python tools/tree_sweep.py --config $c > $O/tree16_$c.json 2> $O/tree16_$c.err
  tail -1 $O/tree16_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['best_T'], d['norm_latency_row'], d['paper']['norm'])" || tail -3 $O/tree16_$c.err
done
