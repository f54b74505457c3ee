cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/exp/abks3.sh
for c in 7b-tree-b32 opt13b-tree 7b-tree; do
  timeout 1500 python tools/tree_sweep.py --config $c > $O/tree_$c.json 2> $O/tree_$c.err
  tail -1 $O/tree_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['best_T'], d['norm_latency_row'], d['paper']['norm'])" || tail -3 $O/tree_$c.err
done
timeout 2400 python tools/advisor_validate.py > $O/advisor_validate.json 2> $O/advisor_validate.err || tail -3 $O/advisor_validate.err
head -6 $O/advisor_validate.json | cut -c1-400
