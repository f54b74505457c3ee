cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build18.log 2>&1 || tail -5 $O/build18.log
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest18.log 2>&1; tail -3 $O/pytest18.log
for c in 7b-tree 7b-tree-b32 opt13b-tree; do
  timeout 1500 python tools/tree_sweep.py --config $c > $O/tree18_$c.json 2> $O/tree18_$c.err
  tail -1 $O/tree18_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['best_T'], d['norm_latency_row'], d['paper']['norm'])" || tail -3 $O/tree18_$c.err
done
timeout 2400 python tools/advisor_validate.py > $O/advisor18.json 2> $O/advisor18.err || tail -3 $O/advisor18.err
tail -1 $O/advisor18.json | cut -c1-300
timeout 2400 python tools/sweep.py --config 70b-long --n-max 8192 --rs 64,128,256,1024 > $O/sweep18_70b.json 2> $O/sweep18_70b.err || tail -3 $O/sweep18_70b.err
tail -1 $O/sweep18_70b.json | cut -c1-300
timeout 900 python tools/exp/growth_cost.py --l3 --reserve > $O/growth18_l3.txt 2>&1; cat $O/growth18_l3.txt | grep -v 'host ms'
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tck -s 3000 -c 1 \
  -o $O/ncu18_tck_l3 python bench.py --config l3-8b --steps 1 --warmup 0 --no-e2e --no-cpu --no-check > $O/ncu18_l3.log 2>&1
ncu -i $O/ncu18_tck_l3.ncu-rep --page raw --csv > $O/ncu18_tck_l3.raw.csv 2>/dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches18_l3.csv python bench.py --config l3-8b --steps 1 --warmup 0 --no-e2e --no-cpu --no-check > /dev/null 2>&1
wc -l $O/launches18_l3.csv
