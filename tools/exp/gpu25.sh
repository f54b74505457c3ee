cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build25.log 2>&1 || tail -5 $O/build25.log
timeout 1200 python bench.py > $O/bench25_default.log 2>&1; tail -1 $O/bench25_default.log | cut -c1-300
timeout 900 python bench.py --config 70b-long --steps 1 --warmup 1 --no-cpu > $O/bench25_70b.log 2>&1; tail -1 $O/bench25_70b.log | cut -c1-300
timeout 900 python tools/tree_sweep.py --config 7b-tree-b32 > $O/tree25_7b-tree-b32.json 2> $O/tree25_7b-tree-b32.err
tail -1 $O/tree25_7b-tree-b32.json | cut -c1-300
timeout 1500 python tools/advisor_validate.py > $O/advisor25.json 2> $O/advisor25.err || tail -3 $O/advisor25.err
timeout 900 python tools/sweep.py --config 7b-sd --rs 32,64,128,256 > $O/sweep25_7bsd.json 2> $O/sweep25_7bsd.err || tail -3 $O/sweep25_7bsd.err
tail -1 $O/sweep25_7bsd.json | cut -c1-300
