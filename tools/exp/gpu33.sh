cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build33.log 2>&1 || tail -5 $O/build33.log
timeout 600 python bench.py --config 7b-sd > $O/bench33_7bsd.log 2>&1; tail -1 $O/bench33_7bsd.log | cut -c1-200
timeout 900 python bench.py --config 70b-long --steps 1 --warmup 1 --no-cpu > $O/bench33_70b.log 2>&1; tail -1 $O/bench33_70b.log | cut -c1-200
timeout 600 python bench.py --config 7b > $O/bench33_7b.log 2>&1; tail -1 $O/bench33_7b.log | cut -c1-200
