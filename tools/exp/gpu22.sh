cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build22.log 2>&1 || tail -5 $O/build22.log
timeout 1200 python bench.py > $O/bench22_default.log 2>&1; tail -1 $O/bench22_default.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches22_l3.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-check > $O/launches22.log 2>&1; wc -l $O/launches22_l3.csv
timeout 600 python bench.py --config 7b > $O/bench22_7b.log 2>&1; tail -1 $O/bench22_7b.log | cut -c1-300
timeout 600 python bench.py --config 7b-sd > $O/bench22_7bsd.log 2>&1; tail -1 $O/bench22_7bsd.log | cut -c1-300
timeout 900 python bench.py --config 70b-long --steps 1 --warmup 1 --no-cpu > $O/bench22_70b.log 2>&1; tail -1 $O/bench22_70b.log | cut -c1-300
timeout 1200 python tools/sweep.py --config 7b-sd --rs 16,32,64,128,256 > $O/sweep22_7bsd.json 2> $O/sweep22_7bsd.err || tail -3 $O/sweep22_7bsd.err
tail -1 $O/sweep22_7bsd.json | cut -c1-200
