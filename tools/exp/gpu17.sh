cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build17.log 2>&1 || tail -5 $O/build17.log
rm -f $O/abpoly17.jsonl
for rep in 1 2; do for lib in base lt p4 p3 p2; do
  L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so
  BMC_LIB=$L timeout 600 python tools/exp/abpoly.py $lib >> $O/abpoly17.jsonl 2> $O/abpoly17_$lib.err || tail -3 $O/abpoly17_$lib.err
done; done
cat $O/abpoly17.jsonl
for lib in p3 p2; do
BMC_LIB=tools/exp/libbmc_$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_steps.py -q -x -k "tcgen05 or speculative or 70b or tree or baselines" > $O/par17_$lib.log 2>&1; tail -2 $O/par17_$lib.log
done
for lib in base p3 p2 base p3 p2; do
  L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so
  BMC_LIB=$L timeout 900 python bench.py --config 70b-long --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/b17.log 2>&1
  tail -1 $O/b17.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$lib', 'value': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))" | tee -a $O/ab70_17.jsonl
done
