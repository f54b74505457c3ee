cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build19.log 2>&1 || tail -5 $O/build19.log
BMC_LIB=tools/exp/libbmc_pf16.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_steps.py tests/test_gpu_fullsize.py -q -x > $O/par19_pf16.log 2>&1; tail -15 $O/par19_pf16.log
for lib in base pf16; do L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so; BMC_LIB=$L timeout 600 python tools/exp/err_probe.py $lib >> $O/err19.jsonl 2>&1; done; cat $O/err19.jsonl
rm -f $O/abshape19.jsonl
for rep in 1 2; do for lib in base pf16 pf16k3; do
  L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so
  BMC_LIB=$L timeout 600 python tools/exp/abshape.py $lib >> $O/abshape19.jsonl 2> $O/abshape19_$lib.err || tail -3 $O/abshape19_$lib.err
done; done
cat $O/abshape19.jsonl
for cl in 70b-long:base 70b-long:pf16 70b-long:pf16k3 70b-long:base 70b-long:pf16 70b-long:pf16k3 l3-8b:base l3-8b:pf16 l3-8b:base l3-8b:pf16; do
  cfg=${cl%%:*}; lib=${cl##*:}
  L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so
  BMC_LIB=$L timeout 900 python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/b19.log 2>&1
  tail -1 $O/b19.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$lib', 'config': '$cfg', 'value': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))" | tee -a $O/ab19.jsonl
done
