cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build20.log 2>&1 || tail -5 $O/build20.log
timeout 400 python tools/exp/growth_cost.py --l3 --vmm > $O/growth20_l3_vmm.txt 2>&1; grep -v 'host ms' $O/growth20_l3_vmm.txt
timeout 400 python tools/exp/growth_cost.py --l3 > $O/growth20_l3_pool_noreserve.txt 2>&1; grep -v 'host ms' $O/growth20_l3_pool_noreserve.txt
for a in vmm pool; do
  timeout 600 python bench.py --config l3-8b --arena $a --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/b20.log 2>&1
  tail -1 $O/b20.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'arena': '$a', 'value': d['value'], 'frac': d['roofline']['frac'], 'growth_frac': d['roofline'].get('growth', {}).get('frac'), 'sm_mhz': d['clocks']['sm_mhz']}))" | tee -a $O/arena20.jsonl
done
BMC_LIB=tools/exp/libbmc_pf16.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_steps.py tests/test_gpu_fullsize.py -q -x > $O/par20_pf16.log 2>&1; tail -15 $O/par20_pf16.log
for lib in base pf16; do L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so; BMC_LIB=$L timeout 600 python tools/exp/err_probe.py $lib >> $O/err20.jsonl 2>&1; done; cat $O/err20.jsonl
for lib in base pf16 pf16k3; do
  L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so
  BMC_LIB=$L timeout 600 python tools/exp/abshape.py $lib >> $O/abshape20.jsonl 2> $O/abshape20_$lib.err || tail -3 $O/abshape20_$lib.err
done
cat $O/abshape20.jsonl
for lib in base pf16 pf16k3; do
  L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so
  BMC_LIB=$L timeout 900 python bench.py --config 70b-long --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/b20.log 2>&1
  tail -1 $O/b20.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$lib', 'config': '70b-long', 'value': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))" | tee -a $O/ab20.jsonl
done
