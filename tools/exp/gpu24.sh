cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build24.log 2>&1 || tail -5 $O/build24.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest24.log 2>&1; tail -5 $O/pytest24.log
for rep in 1 2; do for lib in base m64q4 m64q2; do
  L=tools/exp/libbmc_$lib.so; [ $lib = base ] && L=paper_2511_12031_b200/libbmc.so
  BMC_LIB=$L timeout 600 python tools/exp/abm.py $lib >> $O/abm24.jsonl 2> $O/abm24_$lib.err || tail -3 $O/abm24_$lib.err
done; done
cat $O/abm24.jsonl
BMC_LIB=tools/exp/libbmc_m64q4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05" > $O/par24_m64q4.log 2>&1; tail -2 $O/par24_m64q4.log
for a in region pool; do
  timeout 900 python bench.py --config 70b-long --arena $a --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/b24.log 2>&1
  tail -1 $O/b24.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'config': '70b-long', 'arena': '$a', 'value': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz'], 'gm': d['growth_memory']}))" | tee -a $O/arena24.jsonl || tail -3 $O/b24.log
done
