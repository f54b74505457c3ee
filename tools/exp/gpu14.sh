cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f $O/ab_oldnew.jsonl
run() { # lib tag config
  BMC_LIB=$1 timeout 1200 python bench.py --config $3 --steps 2 --warmup 1 --no-e2e --no-cpu --no-check > $O/b.log 2>&1
  tail -1 $O/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$2', 'config': '$3', 'value': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz']}))" | tee -a $O/ab_oldnew.jsonl
}
for i in 1 2; do
  run tools/exp/libbmc_old.so old l3-8b
  run paper_2511_12031_b200/libbmc.so new l3-8b
done
run tools/exp/libbmc_old.so old 70b-long
run paper_2511_12031_b200/libbmc.so new 70b-long
