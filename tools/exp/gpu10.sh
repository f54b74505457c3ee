cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f $O/ab_reserve.jsonl
for i in 1 2 3; do for a in "" "--pool-reserve"; do
timeout 900 python bench.py --config 7b --steps 2 --warmup 2 --no-e2e --no-cpu --no-check $a > $O/b.log 2>&1
tail -1 $O/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'reserve': '$a' != '', 'value': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz']}))" | tee -a $O/ab_reserve.jsonl
done; done
