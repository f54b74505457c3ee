cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/exp/ab72.py > $O/ab72.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05 or speculative or token_tree" 2>&1 | tail -3 > $O/par7.log
timeout 900 python -m pytest tests/test_gpu_steps.py tests/test_gpu_fullsize.py -q -x -k "70b" 2>&1 | tail -3 >> $O/par7.log
timeout 900 python bench.py --config 70b-long --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/b70_g3.log 2>&1
timeout 900 python bench.py --config 70b-long --steps 1 --warmup 1 --no-e2e --no-cpu --no-check --tck-groups 2 > $O/b70_g2.log 2>&1
cat $O/ab72.log $O/par7.log; for f in $O/b70_g3.log $O/b70_g2.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks'])"; done
