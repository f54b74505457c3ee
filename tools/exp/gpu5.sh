cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build5.log 2>&1 || tail -20 $O/build5.log
timeout 300 python tools/exp/mb70.py 8192,32768 > $O/mb70_v2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05 or speculative or token_tree" 2>&1 | tail -5 > $O/par5.log
timeout 900 python -m pytest tests/test_gpu_steps.py -q -x -k "70b" 2>&1 | tail -5 >> $O/par5.log
cat $O/mb70_v2.log $O/par5.log
