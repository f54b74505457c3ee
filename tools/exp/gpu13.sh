cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build13.log 2>&1 || tail -5 $O/build13.log
timeout 600 python tools/exp/abpair.py > $O/abpair.log 2>&1; cat $O/abpair.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_steps.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3 > $O/par13.log
cat $O/par13.log
