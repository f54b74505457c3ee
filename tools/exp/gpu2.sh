cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_steps.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -30 > gpurun_out/steps.log
cat gpurun_out/steps.log
