cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build3.log 2>&1
timeout 900 python -m pytest tests/test_multirank.py -q -x 2>&1 | tail -5 > $O/multirank.log
timeout 900 python bench.py --steps 1 --warmup 1 --e2e-steps 1 > $O/bench_l3.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu \
  > $O/bench_2rank.log 2>&1
cat $O/multirank.log; tail -1 $O/bench_l3.log | cut -c1-3000; tail -3 $O/bench_2rank.log | cut -c1-3000
