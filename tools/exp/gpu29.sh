cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build29.log 2>&1 || tail -5 $O/build29.log
timeout 1200 python tools/exp/r128.py 64,128,256,128 > $O/r128.jsonl 2> $O/r128.err; cat $O/r128.jsonl; tail -3 $O/r128.err
