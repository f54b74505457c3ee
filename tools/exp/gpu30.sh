cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build30.log 2>&1 || tail -5 $O/build30.log
timeout 900 python tools/exp/r128b.py > $O/r128b.txt 2> $O/r128b.err; tail -3 $O/r128b.err
