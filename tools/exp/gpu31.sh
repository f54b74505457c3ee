cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build31.log 2>&1 || tail -5 $O/build31.log
timeout 900 python tools/exp/r128b.py > $O/r128c.txt 2> $O/r128c.err; grep '^r ' $O/r128c.txt; tail -3 $O/r128c.err
