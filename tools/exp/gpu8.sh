cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build8.log 2>&1 || tail -5 $O/build8.log
timeout 600 python tools/exp/abpf.py > $O/abpf.log 2>&1
cat $O/abpf.log
