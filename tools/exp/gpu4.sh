cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build4.log 2>&1
timeout 900 python -m pytest tests/test_multirank.py -q -x 2>&1 | grep -v "^\s*$" | tail -30 > $O/multirank.log
cat $O/multirank.log
