cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build26.log 2>&1 || tail -5 $O/build26.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest26.log 2>&1; tail -5 $O/pytest26.log
bash tools/sanitize.sh > $O/sanitize26.txt 2>&1; cat $O/sanitize26.txt
