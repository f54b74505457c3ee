cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build32.log 2>&1 || tail -5 $O/build32.log
BMC_LIB=tools/exp/libbmc_oldhash.so timeout 600 python tools/exp/r128.py 128,256 > $O/r128_old.jsonl 2>&1; cat $O/r128_old.jsonl | cut -c1-160
timeout 600 python tools/exp/r128.py 64,128,256 > $O/r128_new.jsonl 2>&1; cat $O/r128_new.jsonl | cut -c1-160
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest32.log 2>&1; tail -2 $O/pytest32.log
