cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for a in "iterative 0" "iterative 1" "upfront 0"; do echo "== $a"; timeout 600 python tools/exp/dbg_iter_sd.py $a 2>&1 | sort -t' ' -k12 -g | tail -4; done
