cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build9.log 2>&1 || tail -5 $O/build9.log
timeout 600 python tools/exp/growth_cost.py > $O/growth_pool.log 2>&1
timeout 600 python tools/exp/growth_cost.py --vmm > $O/growth_vmm.log 2>&1
timeout 600 python tools/exp/growth_cost.py --reserve > $O/growth_reserve.log 2>&1
cat $O/growth_pool.log $O/growth_vmm.log $O/growth_reserve.log
