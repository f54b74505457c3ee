cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for lib in trace trace_new; do for cap in 1024 4096; do
BMC_LIB=tools/exp/libbmc_$lib.so timeout 300 python tools/tck_trace.py 64 8 32 $cap 1 0 > $O/tr_${lib}_$cap.txt 2>&1
done; done
for f in $O/tr_trace_1024.txt $O/tr_trace_new_1024.txt; do head -45 $f | cut -c1-190; done
