cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cap in 32768 8192; do
BMC_LIB=tools/exp/libbmc_trace.so timeout 300 python tools/tck_trace.py 8 8 64 $cap 9 0 > $O/trace72g3_$cap.txt 2>&1
done
tail -8 $O/trace72g3_32768.txt | cut -c1-300; head -24 $O/trace72g3_32768.txt
