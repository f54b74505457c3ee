cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build27.log 2>&1 || tail -5 $O/build27.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest27.log 2>&1; tail -5 $O/pytest27.log
timeout 300 python tools/exp/one70.py 32768 9 > $O/one70_27.log 2>&1; tail -2 $O/one70_27.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tck -s 4 -c 1 \
  -o $O/ncu27_tck72 python tools/exp/one70.py 32768 9 > $O/ncu27_tck72.log 2>&1; tail -2 $O/ncu27_tck72.log
ncu -i $O/ncu27_tck72.ncu-rep --page raw --csv > $O/ncu27_tck72.raw.csv 2>/dev/null
ncu -i $O/ncu27_tck72.ncu-rep --page details --csv > $O/ncu27_tck72.details.csv 2>/dev/null
ls -la $O/ncu27_tck72*
