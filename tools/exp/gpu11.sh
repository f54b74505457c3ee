cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tck -s 4032 -c 1 \
  -o $O/ncu_cor_growth python tools/exp/growth_ncu.py decode > $O/ncu_cor.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:realloc -s 62 -c 1 \
  -o $O/ncu_realloc python tools/exp/growth_ncu.py realloc > $O/ncu_realloc.log 2>&1
for r in ncu_cor_growth ncu_realloc; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null; done
timeout 900 python bench.py --config 7b --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > $O/b7g.log 2>&1
tail -1 $O/b7g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['growth'])"
tail -2 $O/ncu_cor.log $O/ncu_realloc.log
