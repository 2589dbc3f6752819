# A/B of library variants on one box: paper_2011_12895_b200/_lib/variants/lib_<v>.so is
# swapped in for each of $VARIANTS (two rounds, interleaved); C3 step + C4 batch timing.
L=paper_2011_12895_b200/_lib
cp $L/libtlg_b200.so /tmp/libtlg_b200.keep.so
for round in 1 2; do
  for v in ${VARIANTS:-cur}; do
    cp $L/variants/lib_$v.so $L/libtlg_b200.so
    c4=$(timeout 120 python tools/policy_probe.py 2>/dev/null | tail -1)
    c3=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-infer 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);g=d['kernels']['gemm_ms'];print(round(d['ms_per_step'],4), {k: round(x*1e3,1) for k,x in g.items()})")
    echo "$round $v | C3 $c3 | $c4"
  done
done
cp /tmp/libtlg_b200.keep.so $L/libtlg_b200.so
