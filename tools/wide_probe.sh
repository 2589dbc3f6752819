# fwd2 / dX2 tile-width A/B at C3 (gemm_selftest perf shapes, then the C3 step)
B=paper_2011_12895_b200/_lib/gemm_selftest
for w in 0 1; do
  if [ $w = 1 ]; then export TLG_GEMM_WIDE=1; fi
  timeout 300 $B perf 2>&1 | grep -E "perf (fwd|dX) C3 L2" 
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-infer 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('WIDE=$w', d['value']/1e6, d['ms_per_step'], d.get('kernels',{}).get('gemm_ms'))"
done
