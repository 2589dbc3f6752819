# quick A/B: gemm selftest (+ C3 L2 perf shapes), GPU parity of the policy/learner, C3 + C4 bench
B=paper_2011_12895_b200/_lib/gemm_selftest
timeout 300 $B perf 2>&1 | grep -E "FAIL|PASSED|perf (fwd|dX) C3 L2|perf fwd C4"
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);k=d.get('kernels',{});print('C3', d['value']/1e6, d['ms_per_step'], k.get('gemm_ms'));i=k.get('infserver') or d.get('infserver');print('C4', i['value']/1e6, i['ms_per_batch'])"
