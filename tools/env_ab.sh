# A/B of an environment switch on one box (two interleaved rounds): C3 step + C4 batch
# usage: ENVS="TLG_NO_ALR=1 X=0" bash tools/env_ab.sh   ("X=0" = a no-op baseline)
for round in 1 2; do
  for e in $ENVS; do
    c4=$(env $e timeout 120 python tools/policy_probe.py 2>/dev/null | tail -1)
    c3=$(env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-infer 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);g=d['kernels']['gemm_ms'];print(round(d['ms_per_step'],4), {k: round(x*1e3,1) for k,x in g.items()})")
    echo "$round $e | C3 $c3 | $c4"
  done
done
