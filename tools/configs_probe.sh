# the other BASELINE configurations' bench lines (1 GPU)
for c in C1 C2 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-infer > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/cfg_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value']/1e6,2), 'M frames/s', round(d['ms_per_step'],4), 'ms; e2e', round(d['e2e']['value']/1e6,2), d['clocks'])"
done
