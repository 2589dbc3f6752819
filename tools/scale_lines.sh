# bench lines for the scaling table (default settings, 60 steps; N=4 measured twice, the
# second kept: the first run on a fresh multi-GPU box reads slow)
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2957$1 bench.py --gpus $1 --steps 60 --warmup 5 > gpurun_out/scale_n$1.json 2> gpurun_out/scale_n$1.err; }
run 4; run 4; run 2
for n in 2 4; do python -c "
import json; d=json.loads(open('gpurun_out/scale_n$n.json').read().strip().splitlines()[-1])
o=d.get('strong_scaling') or {}
print($n, round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1), 'strong', round(o.get('value',0)/1e6,1), round(o.get('ms_per_step',0),4))"; done
