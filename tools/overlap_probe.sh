# N-GPU C3 weak step: one allreduce after the backward (default) vs bucketed allreduces overlapped with it
NG=${NG:-4}
for round in $(seq 1 ${ROUNDS:-3}); do
for e in X=0 TLG_OVERLAP=1; do
  env $e timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29567 bench.py --gpus $NG --steps ${STEPS:-20} --warmup 5 --no-infer --no-cpu-baseline > gpurun_out/ov.json 2> gpurun_out/ov.err
  python -c "
import json; d=json.loads(open('gpurun_out/ov.json').read().strip().splitlines()[-1])
o=d.get('strong_scaling') or {}
print('$round $e', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'strong', round(o.get('value',0)/1e6,1), round(o.get('ms_per_step',0),4))"
done
done
