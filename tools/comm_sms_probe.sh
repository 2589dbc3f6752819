# N-GPU C3 weak step vs the SMs the dW GEMMs leave to NCCL (TLG_COMM_SMS)
NG=${NG:-2}
timeout 900 python -m pytest tests -m gpu -q -k "multigpu or nccl or bucket or in_process" 2>&1 | tail -2
for round in 1 2; do
for c in 0 8 16; do
  TLG_COMM_SMS=$c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $NG --steps 20 --warmup 5 --no-infer --no-cpu-baseline > gpurun_out/cs_$c.json 2> gpurun_out/cs_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/cs_$c.json').read().strip().splitlines()[-1])
o=d.get('strong_scaling') or {}; g=d['kernels']['gemm_ms']
print('$round COMM_SMS=$c', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'strong', round(o.get('value',0)/1e6,1), round(o.get('ms_per_step',0),4), 'dw1', round(g['dw1']*1e3,1), 'dw2', round(g['dw2']*1e3,1))"
done
done
