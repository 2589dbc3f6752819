# N=4 C3 weak step under NCCL algorithm choices (pinned Ring = the default; tuner; NVLS; Tree)
run() {
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --steps 20 --warmup 5 --no-infer --no-cpu-baseline > gpurun_out/nc_$tag.json 2> gpurun_out/nc_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/nc_$tag.json').read().strip().splitlines()[-1])
o=d.get('strong_scaling') or {}; ph=d['kernels']['phases_ms']
print('$tag', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'strong', round(o.get('value',0)/1e6,1), round(o.get('ms_per_step',0),4), 'eager allreduce', round(ph['allreduce'],3))"
}
run ring TLG_NCCL_PIN=1
run tuner TLG_NCCL_PIN=0
run nvls TLG_NCCL_PIN=0 NCCL_ALGO=NVLS
run tree TLG_NCCL_PIN=0 NCCL_ALGO=Tree
run ring2 TLG_NCCL_PIN=1
