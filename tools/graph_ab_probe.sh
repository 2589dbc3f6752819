# N-GPU C3 weak step: CUDA graph replay vs eager launches, bucket overlap vs one allreduce, PDL
NG=${NG:-2}
for round in 1 2; do
for e in X=0 TLG_NO_GRAPH=1 TLG_OVERLAP=1 TLG_NO_PDL=1; do
  env $e timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29566 bench.py --gpus $NG --steps 20 --warmup 5 --no-infer --no-cpu-baseline > gpurun_out/gab.json 2> gpurun_out/gab.err
  python -c "
import json; d=json.loads(open('gpurun_out/gab.json').read().strip().splitlines()[-1])
print('$round $e', round(d['value']/1e6,1), round(d['ms_per_step'],4))"
done
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-infer --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('N=1', d['ms_per_step'])"
TLG_NO_PDL=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-infer --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('N=1 no PDL', d['ms_per_step'])"
