# N=4 weak/strong ordering check + drop-in acceptance on a multi-GPU box
timeout 900 integration/_build/dropin_test 2>&1 | tail -4
run() {  # $1 tag, rest: bench args
  tag=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --steps 20 --warmup 5 --no-infer "$@" > gpurun_out/n4_$tag.json 2> gpurun_out/n4_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/n4_$tag.json').read().strip().splitlines()[-1])
o=d.get('strong_scaling') or d.get('weak_scaling') or {}
print('$tag', d['scaling'], round(d['value']/1e6,1), round(d['ms_per_step'],4), 'other', round(o.get('value',0)/1e6,1), round(o.get('ms_per_step',0),4))"
}
run weak1
run strong1 --scaling strong
run weak2
