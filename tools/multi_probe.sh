# N-GPU evidence on one box: multi-GPU tests, then bench at N=1..$NG (weak default with the
# strong-scaling figure beside it), each line saved under gpurun_out/
NG=${NG:-4}
timeout 900 python -m pytest tests -m gpu -q -k "multigpu or multirank or nccl or two_gpu" 2>&1 | tail -3
for n in 1 2 4 8; do
  [ $n -gt $NG ] && break
  if [ $n = 1 ]; then
    timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/mp_n1.json 2> gpurun_out/mp_n1.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/mp_n$n.json 2> gpurun_out/mp_n$n.err
  fi
  python - <<PY
import json
d = json.loads(open("gpurun_out/mp_n$n.json").read().strip().splitlines()[-1])
print($n, "value", round(d["value"] / 1e6, 1), "ms", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"] / 1e6, 1),
      "strong", {k: (round(v / 1e6, 1) if isinstance(v, float) else v) for k, v in (d.get("strong_scaling") or {}).items() if k in ("value", "ms_per_step", "segments_per_gpu")})
PY
done
