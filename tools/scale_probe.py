"""Strong-scaling probe (diagnostics, not the bench): C3 single-GPU step time at the
per-rank shard sizes of 1/2/4/8 GPUs, and the flat-gradient allreduce time on its own.

    python tools/scale_probe.py steps            # one GPU
    torchrun --nproc-per-node N tools/scale_probe.py allreduce
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def steps():
    import paper_2011_12895_b200 as tlg
    from paper_2011_12895_b200.configs import CONFIGS
    cfg = CONFIGS["C3"]
    T, D, A, hidden = cfg.unroll_len, cfg.obs_dim, cfg.n_actions, cfg.hidden
    pitch = ((D + 7) // 8 + 15) // 16 * 16
    out = {}
    sizes = [int(x) for x in os.environ.get("TLG_PROBE_S", "512,1024,2048,4096").split(",")]
    for S in sizes:
        l = tlg.Learner("mlp", D, A, hidden, algo="ppo", optimizer="adam", max_segments=S,
                        unroll_len=T, obs_u8=True)
        l.set_hyper(learning_rate=3e-4, batch_size=S, unroll_len=T)
        l.set_params(tlg.synth.init_params_f32(l.n_params, 0.05, seed=1).astype(np.float64))
        nb = max(4, -(-136_000_000 // (S * T * (pitch + 17))))
        dev = []
        for i in range(nb):
            h = tlg.synth.make_segments(S, T, D, A, seed=i, obs_kind="binary", obs_u8=True)
            hb = h.slice(0, S)
            hb.obs = tlg.synth.pack_bits(h.obs)
            dev.append(tlg.DeviceSegmentBatch(hb, 0, bits=True, obs_dim=D, pitch=pitch))
        for i in range(2 * nb):
            l.train_step(dev[i % nb], on_device=True)
        st = torch.cuda.ExternalStream(l.stream())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        n = int(os.environ.get("TLG_PROBE_STEPS", "50"))
        for i in range(n):
            l.train_step(dev[i % nb], on_device=True)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        l.set_timing(True)
        ph = []
        for i in range(10):
            l.train_step(dev[i % nb], on_device=True)
            ph.append(l.phase_ms())
        out[S] = {"ms_per_step": ms, "frames_per_s": S * T / ms * 1e3,
                  "phases_ms": np.mean(ph, 0).round(4).tolist()}
        l.close()
        del dev
        torch.cuda.empty_cache()
    print(json.dumps({"probe": "steps", "C3": out}))


def allreduce():
    """ncclAllReduce of the C3 flat gradient through the library's own NCCL binding,
    timed by a learner step with the compute removed is not possible, so this times
    torch.distributed's NCCL on the same byte count (same NCCL build in-process)."""
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    n = 563_463 + 4
    x = torch.ones(n, device="cuda")
    res = {}
    for _ in range(20):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    for reps in (200,):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        dist.barrier()
        e0.record()
        for _ in range(reps):
            dist.all_reduce(x)
        e1.record()
        torch.cuda.synchronize()
        res["eager_us"] = e0.elapsed_time(e1) / reps * 1e3
    # graph-captured, like the learner's step graph
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        dist.all_reduce(x)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                dist.all_reduce(x)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res["graph_us"] = e0.elapsed_time(e1) / 200 * 1e3
    if rank == 0:
        print(json.dumps({"probe": "allreduce", "world": world, "bytes": n * 4,
                          "env": {k: os.environ.get(k) for k in ("NCCL_ALGO", "NCCL_PROTO")},
                          **res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    {"steps": steps, "allreduce": allreduce}[sys.argv[1]]()
