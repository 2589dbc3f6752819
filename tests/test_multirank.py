"""Data-parallel learners: one rank per GPU, each rank a shard
of the replay draw (learner.cpp:119-125), one sum-allreduce of the flat gradient, then
the identical optimizer step everywhere (learner.cpp:138-152).

* CPU (gloo, world_size 2): the decomposition itself -- per-rank shard gradients from
  the oracle, allreduced over gloo -- reproduces the reference's serial rank-ordered
  multi-shard step.
* GPU (NCCL, 2 GPUs): the CUDA learner's own NCCL allreduce against the oracle, and
  bit-identical parameters on every rank.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _segments(seed, S, T, D, A):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2011_12895_b200.synth import make_segments
    return make_segments(S, T, D, A, seed=seed)


def _to_oracle(b):
    from oracle_ffi import Segments
    return Segments(b.obs.astype(np.float64), b.action.astype(np.uint32),
                    b.reward.astype(np.float64), b.behavior_logp.astype(np.float64),
                    b.value_est.astype(np.float64), b.done.astype(np.uint8),
                    b.bootstrap.astype(np.float64), b.valid_steps.astype(np.uint32))


def _cpu_rank(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    from oracle_ffi import Hyper, Oracle, Shape
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    S, T, D, A = 5, 7, 8, 4
    shape = Shape(2, D, A, (12,))
    hp = Hyper(learning_rate=0.05, batch_size=S, unroll_len=T)
    p = orc.init_params(shape, 0.3, 3)
    for step in range(3):
        # the global draw of this step; rank r takes the contiguous slice r
        seg = _segments(100 + step * 10 + rank, S, T, D, A)
        st, g = orc.shard_loss_grad(shape, p, hp, 0, _to_oracle(seg))
        t = torch.from_numpy(g.copy())
        dist.all_reduce(t)
        p = orc.sgd_step(p, t.numpy() / world, hp.learning_rate)
    q.put((rank, p))
    dist.destroy_process_group()


def test_data_parallel_decomposition_on_gloo(oracle):
    import torch.multiprocessing as mp
    from oracle_ffi import Hyper, Shape
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cpu_rank, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    # every rank holds the same parameters ...
    assert np.array_equal(res[0], res[1])
    # ... equal to the reference's serial num_shards=2 learner step
    S, T, D, A = 5, 7, 8, 4
    shape = Shape(2, D, A, (12,))
    hp = Hyper(learning_rate=0.05, batch_size=S, unroll_len=T)
    p = oracle.init_params(shape, 0.3, 3)
    for step in range(3):
        shards = [_to_oracle(_segments(100 + step * 10 + r, S, T, D, A)) for r in range(world)]
        p, _, _, _ = oracle.learner_step(shape, p, hp, 0, shards)
    assert np.allclose(res[0], p, rtol=0, atol=1e-13)


def _gpu_rank(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    import paper_2011_12895_b200 as tlg
    from oracle_ffi import Oracle, Shape
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    S, T, D, A, hidden = 6, 9, 16, 5, (32, 32)
    lrn = tlg.Learner("mlp", D, A, hidden, algo="ppo", optimizer="adam", max_segments=S,
                      unroll_len=T, device=rank)
    lrn.set_hyper(learning_rate=3e-3, batch_size=S, unroll_len=T)
    p = Oracle().init_params(Shape(2, D, A, hidden), 0.3, 5).astype(np.float32)
    lrn.set_params(p.astype(np.float64))
    uid = [tlg.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    lrn.comm_init(uid[0], world, rank)
    grads = []
    for step in range(3):
        lrn.train_step(_segments(100 + step * 10 + rank, S, T, D, A))
        grads.append(lrn.get_grad())
    q.put((rank, lrn.get_params(), grads))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_learners_match_oracle_and_each_other(oracle):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    import torch.multiprocessing as mp
    from oracle_ffi import Hyper, Shape
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_rank, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, p, g = q.get(timeout=600)
        res[r] = (p, g)
    for pr in procs:
        pr.join(timeout=120)
    assert np.array_equal(res[0][0], res[1][0])  # identical update on every rank
    S, T, D, A, hidden = 6, 9, 16, 5, (32, 32)
    shape = Shape(2, D, A, hidden)
    hp = Hyper(learning_rate=3e-3, batch_size=S, unroll_len=T)
    p = oracle.init_params(shape, 0.3, 5).astype(np.float32).astype(np.float64)
    m = np.zeros_like(p); v = np.zeros_like(p)
    for step in range(3):
        shards = [_to_oracle(_segments(100 + step * 10 + r, S, T, D, A)) for r in range(world)]
        _, g, _, _ = oracle.learner_step(shape, p, hp, 0, shards)
        gpu_g = res[0][1][step]
        assert np.all(np.abs(gpu_g - g) <= 1e-4 * max(1e-30, np.max(np.abs(g)))), step
        p, m, v = oracle.adam_step(p, gpu_g, m, v, step + 1, 3e-3)
    got = res[0][0]
    assert np.all(np.abs(got - p) <= 1e-4 * np.maximum(1, np.abs(p)))
