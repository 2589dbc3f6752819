"""Data parallelism across GPUs inside one process: one learner per
device, one ncclCommInitAll (tlg_learner_comm_init_all), one host thread per device
issuing that device's shard step -- the reference's shard threads of
learner.cpp:117-134 mapped onto GPUs.  Per-layer gradient buckets are allreduced on a
comm stream while the backward continues when TLG_OVERLAP=1 (the default is one
allreduce after the backward: measured faster on NVLink B200s).

Checked against the fp64 checker's serial rank-ordered multi-shard step
(tests/f64_checker.py, pinned to the oracle) at the C3 strong-scaling shard size, and
overlap on / off must give bit-identical parameters.
"""
import threading

import numpy as np
import pytest
import torch

import f64_checker as fc

pytestmark = pytest.mark.gpu

ALGO = {"ppo": 0, "vtrace": 1, "ppo_vtrace": 2}


def _need(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs (gpurun --gpus {n})")


def _bits(tlg, b, D):
    from paper_2011_12895_b200._capi import SegmentBatchView
    pb = b.slice(0, b.n_segments)
    pb.obs = tlg.synth.pack_bits(b.obs)
    return SegmentBatchView(pb, bits=True, obs_dim=D)


def _run(tlg, G, *, D, A, hidden, S, T, algo, steps, bits, overlap, monkeypatch, seed=0):
    if overlap:
        monkeypatch.setenv("TLG_OVERLAP", "1")
    else:
        monkeypatch.delenv("TLG_OVERLAP", raising=False)
    net = fc.Net(2, D, A, hidden)
    rng = np.random.default_rng(seed)
    p0 = (rng.uniform(-1, 1, net.P) * 0.1).astype(np.float32).astype(np.float64)
    for l in range(len(hidden)):
        w0, n_w = net.w_off[l], net.dims[l + 1] * net.dims[l]
        p0[w0:w0 + n_w] = (rng.uniform(-1, 1, n_w) * 1.5 / np.sqrt(net.dims[l])).astype(
            np.float32)
    hp = dict(learning_rate=3e-3, batch_size=S, unroll_len=T)
    ls = []
    for g in range(G):
        l = tlg.Learner("mlp", D, A, hidden, algo=algo, optimizer="sgd", max_segments=S,
                        unroll_len=T, device=g, obs_u8=bits)
        l.set_hyper(**hp)
        l.set_params(p0)
        ls.append(l)
    tlg.comm_init_all(ls)
    hist = []
    for step in range(steps):
        shards = [tlg.synth.make_segments(S, T, D, A, seed=seed * 100 + step * 10 + g,
                                          obs_kind="binary" if bits else "gauss", obs_u8=bits)
                  for g in range(G)]
        views = [_bits(tlg, b, D) if bits else b for b in shards]
        p_prev = ls[0].get_params()
        out, errs = [None] * G, []

        def work(g):
            try:
                out[g] = ls[g].train_step(views[g])
            except Exception as e:  # noqa: BLE001
                errs.append(e)
        th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        ps = [l.get_params() for l in ls]
        for g in range(1, G):
            assert np.array_equal(ps[0], ps[g]), "ranks diverged"
        hist.append((p_prev, ps[0], ls[0].get_grad(), shards, out))
    return hist, hp


@pytest.mark.parametrize("G", [2, 4])
def test_in_process_data_parallel_matches_serial_shards(tlg, monkeypatch, G):
    """C3 net, strong-scaling split: a 4096-segment draw's shard of 4096/G segments per
    GPU (S = 512 here for speed at G=2/4: the shapes of 8 GPUs), bit-packed planes."""
    _need(G)
    D, A, hidden, S, T = 1936, 6, (256, 256), 512, 32
    hist, hp = _run(tlg, G, D=D, A=A, hidden=hidden, S=S, T=T, algo="ppo", steps=2, bits=True,
                    overlap=True, monkeypatch=monkeypatch, seed=4)
    dev = torch.device("cuda", 0)
    net = fc.Net(2, D, A, hidden)
    for p_prev, p_new, g_gpu, shards, sts in hist:
        pt = torch.tensor(p_prev, dtype=torch.float64, device=dev)
        stats, g, _ = fc.learner_step(net, pt, dict(hp, gamma=0.99, lam=0.95, clip_eps=0.2,
                                                    vf_coef=0.5, ent_coef=0.01, rho_bar=1.0,
                                                    c_bar=1.0, adv_norm=True),
                                      0, shards, dev)
        g = g.cpu().numpy()
        assert np.max(np.abs(g_gpu - g)) <= 1e-4 * np.max(np.abs(g))
        want = p_prev - hp["learning_rate"] * g
        assert np.all(np.abs(p_new - want) <= 1e-4 * np.maximum(1, np.abs(want)))
        for st, sw in zip(sts, stats):  # each rank reports its own shard's statistics
            assert abs(st["loss"] - sw["loss"]) <= 1e-4 * max(1, abs(sw["loss"]))


def test_bucket_overlap_is_bit_identical_to_one_allreduce(tlg, monkeypatch):
    """Bucketing changes when each gradient region is reduced, not how: with 2 ranks the
    per-element sum is the same, so parameters must match bit for bit."""
    _need(2)
    kw = dict(D=64, A=6, hidden=(256, 256, 128), S=32, T=16, algo="ppo_vtrace", steps=3,
              bits=False, seed=9)
    a, _ = _run(tlg, 2, overlap=True, monkeypatch=monkeypatch, **kw)
    b, _ = _run(tlg, 2, overlap=False, monkeypatch=monkeypatch, **kw)
    for (_, pa, ga, _, _), (_, pb, gb, _, _) in zip(a, b):
        assert np.array_equal(pa, pb)
        assert np.array_equal(ga, gb)
