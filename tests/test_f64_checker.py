"""Pins the batched torch-float64 checker (tests/f64_checker.py) to the fp64 oracle
(oracle/tlg_oracle.cpp, itself pinned to the reference) at small shapes, on the CPU, so
that the GPU parity tests at the BASELINE shapes can use the checker where the
per-sample oracle would take minutes."""
import numpy as np
import pytest
import torch

import f64_checker as fc
from oracle_ffi import Hyper, Segments, Shape

ALGO = {"ppo": 0, "vtrace": 1, "ppo_vtrace": 2}


def _segments(b):
    return Segments(b.obs.astype(np.float64), b.action.astype(np.uint32),
                    b.reward.astype(np.float64), b.behavior_logp.astype(np.float64),
                    b.value_est.astype(np.float64), b.done.astype(np.uint8),
                    b.bootstrap.astype(np.float64), b.valid_steps.astype(np.uint32))


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))


@pytest.mark.parametrize("algo", list(ALGO))
@pytest.mark.parametrize("case", [
    (2, 16, 6, (32, 24, 16, 8)),   # 4 trunk layers (C5's depth)
    (2, 24, 5, (40,)),
    (1, 10, 4, ()),                # linear_softmax (policy.cpp:82-104)
], ids=["mlp4", "mlp1", "linear"])
def test_checker_matches_oracle(oracle, algo, case):
    from paper_2011_12895_b200 import synth
    family, D, A, hidden = case
    shape = Shape(family, D, A, hidden)
    net = fc.Net(family, D, A, hidden)
    assert net.P == oracle.param_count(shape)
    S, T = 9, 7
    hpd = dict(learning_rate=0.05, gamma=0.97, lam=0.9, clip_eps=0.2, vf_coef=0.5,
               ent_coef=0.01, rho_bar=1.0, c_bar=0.9, batch_size=S, unroll_len=T,
               adv_norm=True)
    p = oracle.init_params(shape, 0.5, 11).astype(np.float32).astype(np.float64)
    shards = [synth.make_segments(S, T, D, A, seed=40 + k, done_p=0.15, ragged_frac=0.4)
              for k in range(2)]
    shards[1].valid_steps[3] = 0  # an empty segment contributes nothing
    shards[1].reward[3] = 0; shards[1].value_est[3] = 0; shards[1].behavior_logp[3] = 0
    shards[1].obs[3] = 0; shards[1].done[3] = 0; shards[1].action[3] = 0
    dev = torch.device("cpu")
    pt = torch.tensor(p, dtype=torch.float64)
    stats, g, (adv, tgt, _) = fc.learner_step(net, pt, hpd, ALGO[algo], shards, dev)
    p_new, g_want, st_want, _ = oracle.learner_step(shape, p, Hyper(**hpd), ALGO[algo],
                                                    [_segments(b) for b in shards])
    assert rel(g.numpy(), g_want) < 1e-10
    for st, sw in zip(stats, st_want):
        for k in ("loss", "clip_fraction", "mean_ratio", "entropy", "value_loss"):
            assert abs(st[k] - sw[k]) <= 1e-10 * max(1.0, abs(sw[k])), (k, st[k], sw[k])
        assert st["n_samples"] == sw["n_samples"]
    wa, wt = oracle.shard_returns(shape, p, Hyper(**hpd), ALGO[algo], _segments(shards[1]))
    assert rel(adv.numpy(), wa) < 1e-12 and rel(tgt.numpy(), wt) < 1e-12
    assert rel(fc.sgd(pt, g, 0.05).numpy(), p_new) < 1e-12
    m = np.zeros_like(p); v = np.zeros_like(p)
    pa, ma, va = oracle.adam_step(p, g_want, m, v, 3, 1e-3)
    pb, mb, vb = fc.adam(pt, torch.tensor(g_want), torch.zeros_like(pt), torch.zeros_like(pt), 3,
                         1e-3)
    assert rel(pb.numpy(), pa) < 1e-13 and rel(mb.numpy(), ma) < 1e-13
