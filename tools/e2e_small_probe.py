#!/usr/bin/env python
"""Host-batch paths at a small config: train_step(host), staged pipeline, device-resident."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_12895_b200 as tlg  # noqa: E402
from paper_2011_12895_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
S, T, D, A, hidden = cfg.batch_size, cfg.unroll_len, cfg.obs_dim, cfg.n_actions, cfg.hidden
lrn = tlg.Learner("mlp", D, A, hidden, algo=cfg.algo, optimizer=cfg.optimizer, max_segments=S,
                  unroll_len=T)
lrn.set_hyper(learning_rate=3e-4, batch_size=S, unroll_len=T)
lrn.set_params(tlg.synth.init_params_f32(lrn.n_params, 0.05, seed=1).astype(np.float64))
hs = [tlg.synth.make_segments(S, T, D, A, seed=i, obs_kind=cfg.obs_kind) for i in range(2)]
views = []
for h in hs:
    v = tlg.SegmentBatchView(h.slice(0, S))
    v.pinned = []
    for k, a in v.arrs.items():
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        v.pinned.append(t)
        v.arrs[k] = t.numpy()
    v.c = tlg._capi.SegmentBatchC(S, T, D, 0, *(v.arrs[k].ctypes.data for k in (
        "obs", "action", "reward", "behavior_logp", "value_est", "done", "bootstrap", "valid_steps")))
    views.append(v)
dev = [tlg.DeviceSegmentBatch(h, 0) for h in hs]
n = 30
F = S * T


def timeit(name, fn):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        fn(i)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{name:28s} {dt * 1e3:.3f} ms/step  {F / dt / 1e6:.1f} M frames/s")


timeit("device-resident", lambda i: lrn.train_step(dev[i % 2], on_device=True))
timeit("train_step(host pinned)", lambda i: lrn.train_step(views[i % 2]))


def staged(i):
    lrn.stage(views[i % 2])
    lrn.train_staged()


timeit("stage+train (no overlap)", staged)
