#!/usr/bin/env python
"""InfServer C4 host path breakdown: device-only forward vs host-buffer forward vs raw copies."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_12895_b200 as tlg  # noqa: E402
from paper_2011_12895_b200.configs import CONFIGS  # noqa: E402

c4 = CONFIGS["C4"]
N, D, A = c4.batch_size, c4.obs_dim, c4.n_actions
pol = tlg.Policy("mlp", D, A, c4.hidden, device=0, max_batch=N)
n_p = (D * c4.hidden[0] + c4.hidden[0] + c4.hidden[0] * c4.hidden[1] + c4.hidden[1] +
       (A + 1) * c4.hidden[1] + A + 1)
pol.set_params(tlg.synth.init_params_f32(n_p, 0.05, seed=1).astype(np.float64))
obs = tlg.synth.make_obs(N, D, seed=2)
ob_t = torch.from_numpy(obs).cuda()
lg_t = torch.empty(N, A, device="cuda"); pr_t = torch.empty_like(lg_t); v_t = torch.empty(N, device="cuda")
obs_pin_t = torch.from_numpy(obs).pin_memory()
outs_t = [torch.empty(N, A, pin_memory=True), torch.empty(N, A, pin_memory=True),
          torch.empty(N, pin_memory=True)]
outs = tuple(t.numpy() for t in outs_t)


def t(name, fn, n=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{name:34s} {dt * 1e3:.3f} ms  {N / dt / 1e6:.1f} M actions/s")


t("forward_device", lambda: (pol.forward_device(ob_t, lg_t, pr_t, v_t), torch.cuda.synchronize()))
t("forward(host pinned in/out)", lambda: pol.forward(obs_pin_t.numpy(), out=outs))
t("forward(host pageable)", lambda: pol.forward(obs))
t("H2D obs pinned (torch)", lambda: ob_t.copy_(obs_pin_t, non_blocking=True))
t("D2H outputs pinned (torch)", lambda: (outs_t[0].copy_(lg_t, non_blocking=True),
                                          outs_t[1].copy_(pr_t, non_blocking=True),
                                          outs_t[2].copy_(v_t, non_blocking=True)))
q = N // 4
t("forward_device x4 chunks of N/4", lambda: ([pol.forward_device(ob_t[i * q:(i + 1) * q], lg_t[i * q:(i + 1) * q], pr_t[i * q:(i + 1) * q], v_t[i * q:(i + 1) * q]) for i in range(4)], torch.cuda.synchronize()))
