#!/usr/bin/env python
"""InfServer C4 batched forward, a few launches (for ncu launch lists / captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_12895_b200 as tlg  # noqa: E402
from paper_2011_12895_b200.configs import CONFIGS  # noqa: E402

c4 = CONFIGS["C4"]
pol = tlg.Policy("mlp", c4.obs_dim, c4.n_actions, c4.hidden, device=0, max_batch=c4.batch_size)
n_p = (c4.obs_dim * c4.hidden[0] + c4.hidden[0] + c4.hidden[0] * c4.hidden[1] + c4.hidden[1] +
       (c4.n_actions + 1) * c4.hidden[1] + c4.n_actions + 1)
pol.set_params(tlg.synth.init_params_f32(n_p, 0.05, seed=c4.seed).astype(np.float64))
ob = torch.from_numpy(tlg.synth.make_obs(c4.batch_size, c4.obs_dim, seed=c4.seed)).cuda()
lg = torch.empty(c4.batch_size, c4.n_actions, device="cuda")
pr = torch.empty_like(lg)
v = torch.empty(c4.batch_size, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    pol.forward_device(ob, lg, pr, v)
torch.cuda.synchronize()
print("ok", float(v.abs().sum()))
