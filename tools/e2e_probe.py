#!/usr/bin/env python
"""Probe of the pipelined host-batch path (stage / train_staged) at C3: per-step wall
time of (a) the H2D copies alone, (b) device-resident steps, (c) the staged pipeline."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_12895_b200 as tlg  # noqa: E402
from paper_2011_12895_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["C3"]
S, T, D, A, hidden = cfg.batch_size, cfg.unroll_len, cfg.obs_dim, cfg.n_actions, cfg.hidden
lrn = tlg.Learner("mlp", D, A, hidden, max_segments=S, unroll_len=T, obs_u8=True)
lrn.set_hyper(learning_rate=3e-4, batch_size=S, unroll_len=T)
lrn.set_params(tlg.synth.init_params_f32(lrn.n_params, 0.05, seed=1).astype(np.float64))
hs = [tlg.synth.make_segments(S, T, D, A, seed=i, obs_kind="binary", obs_u8=True) for i in range(2)]
views = []
for h in hs:
    hb = h.slice(0, S)
    hb.obs = tlg.synth.pack_bits(h.obs)
    v = tlg.SegmentBatchView(hb, bits=True, obs_dim=D)
    v.pinned = []
    for k, a in v.arrs.items():
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        v.pinned.append(t)
        v.arrs[k] = t.numpy()
    v.c = tlg._capi.SegmentBatchC(S, T, D, 2, *(v.arrs[k].ctypes.data for k in (
        "obs", "action", "reward", "behavior_logp", "value_est", "done", "bootstrap", "valid_steps")))
    views.append(v)
nbytes = sum(a.nbytes for a in views[0].arrs.values())
dst = {k: torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), device="cuda")
       for k, a in views[0].arrs.items()}
src = {k: torch.from_numpy(a) for k, a in views[0].arrs.items()}
for _ in range(3):
    for k in dst:
        dst[k].copy_(src[k], non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = 10
for _ in range(n):
    for k in dst:
        dst[k].copy_(src[k], non_blocking=True)
torch.cuda.synchronize()
h2d = (time.perf_counter() - t0) / n
print(f"H2D alone: {h2d * 1e3:.3f} ms/step  {nbytes / h2d / 1e9:.1f} GB/s  ({nbytes / 1e6:.1f} MB)")
dev = tlg.DeviceSegmentBatch(hs[0].slice(0, S), 0) if False else None
lrn.stage(views[0]); lrn.train_staged()
t0 = time.perf_counter()
lrn.stage(views[0])
for i in range(n):
    if i + 1 < n:
        lrn.stage(views[(i + 1) % 2])
    lrn.train_staged()
dt = (time.perf_counter() - t0) / n
print(f"staged pipeline: {dt * 1e3:.3f} ms/step  {S * T / dt / 1e6:.1f} M frames/s")
t0 = time.perf_counter()
for i in range(n):
    lrn.stage(views[i % 2])
    lrn.train_staged()
dt = (time.perf_counter() - t0) / n
print(f"staged, no overlap: {dt * 1e3:.3f} ms/step")
for i in range(n):
    lrn.train_step(views[i % 2])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    lrn.train_step(views[i % 2])
dt = (time.perf_counter() - t0) / n
print(f"train_step(host bits): {dt * 1e3:.3f} ms/step")

# device-resident steps alone, and with an unrelated H2D stream running concurrently
dv = [tlg.DeviceSegmentBatch(h.slice(0, S), 0, bits=False) for h in hs]
for i in range(3):
    lrn.train_step(dv[i % 2], on_device=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    lrn.train_step(dv[i % 2], on_device=True)
dt = (time.perf_counter() - t0) / n
print(f"device-resident u8 steps: {dt * 1e3:.3f} ms/step")
side = torch.cuda.Stream()
big_src = torch.empty(n * 40 << 20, dtype=torch.uint8, pin_memory=True)
big_dst = torch.empty_like(big_src, device="cuda")
torch.cuda.synchronize()
with torch.cuda.stream(side):
    big_dst.copy_(big_src, non_blocking=True)
t0 = time.perf_counter()
for i in range(n):
    lrn.train_step(dv[i % 2], on_device=True)
dt = (time.perf_counter() - t0) / n
torch.cuda.synchronize()
print(f"device-resident u8 steps with a concurrent H2D: {dt * 1e3:.3f} ms/step")
