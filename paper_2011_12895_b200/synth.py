"""Synthetic rollout segments of a named shape.

Mirrors the reference's synthetic generators (learner_test.cpp:43-60,
acceptance.cpp:545-562) at the BASELINE shapes.  Every value is exactly
representable in fp32, so the fp64 oracle and the fp32 GPU path consume
bit-identical operands:

* obs ~ N(0,1) rounded to fp32, or Bernoulli(0.1) {0,1} planes ("binary", C3)
* action ~ U{0..A-1}; reward, value_est, bootstrap ~ U(-1,1)
* behavior_logp = log(1/A) + 0.1*U(-1,1) (V-trace rho straddles rho_bar = 1)
* done ~ Bernoulli(0.01); 1/16 of segments ragged with valid_steps ~ U{1..T};
  padding steps are all-zero with done = false (segmenter.cpp:26-31).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SegmentBatch:
    """SoA [S][T] segment batch as the C-ABI consumes it (include/tlg_b200.h)."""
    obs: np.ndarray            # [S, T, D] float32, or uint8 when obs_u8
    action: np.ndarray         # [S, T] int32
    reward: np.ndarray         # [S, T] float32
    behavior_logp: np.ndarray  # [S, T] float32
    value_est: np.ndarray      # [S, T] float32
    done: np.ndarray           # [S, T] uint8
    bootstrap: np.ndarray      # [S] float32
    valid_steps: np.ndarray    # [S] int32

    @property
    def n_segments(self):
        return self.action.shape[0]

    @property
    def unroll_len(self):
        return self.action.shape[1]

    @property
    def obs_dim(self):
        return self.obs.shape[2]

    @property
    def obs_u8(self):
        return self.obs.dtype == np.uint8

    def frames(self):
        return int(self.valid_steps.sum())

    def slice(self, lo, hi):
        return SegmentBatch(*(np.ascontiguousarray(getattr(self, k)[lo:hi]) for k in (
            "obs", "action", "reward", "behavior_logp", "value_est", "done", "bootstrap",
            "valid_steps")))

    def nbytes(self):
        return sum(getattr(self, k).nbytes for k in (
            "obs", "action", "reward", "behavior_logp", "value_est", "done", "bootstrap",
            "valid_steps"))

    def to_f64(self):
        """fp64 views for the oracle (exact widening)."""
        from types import SimpleNamespace
        return SimpleNamespace(
            obs=self.obs.astype(np.float64), action=self.action.astype(np.uint32),
            reward=self.reward.astype(np.float64),
            behavior_logp=self.behavior_logp.astype(np.float64),
            value_est=self.value_est.astype(np.float64), done=self.done.astype(np.uint8),
            bootstrap=self.bootstrap.astype(np.float64),
            valid_steps=self.valid_steps.astype(np.uint32))


def make_segments(n_segments: int, unroll_len: int, obs_dim: int, n_actions: int, *,
                  seed: int, obs_kind: str = "gauss", obs_u8: bool = False,
                  done_p: float = 0.01, ragged_frac: float = 1.0 / 16) -> SegmentBatch:
    rng = np.random.default_rng(seed)
    S, T, D = n_segments, unroll_len, obs_dim
    if obs_kind == "binary":
        planes = rng.random((S, T, D), dtype=np.float32) < 0.1
        obs = planes.astype(np.uint8) if obs_u8 else planes.astype(np.float32)
    else:
        if obs_u8:
            raise ValueError("uint8 observations require obs_kind='binary'")
        obs = rng.standard_normal((S, T, D), dtype=np.float32)
    action = rng.integers(0, n_actions, size=(S, T), dtype=np.int32)
    reward = rng.uniform(-1, 1, size=(S, T)).astype(np.float32)
    value = rng.uniform(-1, 1, size=(S, T)).astype(np.float32)
    blogp = (np.log(1.0 / n_actions) + 0.1 * rng.uniform(-1, 1, size=(S, T))).astype(np.float32)
    done = (rng.random((S, T)) < done_p).astype(np.uint8)
    boot = rng.uniform(-1, 1, size=S).astype(np.float32)
    valid = np.full(S, T, dtype=np.int32)
    ragged = rng.random(S) < ragged_frac
    valid[ragged] = rng.integers(1, T + 1, size=int(ragged.sum()), dtype=np.int32)
    # padding steps are all-zero with done=false (segmenter.cpp:26-31)
    pad = np.arange(T)[None, :] >= valid[:, None]
    for a in (reward, value, blogp):
        a[pad] = 0
    action[pad] = 0
    done[pad] = 0
    obs[pad] = 0
    # a segment whose episode ended bootstraps with 0 (segmenter.cpp:21-25)
    last_done = done[np.arange(S), valid - 1] != 0
    boot[last_done] = 0.0
    return SegmentBatch(obs, action, reward, blogp, value, done, boot, valid)


def make_obs(n: int, obs_dim: int, *, seed: int, obs_kind: str = "gauss") -> np.ndarray:
    rng = np.random.default_rng(seed)
    if obs_kind == "binary":
        return (rng.random((n, obs_dim), dtype=np.float32) < 0.1).astype(np.float32)
    return rng.standard_normal((n, obs_dim), dtype=np.float32)


def init_params_f32(n_params: int, scale: float, seed: int) -> np.ndarray:
    """U[-s,s] fp32-representable parameters (for MLP parity runs; the reference's
    mt19937_64 InitParams (policy.cpp:29-43) is reproduced bit-exactly by the C++
    host layer for the tabular/linear families)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-scale, scale, size=n_params).astype(np.float32)


def pack_bits(obs_u8: np.ndarray) -> np.ndarray:
    """0/1 planes [..., D] -> LSB-first packed bytes [..., ceil(D/8)] (TLG_OBS_BITS)."""
    return np.ascontiguousarray(np.packbits(obs_u8.astype(np.uint8), axis=-1, bitorder="little"))
