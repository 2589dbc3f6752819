"""ctypes binding of libtlg_b200.so (include/tlg_b200.h) for the tests and bench.

This is plumbing, not the product: the hot path is the CUDA library itself and
its C++ host layer (paper_2011_12895_b200/host).  Status codes map onto the
reference's exception types: TLG_INVALID_ARGUMENT -> InvalidArgument
(std::invalid_argument), TLG_RUNTIME_ERROR -> LearnerRuntimeError
(std::runtime_error), TLG_CUDA_ERROR -> CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtlg_b200.so")

ALGOS = {"ppo": 0, "vtrace": 1, "ppo_vtrace": 2}
FAMILIES = {"tabular": 0, "linear": 1, "mlp": 2}


class InvalidArgument(ValueError):
    """std::invalid_argument at the reference boundary."""


class LearnerRuntimeError(RuntimeError):
    """std::runtime_error (e.g. non-finite loss at update step k)."""


class CudaError(RuntimeError):
    """Device / driver failure."""


class PolicyShape(C.Structure):
    _fields_ = [("family", C.c_uint32), ("obs_dim", C.c_uint32), ("n_actions", C.c_uint32),
                ("n_hidden", C.c_uint32), ("hidden", C.c_uint32 * 8)]

    @classmethod
    def make(cls, family, obs_dim, n_actions, hidden=()):
        s = cls()
        s.family = FAMILIES.get(family, family)
        s.obs_dim, s.n_actions, s.n_hidden = obs_dim, n_actions, len(hidden)
        for i, h in enumerate(hidden):
            s.hidden[i] = h
        return s


class Hyper(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("learning_rate", "gamma", "lam", "clip_eps", "vf_coef",
                                          "ent_coef", "kl_teacher_coef", "rho_bar", "c_bar")] + \
               [("batch_size", C.c_uint32), ("unroll_len", C.c_uint32), ("max_reuse", C.c_uint32),
                ("adv_norm", C.c_int32)]

    @classmethod
    def make(cls, **kw):
        """Defaults of tleague::HyperParams (types.hpp:36-51)."""
        d = dict(learning_rate=1e-2, gamma=0.99, lam=0.95, clip_eps=0.2, vf_coef=0.5,
                 ent_coef=0.01, kl_teacher_coef=0.0, rho_bar=1.0, c_bar=1.0, batch_size=32,
                 unroll_len=1, max_reuse=1, adv_norm=True)
        d.update(kw)
        h = cls()
        for k, v in d.items():
            setattr(h, k, int(v) if k == "adv_norm" else v)
        return h


class LearnerConfig(C.Structure):
    _fields_ = [("algo", C.c_uint32), ("optimizer", C.c_uint32), ("adam_beta1", C.c_double),
                ("adam_beta2", C.c_double), ("adam_eps", C.c_double),
                ("max_segments", C.c_uint32), ("unroll_len", C.c_uint32), ("device", C.c_int32),
                ("obs_dtype", C.c_uint32), ("timing", C.c_uint32)]


class SegmentBatchC(C.Structure):
    _fields_ = [("n_segments", C.c_uint32), ("unroll_len", C.c_uint32), ("obs_dim", C.c_uint32),
                ("obs_dtype", C.c_uint32), ("obs", C.c_void_p), ("action", C.c_void_p),
                ("reward", C.c_void_p), ("behavior_logp", C.c_void_p),
                ("value_est", C.c_void_p), ("done", C.c_void_p), ("bootstrap", C.c_void_p),
                ("valid_steps", C.c_void_p), ("obs_pitch", C.c_uint32)]


class StepStats(C.Structure):
    _fields_ = [("loss", C.c_double), ("clip_fraction", C.c_double), ("mean_ratio", C.c_double),
                ("entropy", C.c_double), ("value_loss", C.c_double), ("n_samples", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run __graft_entry__.build() "
                              "(make -C paper_2011_12895_b200/csrc); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.tlg_last_error.restype = C.c_char_p
        L.tlg_version.restype = C.c_char_p
        L.tlg_learner_create.argtypes = [C.POINTER(LearnerConfig), C.POINTER(PolicyShape),
                                         C.POINTER(C.c_void_p)]
        L.tlg_learner_destroy.argtypes = [C.c_void_p]
        L.tlg_learner_param_count.restype = C.c_size_t
        L.tlg_learner_param_count.argtypes = [C.c_void_p]
        for fn in ("tlg_learner_set_params", "tlg_learner_get_params", "tlg_learner_get_grad",
                   "tlg_learner_set_teacher"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        L.tlg_learner_set_hyper.argtypes = [C.c_void_p, C.POINTER(Hyper)]
        L.tlg_replay_create.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]
        L.tlg_replay_destroy.argtypes = [C.c_void_p]
        L.tlg_replay_put.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(SegmentBatchC)]
        L.tlg_learner_train_step_replay.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p,
                                                    C.c_uint32, C.c_uint32, C.c_void_p]
        L.tlg_comm_unique_id.argtypes = [C.c_void_p]
        L.tlg_learner_comm_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.tlg_learner_comm_init_all.argtypes = [C.c_void_p, C.c_int]
        L.tlg_learner_train_step.argtypes = [C.c_void_p, C.POINTER(SegmentBatchC), C.c_int,
                                             C.POINTER(StepStats)]
        L.tlg_learner_train_step_shards.argtypes = [C.c_void_p, C.POINTER(SegmentBatchC), C.c_int,
                                                    C.c_int, C.POINTER(StepStats)]
        L.tlg_learner_stage.argtypes = [C.c_void_p, C.POINTER(SegmentBatchC)]
        L.tlg_learner_train_staged.argtypes = [C.c_void_p, C.POINTER(StepStats)]
        L.tlg_learner_train_staged_next.argtypes = [C.c_void_p, C.POINTER(SegmentBatchC),
                                                    C.POINTER(StepStats)]
        L.tlg_learner_get_returns.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
        L.tlg_learner_stream.restype = C.c_void_p
        L.tlg_learner_stream.argtypes = [C.c_void_p]
        L.tlg_learner_phase_ms.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.tlg_learner_last_launches.argtypes = [C.c_void_p]
        L.tlg_learner_set_timing.argtypes = [C.c_void_p, C.c_int]
        L.tlg_learner_kernel_ms.argtypes = [C.c_void_p, C.c_int, C.c_int,
                                            C.POINTER(C.c_float)]
        L.tlg_policy_create.argtypes = [C.POINTER(PolicyShape), C.c_int32, C.c_uint32,
                                        C.POINTER(C.c_void_p)]
        L.tlg_policy_destroy.argtypes = [C.c_void_p]
        L.tlg_policy_set_params.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        L.tlg_policy_set_params_from_learner.argtypes = [C.c_void_p, C.c_void_p]
        L.tlg_policy_forward_async.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
        L.tlg_policy_wait.argtypes = [C.c_void_p, C.c_uint64]
        L.tlg_policy_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_int]
        L.tlg_policy_stream.restype = C.c_void_p
        L.tlg_policy_stream.argtypes = [C.c_void_p]
        L.tlg_returns.argtypes = [C.c_uint32, C.POINTER(Hyper), C.c_uint32, C.c_uint32] + \
            [C.c_void_p] * 9 + [C.c_void_p]
        _lib = L
    return _lib


def check(rc):
    if rc == 0:
        return
    msg = lib().tlg_last_error().decode()
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 2:
        raise LearnerRuntimeError(msg)
    raise CudaError(msg)


EXPORTS = [
    "tlg_last_error", "tlg_version", "tlg_device_count", "tlg_host_alloc", "tlg_host_free", "tlg_learner_create", "tlg_learner_destroy",
    "tlg_learner_param_count", "tlg_learner_set_params", "tlg_learner_get_params",
    "tlg_learner_set_teacher", "tlg_replay_create", "tlg_replay_destroy", "tlg_replay_put",
    "tlg_learner_train_step_replay",
    "tlg_learner_set_hyper", "tlg_comm_unique_id", "tlg_learner_comm_init",
    "tlg_learner_comm_init_all",
    "tlg_learner_train_step", "tlg_learner_train_step_shards", "tlg_learner_get_grad",
    "tlg_learner_stage", "tlg_learner_train_staged", "tlg_learner_train_staged_next",
    "tlg_learner_get_returns",
    "tlg_learner_stream", "tlg_learner_phase_ms", "tlg_learner_last_launches",
    "tlg_learner_kernel_ms", "tlg_learner_set_timing",
    "tlg_policy_create", "tlg_policy_destroy", "tlg_policy_set_params", "tlg_policy_forward",
    "tlg_policy_forward_async", "tlg_policy_wait",
    "tlg_policy_set_params_from_learner",
    "tlg_policy_stream", "tlg_returns",
]


def _ptr(a):
    return None if a is None else a.ctypes.data


class SegmentBatchView:
    """Keeps host arrays alive and exposes the C struct (host pointers).  `bits=True`:
    b.obs holds 0/1 planes bit-packed LSB-first (synth.pack_bits), obs_dim given."""

    def __init__(self, b, bits=False, obs_dim=None):
        self.arrs = dict(
            obs=np.ascontiguousarray(b.obs),
            action=np.ascontiguousarray(b.action, np.int32),
            reward=np.ascontiguousarray(b.reward, np.float32),
            behavior_logp=np.ascontiguousarray(b.behavior_logp, np.float32),
            value_est=np.ascontiguousarray(b.value_est, np.float32),
            done=np.ascontiguousarray(b.done, np.uint8),
            bootstrap=np.ascontiguousarray(b.bootstrap, np.float32),
            valid_steps=np.ascontiguousarray(b.valid_steps, np.int32))
        o = self.arrs["obs"]
        if o.dtype not in (np.float32, np.uint8):
            self.arrs["obs"] = o = o.astype(np.float32)
        S, T = self.arrs["action"].shape
        self.c = SegmentBatchC(S, T, obs_dim if bits else o.shape[2],
                               2 if bits else (1 if o.dtype == np.uint8 else 0),
                               *(self.arrs[k].ctypes.data for k in (
                                   "obs", "action", "reward", "behavior_logp", "value_est",
                                   "done", "bootstrap", "valid_steps")))


class DeviceSegmentBatch:
    """The same batch resident in HBM (torch tensors as device allocations)."""

    def __init__(self, b, device=0, bits=False, obs_dim=None, pitch=0):
        """bits=True: b.obs holds bit-packed rows; pitch > 0 pads each frame row to `pitch`
        bytes (a multiple of 16 feeds the int8 GEMM without re-pitching)."""
        import torch
        dev = torch.device("cuda", device)
        v = SegmentBatchView(b, bits=bits, obs_dim=obs_dim)
        if bits and pitch:
            o = v.arrs["obs"]
            padded = np.zeros(o.shape[:-1] + (pitch,), np.uint8)
            padded[..., :o.shape[-1]] = o
            v.arrs["obs"] = padded
        self.t = {k: torch.from_numpy(a).to(dev) for k, a in v.arrs.items()}
        o = self.t["obs"]
        S, T = self.t["action"].shape
        self.c = SegmentBatchC(S, T, obs_dim if bits else o.shape[2],
                               2 if bits else (1 if o.dtype == torch.uint8 else 0),
                               *(self.t[k].data_ptr() for k in (
                                   "obs", "action", "reward", "behavior_logp", "value_est",
                                   "done", "bootstrap", "valid_steps")), pitch if bits else 0)


class Learner:
    """One GPU shard of learner::Learner::TrainStep (learner.cpp:104-158)."""

    def __init__(self, family, obs_dim, n_actions, hidden=(), *, algo="ppo", optimizer="adam",
                 max_segments, unroll_len, device=0, obs_u8=False, timing=False,
                 adam=(0.9, 0.999, 1e-8)):
        L = lib()
        self.shape = PolicyShape.make(family, obs_dim, n_actions, hidden)
        cfg = LearnerConfig(ALGOS[algo], 1 if optimizer == "adam" else 0, adam[0], adam[1],
                            adam[2], max_segments, unroll_len, device, 1 if obs_u8 else 0,
                            1 if timing else 0)
        h = C.c_void_p()
        check(L.tlg_learner_create(C.byref(cfg), C.byref(self.shape), C.byref(h)))
        self.h = h
        self.n_params = L.tlg_learner_param_count(h)

    def close(self):
        if getattr(self, "h", None):
            lib().tlg_learner_destroy(self.h)
            self.h = None

    __del__ = close

    def set_params(self, values):
        v = np.ascontiguousarray(values, np.float64)
        check(lib().tlg_learner_set_params(self.h, v.ctypes.data, v.size))

    def get_params(self):
        out = np.zeros(self.n_params)
        check(lib().tlg_learner_get_params(self.h, out.ctypes.data, out.size))
        return out

    def set_teacher(self, values):
        """Teacher policy for the PPO KL term (None clears it)."""
        if values is None:
            check(lib().tlg_learner_set_teacher(self.h, None, 0))
            return
        v = np.ascontiguousarray(values, np.float64)
        check(lib().tlg_learner_set_teacher(self.h, v.ctypes.data, v.size))

    def get_grad(self):
        out = np.zeros(self.n_params)
        check(lib().tlg_learner_get_grad(self.h, out.ctypes.data, out.size))
        return out

    def set_hyper(self, **kw):
        self.hyper = Hyper.make(**kw)
        check(lib().tlg_learner_set_hyper(self.h, C.byref(self.hyper)))

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        check(lib().tlg_learner_comm_init(self.h, buf, nranks, rank))

    def train_step(self, batch, on_device=False):
        st = StepStats()
        view = batch if isinstance(batch, (SegmentBatchView, DeviceSegmentBatch)) else \
            SegmentBatchView(batch)
        check(lib().tlg_learner_train_step(self.h, C.byref(view.c), 1 if on_device else 0,
                                           C.byref(st)))
        return st.as_dict()

    def train_step_shards(self, batches, on_device=False):
        """Several in-process shards on this GPU (learner.cpp:117-149)."""
        views = [b if isinstance(b, (SegmentBatchView, DeviceSegmentBatch)) else
                 SegmentBatchView(b) for b in batches]
        arr = (SegmentBatchC * len(views))(*[v.c for v in views])
        sts = (StepStats * len(views))()
        check(lib().tlg_learner_train_step_shards(self.h, arr, len(views), 1 if on_device else 0,
                                                  sts))
        return [s.as_dict() for s in sts]

    def stage(self, batch_view):
        """Queue the async H2D of a host batch (keep `batch_view` alive until trained)."""
        check(lib().tlg_learner_stage(self.h, C.byref(batch_view.c)))

    def train_staged(self, next_view=None):
        """Train the oldest staged batch; `next_view` (kept alive by the caller) is staged
        while that step runs."""
        st = StepStats()
        if next_view is None:
            check(lib().tlg_learner_train_staged(self.h, C.byref(st)))
        else:
            check(lib().tlg_learner_train_staged_next(self.h, C.byref(next_view.c), C.byref(st)))
        return st.as_dict()

    def get_returns(self, n_frames):
        adv = np.zeros(n_frames, np.float32)
        tgt = np.zeros(n_frames, np.float32)
        check(lib().tlg_learner_get_returns(self.h, adv.ctypes.data, tgt.ctypes.data, n_frames))
        return adv, tgt

    def stream(self):
        return lib().tlg_learner_stream(self.h)

    def phase_ms(self):
        out = np.zeros(7, np.float32)
        check(lib().tlg_learner_phase_ms(self.h, out.ctypes.data, 7))
        return out

    def last_launches(self):
        return lib().tlg_learner_last_launches(self.h)

    def set_timing(self, on: bool):
        check(lib().tlg_learner_set_timing(self.h, 1 if on else 0))

    def kernel_ms(self, kind, layer):
        """kind: 'fwd' | 'dw' | 'dx' (0-based layer)."""
        ms = C.c_float()
        check(lib().tlg_learner_kernel_ms(self.h, {"fwd": 0, "dw": 1, "dx": 2}[kind], layer,
                                          C.byref(ms)))
        return ms.value


class Replay:
    """Device-resident replay ring of `capacity` segment slots (tlg_replay_*)."""

    def __init__(self, learner, capacity, bits=False):
        h = C.c_void_p()
        check(lib().tlg_replay_create(learner.h, capacity, 2 if bits else 0, C.byref(h)))
        self.h = h
        self.learner = learner  # keeps the learner alive

    def close(self):
        if getattr(self, "h", None):
            lib().tlg_replay_destroy(self.h)
            self.h = None

    __del__ = close

    def put(self, slots, batch):
        """Copy the batch's segments (a SegmentBatchView or SegmentBatch) into `slots`."""
        view = batch if isinstance(batch, SegmentBatchView) else SegmentBatchView(batch)
        sl = np.ascontiguousarray(slots, np.uint32)
        check(lib().tlg_replay_put(self.h, sl.ctypes.data, C.byref(view.c)))

    def train_step(self, slots, n_shards=1):
        """One learner step over n_shards shards of len(slots) // n_shards slots each;
        returns the per-shard statistics."""
        sl = np.ascontiguousarray(slots, np.uint32)
        sts = (StepStats * n_shards)()
        check(lib().tlg_learner_train_step_replay(self.learner.h, self.h, sl.ctypes.data,
                                                  n_shards, sl.size // n_shards, sts))
        return [s.as_dict() for s in sts]


def comm_init_all(learners):
    """One ncclCommInitAll over learners on distinct devices (learners[i] = rank i)."""
    arr = (C.c_void_p * len(learners))(*[l.h.value for l in learners])
    check(lib().tlg_learner_comm_init_all(arr, len(learners)))


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().tlg_comm_unique_id(buf))
    return bytes(buf)


class Policy:
    """InfServer batched forward (inf_server.cpp:125-144) on one GPU."""

    def __init__(self, family, obs_dim, n_actions, hidden=(), *, device=0, max_batch=65536):
        self.shape = PolicyShape.make(family, obs_dim, n_actions, hidden)
        h = C.c_void_p()
        check(lib().tlg_policy_create(C.byref(self.shape), device, max_batch, C.byref(h)))
        self.h = h
        self.A = n_actions

    def close(self):
        if getattr(self, "h", None):
            lib().tlg_policy_destroy(self.h)
            self.h = None

    __del__ = close

    def set_params(self, values):
        v = np.ascontiguousarray(values, np.float64)
        check(lib().tlg_policy_set_params(self.h, v.ctypes.data, v.size))

    def refresh_from(self, learner):
        """Device-to-device refresh from a co-located Learner (no fp64 host round trip)."""
        check(lib().tlg_policy_set_params_from_learner(self.h, learner.h))

    def forward(self, obs, out=None):
        """Host batch in, host results out.  `out` = (logits, probs, value) arrays to fill
        (e.g. views of pinned buffers); new arrays otherwise."""
        obs = np.ascontiguousarray(obs, np.float32)
        n = obs.shape[0]
        if out is None:
            lg = np.zeros((n, self.A), np.float32)
            pr = np.zeros((n, self.A), np.float32)
            v = np.zeros(n, np.float32)
        else:
            lg, pr, v = out
        check(lib().tlg_policy_forward(self.h, obs.ctypes.data, n, lg.ctypes.data, pr.ctypes.data,
                                       v.ctypes.data, 0))
        return lg, pr, v

    def forward_async(self, obs, out):
        """Enqueue a host batch (obs and the (logits, probs, value) arrays must stay alive,
        page-locked for overlap, until wait(ticket)); returns the ticket."""
        t = C.c_uint64()
        lg, pr, v = out
        check(lib().tlg_policy_forward_async(self.h, obs.ctypes.data, obs.shape[0],
                                             lg.ctypes.data, pr.ctypes.data, v.ctypes.data,
                                             C.byref(t)))
        return t.value

    def wait(self, ticket):
        check(lib().tlg_policy_wait(self.h, ticket))

    def forward_device(self, obs_t, logits_t, probs_t, value_t):
        check(lib().tlg_policy_forward(self.h, obs_t.data_ptr(), obs_t.shape[0],
                                       logits_t.data_ptr(), probs_t.data_ptr(),
                                       value_t.data_ptr(), 1))

    def stream(self):
        return lib().tlg_policy_stream(self.h)
