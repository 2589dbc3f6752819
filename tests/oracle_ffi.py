"""ctypes bindings for the CHECKERS under oracle/ (test infrastructure only).

* ``Oracle``  -- oracle/lib/libtlg_oracle.so, the fp64 restatement (tlg_oracle.h).
* ``RefLib``  -- oracle/_ref/libtleague_ref_capi.so, the UNMODIFIED reference
  library compiled from /root/reference/proj/src plus an extern "C" shim
  (oracle/ref_capi.cpp).  Absent on a checkout that never saw /root/reference;
  tests that need it skip, and tests/golden/ carries its outputs instead.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline arm import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_LIB = os.path.join(ROOT, "oracle", "lib", "libtlg_oracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libtleague_ref_capi.so")

f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


class OracleError(Exception):
    pass


class InvalidArgument(OracleError, ValueError):
    """Maps std::invalid_argument."""


class RuntimeErr(OracleError, RuntimeError):
    """Maps std::runtime_error."""


def _raise(rc: int, msg: bytes):
    if rc == 0:
        return
    text = msg.decode() if msg else ""
    raise (InvalidArgument if rc == 1 else RuntimeErr)(text)


# ---------------------------------------------------------------------------
# Shared value types
@dataclass
class Shape:
    family: int            # 0 tabular, 1 linear, 2 mlp
    obs_dim: int
    n_actions: int
    hidden: tuple = ()

    def c(self):
        s = OrcShape()
        s.family = self.family
        s.obs_dim = self.obs_dim
        s.n_actions = self.n_actions
        s.n_hidden = len(self.hidden)
        for i, h in enumerate(self.hidden):
            s.hidden[i] = h
        return s


@dataclass
class Hyper:
    """Defaults of tleague::HyperParams (types.hpp:36-51)."""
    learning_rate: float = 1e-2
    gamma: float = 0.99
    lam: float = 0.95
    clip_eps: float = 0.2
    vf_coef: float = 0.5
    ent_coef: float = 0.01
    kl_teacher_coef: float = 0.0
    rho_bar: float = 1.0
    c_bar: float = 1.0
    batch_size: int = 32
    unroll_len: int = 1
    max_reuse: int = 1
    adv_norm: bool = True

    def c(self, cls):
        h = cls()
        for k in ("learning_rate", "gamma", "lam", "clip_eps", "vf_coef", "ent_coef",
                  "kl_teacher_coef", "rho_bar", "c_bar", "batch_size", "unroll_len",
                  "max_reuse"):
            setattr(h, k, getattr(self, k))
        h.adv_norm = 1 if self.adv_norm else 0
        return h


class OrcShape(C.Structure):
    _fields_ = [("family", C.c_uint32), ("obs_dim", C.c_uint32), ("n_actions", C.c_uint32),
                ("n_hidden", C.c_uint32), ("hidden", C.c_uint32 * 8)]


class OrcHyper(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("learning_rate", "gamma", "lam", "clip_eps",
                                          "vf_coef", "ent_coef", "kl_teacher_coef",
                                          "rho_bar", "c_bar")] + \
               [("batch_size", C.c_uint32), ("unroll_len", C.c_uint32),
                ("max_reuse", C.c_uint32), ("adv_norm", C.c_int32)]


RefHyper = OrcHyper  # identical field order (ref_capi.cpp ref_hyper)


class OrcSegments(C.Structure):
    _fields_ = [("n_segments", C.c_uint32), ("unroll_len", C.c_uint32),
                ("obs_dim", C.c_uint32),
                ("obs", C.c_void_p), ("action", C.c_void_p), ("reward", C.c_void_p),
                ("behavior_logp", C.c_void_p), ("value_est", C.c_void_p),
                ("done", C.c_void_p), ("bootstrap", C.c_void_p),
                ("valid_steps", C.c_void_p)]


class RefSegments(C.Structure):
    _fields_ = OrcSegments._fields_ + [("segment_seq", C.c_void_p)]


class OrcStats(C.Structure):
    _fields_ = [("loss", C.c_double), ("clip_fraction", C.c_double),
                ("mean_ratio", C.c_double), ("entropy", C.c_double),
                ("value_loss", C.c_double), ("n_samples", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


@dataclass
class Segments:
    """SoA segments, [S][T] frame-major, fp64 host copy (fp32-representable values)."""
    obs: np.ndarray            # [S, T, D] f64
    action: np.ndarray         # [S, T] u32
    reward: np.ndarray         # [S, T] f64
    behavior_logp: np.ndarray  # [S, T] f64
    value_est: np.ndarray      # [S, T] f64
    done: np.ndarray           # [S, T] u8
    bootstrap: np.ndarray      # [S] f64
    valid_steps: np.ndarray    # [S] u32
    segment_seq: np.ndarray = None
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n_segments(self):
        return self.action.shape[0]

    @property
    def unroll_len(self):
        return self.action.shape[1]

    @property
    def obs_dim(self):
        return self.obs.shape[2]

    def slice(self, lo, hi):
        return Segments(*(np.ascontiguousarray(getattr(self, k)[lo:hi]) for k in (
            "obs", "action", "reward", "behavior_logp", "value_est", "done", "bootstrap",
            "valid_steps")), segment_seq=None if self.segment_seq is None
            else np.ascontiguousarray(self.segment_seq[lo:hi]))

    def _fill(self, s):
        arrs = {
            "obs": np.ascontiguousarray(self.obs, np.float64),
            "action": np.ascontiguousarray(self.action, np.uint32),
            "reward": np.ascontiguousarray(self.reward, np.float64),
            "behavior_logp": np.ascontiguousarray(self.behavior_logp, np.float64),
            "value_est": np.ascontiguousarray(self.value_est, np.float64),
            "done": np.ascontiguousarray(self.done, np.uint8),
            "bootstrap": np.ascontiguousarray(self.bootstrap, np.float64),
            "valid_steps": np.ascontiguousarray(self.valid_steps, np.uint32),
        }
        s.n_segments, s.unroll_len, s.obs_dim = self.n_segments, self.unroll_len, self.obs_dim
        for k, a in arrs.items():
            setattr(s, k, a.ctypes.data)
        self._keep = list(arrs.values())
        return s

    def c_orc(self):
        return self._fill(OrcSegments())

    def c_ref(self):
        s = self._fill(RefSegments())
        if self.segment_seq is not None:
            seq = np.ascontiguousarray(self.segment_seq, np.uint64)
            self._keep.append(seq)
            s.segment_seq = seq.ctypes.data
        else:
            s.segment_seq = None
        return s


# ---------------------------------------------------------------------------
class Oracle:
    """The fp64 restatement (oracle/tlg_oracle.cpp)."""

    def __init__(self, path: str = ORACLE_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle lib)")
        L = self.L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_param_count.restype = C.c_size_t
        L.orc_param_count.argtypes = [C.POINTER(OrcShape)]
        L.orc_init_params.argtypes = [C.POINTER(OrcShape), C.c_double, C.c_uint64, f64p]
        L.orc_forward.argtypes = [C.POINTER(OrcShape), f64p, f64p, C.c_size_t, f64p, f64p, f64p]
        for fn in ("orc_gae", "orc_lambda_return"):
            getattr(L, fn).argtypes = [f64p, f64p, u8p, C.c_size_t, C.c_double, C.c_double,
                                       C.c_double, f64p]
        L.orc_vtrace.argtypes = [f64p, f64p, f64p, f64p, u8p, C.c_size_t, C.c_double,
                                 C.c_double, C.c_double, C.c_double, f64p, f64p]
        L.orc_ppo_loss_grad.argtypes = [C.POINTER(OrcShape), f64p, C.c_void_p, C.c_size_t, f64p,
                                        u32p, f64p, f64p, f64p, C.POINTER(OrcHyper), f64p,
                                        C.POINTER(OrcStats)]
        L.orc_pg_loss_grad.argtypes = [C.POINTER(OrcShape), f64p, C.c_size_t, f64p, u32p, f64p,
                                       f64p, f64p, C.POINTER(OrcHyper), f64p,
                                       C.POINTER(OrcStats)]
        L.orc_shard_loss_grad.argtypes = [C.POINTER(OrcShape), f64p, C.POINTER(OrcHyper),
                                          C.c_uint32, C.POINTER(OrcSegments), f64p,
                                          C.POINTER(OrcStats)]
        L.orc_shard_returns.argtypes = [C.POINTER(OrcShape), f64p, C.POINTER(OrcHyper),
                                        C.c_uint32, C.POINTER(OrcSegments), f64p, f64p]
        L.orc_sgd_step.argtypes = [f64p, f64p, C.c_size_t, C.c_double, f64p]
        L.orc_adam_step.argtypes = [f64p, f64p, f64p, f64p, C.c_size_t, C.c_uint64, C.c_double,
                                    C.c_double, C.c_double, C.c_double]

    def _chk(self, rc):
        _raise(rc, self.L.orc_last_error())

    def param_count(self, shape: Shape) -> int:
        n = self.L.orc_param_count(C.byref(shape.c()))
        if n == 0:
            raise InvalidArgument(self.L.orc_last_error().decode())
        return n

    def init_params(self, shape: Shape, scale: float, seed: int) -> np.ndarray:
        out = np.zeros(self.param_count(shape))
        self._chk(self.L.orc_init_params(C.byref(shape.c()), scale, seed, out))
        return out

    def forward(self, shape: Shape, params, obs):
        obs = np.ascontiguousarray(obs, np.float64).reshape(-1, shape.obs_dim)
        n = obs.shape[0]
        lg = np.zeros((n, shape.n_actions)); pr = np.zeros_like(lg); v = np.zeros(n)
        self._chk(self.L.orc_forward(C.byref(shape.c()), np.ascontiguousarray(params, np.float64),
                                     obs, n, lg, pr, v))
        return lg, pr, v

    def gae(self, r, v, done, boot, gamma, lam):
        out = np.zeros(len(r))
        self._chk(self.L.orc_gae(np.ascontiguousarray(r, np.float64),
                                 np.ascontiguousarray(v, np.float64),
                                 np.ascontiguousarray(done, np.uint8), len(r), boot, gamma,
                                 lam, out))
        return out

    def lambda_return(self, r, v, done, boot, gamma, lam):
        out = np.zeros(len(r))
        self._chk(self.L.orc_lambda_return(np.ascontiguousarray(r, np.float64),
                                           np.ascontiguousarray(v, np.float64),
                                           np.ascontiguousarray(done, np.uint8), len(r), boot,
                                           gamma, lam, out))
        return out

    def vtrace(self, bl, tl, r, v, done, boot, gamma, rho_bar, c_bar):
        vs = np.zeros(len(r)); pg = np.zeros(len(r))
        self._chk(self.L.orc_vtrace(*(np.ascontiguousarray(x, np.float64) for x in (bl, tl, r, v)),
                                    np.ascontiguousarray(done, np.uint8), len(r), boot, gamma,
                                    rho_bar, c_bar, vs, pg))
        return vs, pg

    def _loss(self, fn, shape, params, teacher, obs, action, blogp, adv, vtarget, hyper):
        n = len(action)
        grad = np.zeros(self.param_count(shape))
        st = OrcStats()
        args = [C.byref(shape.c()), np.ascontiguousarray(params, np.float64)]
        if fn == "ppo":
            t = None if teacher is None else np.ascontiguousarray(teacher, np.float64)
            args.append(None if t is None else t.ctypes.data)
        args += [n, np.ascontiguousarray(obs, np.float64).reshape(-1),
                 np.ascontiguousarray(action, np.uint32),
                 *(np.ascontiguousarray(x, np.float64) for x in (blogp, adv, vtarget)),
                 C.byref(hyper.c(OrcHyper)), grad, C.byref(st)]
        self._chk(getattr(self.L, f"orc_{fn}_loss_grad")(*args))
        return st.as_dict(), grad

    def ppo_loss_grad(self, shape, params, obs, action, blogp, adv, vtarget, hyper, teacher=None):
        return self._loss("ppo", shape, params, teacher, obs, action, blogp, adv, vtarget, hyper)

    def pg_loss_grad(self, shape, params, obs, action, blogp, adv, vtarget, hyper):
        return self._loss("pg", shape, params, None, obs, action, blogp, adv, vtarget, hyper)

    def shard_loss_grad(self, shape, params, hyper, algo, segs: Segments):
        grad = np.zeros(self.param_count(shape))
        st = OrcStats()
        cs = segs.c_orc()
        self._chk(self.L.orc_shard_loss_grad(C.byref(shape.c()),
                                             np.ascontiguousarray(params, np.float64),
                                             C.byref(hyper.c(OrcHyper)), algo, C.byref(cs), grad,
                                             C.byref(st)))
        return st.as_dict(), grad

    def shard_returns(self, shape, params, hyper, algo, segs: Segments):
        F = segs.n_segments * segs.unroll_len
        adv = np.zeros(F); tgt = np.zeros(F)
        cs = segs.c_orc()
        self._chk(self.L.orc_shard_returns(C.byref(shape.c()),
                                           np.ascontiguousarray(params, np.float64),
                                           C.byref(hyper.c(OrcHyper)), algo, C.byref(cs), adv,
                                           tgt))
        return adv.reshape(segs.n_segments, -1), tgt.reshape(segs.n_segments, -1)

    def sgd_step(self, params, grad, lr):
        out = np.zeros(len(params))
        self._chk(self.L.orc_sgd_step(np.ascontiguousarray(params, np.float64),
                                      np.ascontiguousarray(grad, np.float64), len(params), lr,
                                      out))
        return out

    def adam_step(self, params, grad, m, v, step, lr, b1=0.9, b2=0.999, eps=1e-8):
        p = np.array(params, np.float64); m = np.array(m, np.float64); v = np.array(v, np.float64)
        self._chk(self.L.orc_adam_step(p, np.ascontiguousarray(grad, np.float64), m, v, len(p),
                                       step, lr, b1, b2, eps))
        return p, m, v

    def learner_step(self, shape, params, hyper, algo, shards, optimizer="sgd", adam=None,
                     step=1):
        """Rank-ordered shard average + optimizer (learner.cpp:138-152)."""
        avg = np.zeros(len(params))
        stats = []
        for k, seg in enumerate(shards):
            st, g = self.shard_loss_grad(shape, params, hyper, algo, seg)
            if not np.isfinite(st["loss"]):
                raise RuntimeErr(f"non-finite loss at update step {step}")
            avg += g
            stats.append(st)
        avg *= 1.0 / len(shards)
        if optimizer == "sgd":
            return self.sgd_step(params, avg, hyper.learning_rate), avg, stats, adam
        m, v, lr, b1, b2, eps = adam
        p, m, v = self.adam_step(params, avg, m, v, step, lr, b1, b2, eps)
        return p, avg, stats, (m, v, lr, b1, b2, eps)


class RefLib:
    """The reference library itself (oracle/_ref)."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        for fn in ("ref_gae", "ref_lambda_return"):
            getattr(L, fn).argtypes = [f64p, f64p, u8p, C.c_size_t, C.c_double, C.c_double,
                                       C.c_double, f64p]
        L.ref_vtrace.argtypes = [f64p, f64p, f64p, f64p, u8p, C.c_size_t, C.c_double,
                                 C.c_double, C.c_double, C.c_double, f64p, f64p]
        L.ref_param_count.restype = C.c_size_t
        L.ref_param_count.argtypes = [C.c_uint32] * 3
        L.ref_init_params.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                      f64p]
        L.ref_batch_forward.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, f64p, f64p,
                                        C.c_size_t, f64p, f64p, f64p]
        L.ref_ppo_loss_grad.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, f64p, C.c_void_p,
                                        C.c_size_t, f64p, u32p, f64p, f64p, f64p,
                                        C.POINTER(RefHyper), f64p, f64p, f64p]
        L.ref_pg_loss_grad.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, f64p, C.c_size_t,
                                       f64p, u32p, f64p, f64p, f64p, C.POINTER(RefHyper), f64p,
                                       f64p, f64p]
        L.ref_sgd_step.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, f64p, f64p, C.c_double,
                                   f64p]
        L.ref_replay_create.restype = C.c_void_p
        L.ref_replay_create.argtypes = [C.c_size_t, C.c_uint32, C.c_uint64]
        L.ref_replay_destroy.argtypes = [C.c_void_p]
        L.ref_replay_push.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
        L.ref_replay_sample.argtypes = [C.c_void_p, C.c_size_t, u64p]
        L.ref_replay_consumed.restype = C.c_uint64
        L.ref_replay_consumed.argtypes = [C.c_void_p]
        L.ref_replay_size.restype = C.c_size_t
        L.ref_replay_size.argtypes = [C.c_void_p]
        L.ref_learner_create.restype = C.c_void_p
        L.ref_learner_create.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                         C.c_uint64, C.POINTER(RefHyper), C.c_uint32,
                                         C.c_uint32, C.c_uint32, C.c_size_t, C.c_uint64]
        L.ref_learner_destroy.argtypes = [C.c_void_p]
        L.ref_learner_push.argtypes = [C.c_void_p, C.POINTER(RefSegments)]
        L.ref_learner_train_step.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.ref_learner_param_count.restype = C.c_size_t
        L.ref_learner_param_count.argtypes = [C.c_void_p]
        L.ref_learner_params.argtypes = [C.c_void_p, f64p]
        L.ref_learner_pool_params.argtypes = [C.c_void_p, C.c_char_p, f64p]
        L.ref_learner_consumed.restype = C.c_uint64
        L.ref_learner_consumed.argtypes = [C.c_void_p]
        L.ref_learner_replay_size.restype = C.c_size_t
        L.ref_learner_replay_size.argtypes = [C.c_void_p]

    def _chk(self, rc):
        _raise(rc, self.L.ref_last_error())

    def gae(self, r, v, done, boot, gamma, lam):
        out = np.zeros(len(r))
        self._chk(self.L.ref_gae(np.ascontiguousarray(r, np.float64),
                                 np.ascontiguousarray(v, np.float64),
                                 np.ascontiguousarray(done, np.uint8), len(r), boot, gamma, lam,
                                 out))
        return out

    def lambda_return(self, r, v, done, boot, gamma, lam):
        out = np.zeros(len(r))
        self._chk(self.L.ref_lambda_return(np.ascontiguousarray(r, np.float64),
                                           np.ascontiguousarray(v, np.float64),
                                           np.ascontiguousarray(done, np.uint8), len(r), boot,
                                           gamma, lam, out))
        return out

    def vtrace(self, bl, tl, r, v, done, boot, gamma, rho_bar, c_bar):
        vs = np.zeros(len(r)); pg = np.zeros(len(r))
        self._chk(self.L.ref_vtrace(*(np.ascontiguousarray(x, np.float64) for x in (bl, tl, r, v)),
                                    np.ascontiguousarray(done, np.uint8), len(r), boot, gamma,
                                    rho_bar, c_bar, vs, pg))
        return vs, pg

    def param_count(self, shape: Shape):
        return self.L.ref_param_count(shape.family, shape.obs_dim, shape.n_actions)

    def init_params(self, shape: Shape, scale, seed):
        out = np.zeros(self.param_count(shape))
        self._chk(self.L.ref_init_params(shape.family, shape.obs_dim, shape.n_actions, scale,
                                         seed, out))
        return out

    def batch_forward(self, shape: Shape, params, obs):
        obs = np.ascontiguousarray(obs, np.float64).reshape(-1, shape.obs_dim)
        n = obs.shape[0]
        lg = np.zeros((n, shape.n_actions)); pr = np.zeros_like(lg); v = np.zeros(n)
        self._chk(self.L.ref_batch_forward(shape.family, shape.obs_dim, shape.n_actions,
                                           np.ascontiguousarray(params, np.float64), obs, n, lg,
                                           pr, v))
        return lg, pr, v

    def _loss(self, fn, shape, params, teacher, obs, action, blogp, adv, vtarget, hyper):
        n = len(action)
        grad = np.zeros(self.param_count(shape)); loss = np.zeros(1); st = np.zeros(4)
        args = [shape.family, shape.obs_dim, shape.n_actions,
                np.ascontiguousarray(params, np.float64)]
        if fn == "ppo":
            t = None if teacher is None else np.ascontiguousarray(teacher, np.float64)
            args.append(None if t is None else t.ctypes.data)
        args += [n, np.ascontiguousarray(obs, np.float64).reshape(-1),
                 np.ascontiguousarray(action, np.uint32),
                 *(np.ascontiguousarray(x, np.float64) for x in (blogp, adv, vtarget)),
                 C.byref(hyper.c(RefHyper)), loss, grad, st]
        self._chk(getattr(self.L, f"ref_{fn}_loss_grad")(*args))
        stats = dict(loss=loss[0], clip_fraction=st[0], mean_ratio=st[1], entropy=st[2],
                     value_loss=st[3])
        return stats, grad

    def ppo_loss_grad(self, shape, params, obs, action, blogp, adv, vtarget, hyper, teacher=None):
        return self._loss("ppo", shape, params, teacher, obs, action, blogp, adv, vtarget, hyper)

    def pg_loss_grad(self, shape, params, obs, action, blogp, adv, vtarget, hyper):
        return self._loss("pg", shape, params, None, obs, action, blogp, adv, vtarget, hyper)

    def sgd_step(self, shape, params, grad, lr):
        out = np.zeros(len(params))
        self._chk(self.L.ref_sgd_step(shape.family, shape.obs_dim, shape.n_actions,
                                      np.ascontiguousarray(params, np.float64),
                                      np.ascontiguousarray(grad, np.float64), lr, out))
        return out


class RefLearner:
    """The reference Learner (learner.cpp) behind LeagueState + DirectPool."""

    def __init__(self, ref: RefLib, shape: Shape, hyper: Hyper, *, init_scale=0.3,
                 league_seed=42, num_shards=1, algo=0, publish_interval=10,
                 replay_capacity=4096, seed=0):
        self.ref = ref
        self.h = ref.L.ref_learner_create(shape.family, shape.obs_dim, shape.n_actions,
                                          init_scale, league_seed, C.byref(hyper.c(RefHyper)),
                                          num_shards, algo, publish_interval, replay_capacity,
                                          seed)
        if not self.h:
            raise InvalidArgument(ref.L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.ref_learner_destroy(self.h)
            self.h = None

    def push(self, segs: Segments):
        cs = segs.c_ref()
        self.ref._chk(self.ref.L.ref_learner_push(self.h, C.byref(cs)))

    def train_step(self) -> bool:
        ok = C.c_int32(0)
        self.ref._chk(self.ref.L.ref_learner_train_step(self.h, C.byref(ok)))
        return bool(ok.value)

    def params(self):
        out = np.zeros(self.ref.L.ref_learner_param_count(self.h))
        self.ref._chk(self.ref.L.ref_learner_params(self.h, out))
        return out

    def consumed(self):
        return self.ref.L.ref_learner_consumed(self.h)


def try_ref():
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None
