"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs oracle/_ref, i.e. `make -C oracle ref`, which
compiles /root/reference/proj/src):

    python tests/golden/make_golden.py

Every output array below is produced by the reference's own routines through
oracle/ref_capi.cpp; the inputs are seeded numpy draws shaped like the
reference's own test generators (rlmath_test.cpp:32-54, :292-328,
learner_test.cpp:43-60).  The committed .npz files let the oracle be pinned on
machines where /root/reference does not exist (the GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_ffi import Hyper, RefLearner, RefLib, Segments, Shape  # noqa: E402


def random_instance(rng, with_dones=True, n=None):
    """rlmath_test.cpp:32-54 distribution (len 1..12 unless given)."""
    n = int(rng.integers(1, 13)) if n is None else n
    r = rng.uniform(-1, 1, n)
    v = rng.uniform(-1, 1, n)
    bl = -0.2 - rng.uniform(0, 1, n)
    tl = bl + 0.4 * rng.uniform(-1, 1, n)
    done = ((rng.uniform(0, 1, n) < 0.2) & with_dones).astype(np.uint8)
    boot = rng.uniform(-1, 1)
    gamma = 0.5 + 0.5 * rng.uniform(0, 1)
    lam = rng.uniform(0, 1)
    return r, v, bl, tl, done, boot, gamma, lam


def gen_returns(ref, path):
    rng = np.random.default_rng(2024)
    recs = {k: [] for k in ("r", "v", "bl", "tl", "done", "gae", "lr", "vs", "pg")}
    scal = []
    lengths = [None] * 400 + [32] * 20 + [80] * 10 + [64] * 10
    for n in lengths:
        r, v, bl, tl, done, boot, gamma, lam = random_instance(rng, n=n)
        c_bar = 0.5 + rng.uniform(0, 1)
        rho_bar = c_bar + rng.uniform(0, 1)
        gae = ref.gae(r, v, done, boot, gamma, lam)
        lr = ref.lambda_return(r, v, done, boot, gamma, lam)
        vs, pg = ref.vtrace(bl, tl, r, v, done, boot, gamma, rho_bar, c_bar)
        for k, a in zip(recs, (r, v, bl, tl, done, gae, lr, vs, pg)):
            recs[k].append(a)
        scal.append((len(r), boot, gamma, lam, rho_bar, c_bar))
    np.savez_compressed(path, scal=np.array(scal),
                        **{k: np.concatenate(v) for k, v in recs.items()})


def gen_policy(ref, path):
    rng = np.random.default_rng(77)
    out = {}
    cases = []
    for i in range(24):
        fam = i % 2
        shape = Shape(fam, int(2 + rng.integers(0, 7)), int(2 + rng.integers(0, 5)))
        scale = [0.0, 0.3, 1.0][i % 3]
        seed = int(rng.integers(0, 2**63))
        p = ref.init_params(shape, scale, seed)
        n = 16
        if fam == 0:
            obs = np.zeros((n, shape.obs_dim))
            obs[np.arange(n), rng.integers(0, shape.obs_dim, n)] = 1.0
        else:
            obs = rng.standard_normal((n, shape.obs_dim))
        lg, pr, v = ref.batch_forward(shape, p, obs)
        cases.append((fam, shape.obs_dim, shape.n_actions, scale, seed))
        for k, a in (("params", p), ("obs", obs), ("logits", lg), ("probs", pr), ("value", v)):
            out[f"{k}_{i}"] = a
    np.savez_compressed(path, cases=np.array(cases, dtype=np.float64),
                        seeds=np.array([c[4] for c in cases], dtype=np.uint64), **out)


def fd_case(rng, ref, near_on_policy):
    """rlmath_test.cpp:292-328 / acceptance.cpp:489-523 shape."""
    fam = int(rng.integers(0, 2))
    shape = Shape(fam, int(2 + rng.integers(0, 3)), int(2 + rng.integers(0, 3)))
    params = ref.init_params(shape, 1.0, int(rng.integers(0, 2**63)))
    teacher = ref.init_params(shape, 1.0, int(rng.integers(0, 2**63)))
    n = int(4 + rng.integers(0, 8))
    obs = np.zeros((n, shape.obs_dim))
    if fam == 0:
        obs[np.arange(n), rng.integers(0, shape.obs_dim, n)] = 1.0
    else:
        obs = rng.standard_normal((n, shape.obs_dim))
    _, probs, _ = ref.batch_forward(shape, params, obs)
    action = rng.integers(0, shape.n_actions, n).astype(np.uint32)
    jit = (0.02 if near_on_policy else 0.08) * rng.uniform(-1, 1, n)
    blogp = np.log(probs[np.arange(n), action]) + jit
    adv = rng.uniform(-1, 1, n)
    vt = rng.uniform(-1, 1, n)
    hp = Hyper(clip_eps=0.2, vf_coef=0.3 + 0.4 * rng.uniform(0, 1),
               ent_coef=0.01 * rng.uniform(0, 1), adv_norm=bool(rng.integers(0, 2)))
    return shape, params, teacher, obs, action, blogp, adv, vt, hp


def gen_losses(ref, path):
    rng = np.random.default_rng(8080)
    out = {}
    meta = []
    for i in range(60):
        kind = ["ppo", "ppo_teacher", "pg", "ppo_far"][i % 4]
        shape, params, teacher, obs, action, blogp, adv, vt, hp = fd_case(
            rng, ref, near_on_policy=kind != "ppo_far")
        if kind == "ppo_teacher":
            hp.kl_teacher_coef = 0.1
        if kind.startswith("ppo"):
            st, g = ref.ppo_loss_grad(shape, params, obs, action, blogp, adv, vt, hp,
                                      teacher if kind == "ppo_teacher" else None)
        else:
            st, g = ref.pg_loss_grad(shape, params, obs, action, blogp, adv, vt, hp)
        meta.append((["ppo", "ppo_teacher", "pg", "ppo_far"].index(kind), shape.family,
                     shape.obs_dim, shape.n_actions, hp.vf_coef, hp.ent_coef, float(hp.adv_norm),
                     hp.kl_teacher_coef, st["loss"], st["clip_fraction"], st["mean_ratio"],
                     st["entropy"], st["value_loss"]))
        for k, a in (("params", params), ("teacher", teacher), ("obs", obs), ("action", action),
                     ("blogp", blogp), ("adv", adv), ("vt", vt), ("grad", g)):
            out[f"{k}_{i}"] = a
    np.savez_compressed(path, meta=np.array(meta), **out)


def make_stream(rng, n, T, D, A, one_state=False):
    """learner_test.cpp:43-60 (one_state) or a C1-like linear stream."""
    if one_state:
        obs = np.ones((n, T, 1))
        action = rng.integers(0, 3, (n, T)).astype(np.uint32)
        reward = rng.uniform(-1, 1, (n, T))
        blogp = np.log(1.0 / 3) + 0.1 * rng.uniform(-1, 1, (n, T))
        value = rng.uniform(-1, 1, (n, T))
        done = np.zeros((n, T), np.uint8)
        done[:, -1] = 1
        boot = np.zeros(n)
        valid = np.full(n, T, np.uint32)
    else:
        obs = rng.standard_normal((n, T, D)).astype(np.float32).astype(np.float64)
        action = rng.integers(0, A, (n, T)).astype(np.uint32)
        reward = rng.uniform(-1, 1, (n, T)).astype(np.float32).astype(np.float64)
        blogp = (np.log(1.0 / A) + 0.1 * rng.uniform(-1, 1, (n, T))).astype(np.float32).astype(np.float64)
        value = rng.uniform(-1, 1, (n, T)).astype(np.float32).astype(np.float64)
        done = (rng.uniform(0, 1, (n, T)) < 0.01).astype(np.uint8)
        boot = rng.uniform(-1, 1, n).astype(np.float32).astype(np.float64)
        valid = np.full(n, T, np.uint32)
        rag = rng.uniform(0, 1, n) < 1 / 16
        valid[rag] = rng.integers(1, T + 1, int(rag.sum()))
        pad = np.arange(T)[None, :] >= valid[:, None]
        for a in (reward, value, blogp):
            a[pad] = 0
        action[pad] = 0
        done[pad] = 0
        obs[pad] = 0
    return Segments(obs, action, reward, blogp, value, done, boot, valid)


def gen_learner(ref, path):
    out = {}
    meta = []
    runs = [
        # name, family, D, A, T, B(per shard), shards, algo, max_reuse, steps
        ("tab_ppo", 0, 1, 3, 3, 4, 2, 0, 1, 12),
        ("tab_vtrace", 0, 1, 3, 3, 4, 2, 1, 2, 12),
        ("lin_ppo", 1, 64, 6, 32, 8, 1, 0, 1, 4),
        ("lin_vtrace", 1, 16, 6, 20, 6, 2, 1, 2, 4),
    ]
    for ri, (name, fam, D, A, T, B, shards, algo, reuse, steps) in enumerate(runs):
        hp = Hyper(learning_rate=0.05, batch_size=B, max_reuse=reuse, unroll_len=T)
        shape = Shape(fam, D, A)
        lrn = RefLearner(ref, shape, hp, init_scale=0.3, league_seed=42, num_shards=shards,
                         algo=algo, publish_interval=1, seed=99)
        rng = np.random.default_rng(2024 + ri)
        out[f"{name}_p0"] = lrn.params()
        draw = B * shards
        for s in range(steps):
            seg = make_stream(rng, draw, T, D, A, one_state=(fam == 0))
            seg.segment_seq = np.arange(s * draw, (s + 1) * draw, dtype=np.uint64)
            lrn.push(seg)
            assert lrn.train_step()
            for k in ("obs", "action", "reward", "behavior_logp", "value_est", "done",
                      "bootstrap", "valid_steps"):
                out[f"{name}_s{s}_{k}"] = getattr(seg, k)
            out[f"{name}_p{s + 1}"] = lrn.params()
        meta.append((ri, fam, D, A, T, B, shards, algo, reuse, steps))
    np.savez_compressed(path, meta=np.array(meta), **out)


def gen_replay(ref, path):
    L = ref.L
    out = {}
    meta = []
    for ci, (cap, reuse, seed, pushes, draws) in enumerate(
            [(64, 1, 99, 200, 8), (64, 3, 7, 200, 8), (16, 2, 123, 100, 4), (4096, 1, 5, 3000, 64)]):
        h = L.ref_replay_create(cap, reuse, seed)
        rng = np.random.default_rng(ci)
        seqs = []
        valid = rng.integers(1, 33, pushes).astype(np.uint32)
        seq = 0
        consumed = []
        while seq < pushes:
            for _ in range(draws):
                if seq < pushes:
                    L.ref_replay_push(h, seq, int(valid[seq]))
                    seq += 1
            n = draws // 2
            if L.ref_replay_size(h) >= n:
                o = np.zeros(n, np.uint64)
                assert L.ref_replay_sample(h, n, o) == 0
                seqs.append(o)
                consumed.append(L.ref_replay_consumed(h))
        L.ref_replay_destroy(h)
        out[f"valid_{ci}"] = valid
        out[f"draws_{ci}"] = np.concatenate(seqs)
        out[f"consumed_{ci}"] = np.array(consumed, np.uint64)
        meta.append((cap, reuse, seed, pushes, draws))
    np.savez_compressed(path, meta=np.array(meta, np.uint64), **out)


def main():
    ref = RefLib()
    gen_returns(ref, os.path.join(HERE, "returns.npz"))
    gen_policy(ref, os.path.join(HERE, "policy.npz"))
    gen_losses(ref, os.path.join(HERE, "losses.npz"))
    gen_learner(ref, os.path.join(HERE, "learner.npz"))
    gen_replay(ref, os.path.join(HERE, "replay.npz"))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
