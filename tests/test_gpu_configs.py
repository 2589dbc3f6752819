"""GPU parity at the BASELINE.json configurations' real shapes.

Every config runs through the C ABI (the product path) and is checked step by step
against the fp64 checker (tests/f64_checker.py: the oracle's arithmetic as batched
float64 GEMMs on the device, pinned to oracle/tlg_oracle.cpp by
tests/test_f64_checker.py); C1 is also checked against the per-sample oracle itself.

Per step, at the GPU's own current parameters (so no drift is amplified):
* returns / advantages (adv, value target per frame): Close(., 1e-5) for GAE /
  lambda-return.  V-trace targets are a function of the learner's own forward (the
  target log-probs under the current parameters, learner.cpp:80-84), so end to end they
  carry the forward's 1e-4 class; the returns kernel itself is checked at 1e-5 at the
  config's shape through tlg_returns on the checker's target log-probs
* loss, clip_fraction, mean_ratio, entropy, value_loss: Close(., 1e-4)
* the averaged gradient: within 1e-4 of the gradient's largest magnitude
* SGD: updated parameters Close(., 1e-4) against p - lr * g_checker
* Adam: updated parameters Close(., 1e-4) against torch-semantics Adam applied to
  the GPU's gradient history (a gradient entry of ~1e-9 can flip sign under fp32
  rounding, which Adam's normalisation turns into a +-lr step; the gradient itself is
  checked against fp64 above)

Close(a, b, tol) = |a-b| <= tol * max(1, |a|, |b|) (acceptance.cpp:439-441).  The worst
errors are printed (and appended to $TLG_PARITY_LOG as JSON lines when set).
"""
import json
import os

import numpy as np
import pytest
import torch

import f64_checker as fc

pytestmark = pytest.mark.gpu

ALGO = {"ppo": 0, "vtrace": 1, "ppo_vtrace": 2}


def worst(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))


def _log(rec):
    print(json.dumps(rec))
    path = os.environ.get("TLG_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _bits_view(tlg, b, D, device_pitch=0):
    from paper_2011_12895_b200._capi import DeviceSegmentBatch, SegmentBatchView
    pb = b.slice(0, b.n_segments)
    pb.obs = tlg.synth.pack_bits(b.obs)
    if device_pitch:
        return DeviceSegmentBatch(pb, bits=True, obs_dim=D, pitch=device_pitch), True
    return SegmentBatchView(pb, bits=True, obs_dim=D), False


def _vtrace_kernel_worst(b, tl, hp):
    """tlg_returns (K1, V-trace) at the batch's shape on the checker's target log-probs
    rounded to fp32, against the checker's V-trace on the same rounded inputs."""
    import ctypes as C
    from paper_2011_12895_b200._capi import Hyper, check, lib
    dev = torch.device("cuda", 0)
    S, T = b.action.shape
    tl32 = tl.to(torch.float32).contiguous()
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in dict(
        r=b.reward, v=b.value_est, d=b.done, boot=b.bootstrap, valid=b.valid_steps,
        bl=b.behavior_logp).items()}
    adv = torch.zeros(S, T, device=dev)
    tgt = torch.zeros(S, T, device=dev)
    h = Hyper.make(gamma=hp["gamma"], lam=hp["lam"], rho_bar=hp["rho_bar"], c_bar=hp["c_bar"])
    torch.cuda.synchronize()
    check(lib().tlg_returns(1, C.byref(h), S, T, t["r"].data_ptr(), t["v"].data_ptr(),
                            t["d"].data_ptr(), t["boot"].data_ptr(), t["valid"].data_ptr(),
                            t["bl"].data_ptr(), tl32.data_ptr(), adv.data_ptr(),
                            tgt.data_ptr(), None))
    d64 = {k: v.double() for k, v in t.items() if k not in ("d", "valid")}
    wa, wt = fc.returns(1, hp, d64["r"], d64["v"], t["d"], d64["boot"], t["valid"].long(),
                        d64["bl"], tl32.double())
    return max(worst(adv.cpu().numpy(), wa.cpu().numpy()), worst(tgt.cpu().numpy(),
                                                                  wt.cpu().numpy()))


def run_config(tlg, name, *, D, A, hidden, S, T, algo, optimizer, steps, lr, obs_kind="gauss",
               seed=0, oracle=None, n_shards=1):
    dev = torch.device("cuda", 0)
    bits = obs_kind == "binary"
    net = fc.Net(2, D, A, hidden)
    lrn = tlg.Learner("mlp", D, A, hidden, algo=algo, optimizer=optimizer, max_segments=S,
                      unroll_len=T, obs_u8=bits)
    hp = dict(learning_rate=lr, gamma=0.99, lam=0.95, clip_eps=0.2, vf_coef=0.5,
              ent_coef=0.01, rho_bar=1.0, c_bar=1.0, batch_size=S, unroll_len=T,
              adv_norm=True)
    lrn.set_hyper(**hp)
    rng = np.random.default_rng(1000 + seed)
    # InitParams-style U[-s, s] over the flat vector, fp32-representable; a 1/sqrt(fan-in)
    # scale keeps the tanh trunk out of saturation at widths up to 2048
    p0 = np.concatenate([
        rng.uniform(-1, 1, net.P).astype(np.float32).astype(np.float64)])
    scale = np.full(net.P, 0.1)  # biases
    for l in range(len(hidden)):
        w0, n_w = net.w_off[l], net.dims[l + 1] * net.dims[l]
        scale[w0:w0 + n_w] = 1.5 / np.sqrt(net.dims[l])
    H = net.dims[-1]
    scale[net.wpi:net.wpi + A * H] = 1.0 / np.sqrt(H)  # policy head
    scale[net.wv:net.wv + H] = 1.0 / np.sqrt(H)        # value head
    p0 = (p0 * scale).astype(np.float32).astype(np.float64)
    lrn.set_params(p0)
    m = torch.zeros(net.P, dtype=torch.float64, device=dev)
    v = torch.zeros_like(m)
    rec = dict(config=name, S=S, T=T, D=D, hidden=list(hidden), algo=algo, optimizer=optimizer,
               shards=n_shards, steps=steps, worst_returns=0.0, worst_stats=0.0, worst_grad=0.0,
               worst_params=0.0)
    for step in range(1, steps + 1):
        shards = [tlg.synth.make_segments(S, T, D, A, seed=seed * 100 + step * 10 + k,
                                          obs_kind=obs_kind, obs_u8=bits)
                  for k in range(n_shards)]
        p_prev = lrn.get_params()
        if bits:
            views = [_bits_view(tlg, b, D, device_pitch=(((D + 7) // 8 + 15) // 16 * 16)
                                if step % 2 == 0 else 0) for b in shards]
            on_dev = views[0][1]
            views = [x[0] for x in views]
        else:
            views, on_dev = shards, False
        if n_shards == 1:
            sts = [lrn.train_step(views[0], on_device=on_dev)]
        else:
            sts = lrn.train_step_shards(views, on_device=on_dev)
        g_gpu = lrn.get_grad()
        adv_gpu, tgt_gpu = lrn.get_returns(S * T)
        p_gpu = lrn.get_params()
        pt = torch.tensor(p_prev, dtype=torch.float64, device=dev)
        stats, g, (adv, tgt, tl) = fc.learner_step(net, pt, hp, ALGO[algo], shards, dev)
        g = g.cpu().numpy()
        wr = max(worst(adv_gpu, adv.reshape(-1).cpu().numpy()),
                 worst(tgt_gpu, tgt.reshape(-1).cpu().numpy()))
        if algo == "ppo":
            assert wr <= 1e-5, (name, step, "returns", wr)
        else:
            assert wr <= 1e-4, (name, step, "returns (through the forward)", wr)
            wk = _vtrace_kernel_worst(shards[-1], tl, hp)
            rec["worst_returns_kernel"] = max(rec.get("worst_returns_kernel", 0.0), wk)
            assert wk <= 1e-5, (name, step, "V-trace returns kernel", wk)
        ws = 0.0
        for st, sw in zip(sts, stats):
            assert st["n_samples"] == sw["n_samples"]
            for k in ("loss", "clip_fraction", "mean_ratio", "entropy", "value_loss"):
                e = worst(st[k], sw[k])
                ws = max(ws, e)
                assert e <= 1e-4, (name, step, k, st[k], sw[k])
        gscale = float(np.max(np.abs(g)))
        wg = float(np.max(np.abs(g_gpu - g))) / max(gscale, 1e-30)
        assert wg <= 1e-4, (name, step, "grad", wg)
        if optimizer == "sgd":
            want = p_prev - lr * g
        else:
            gg = torch.tensor(g_gpu, dtype=torch.float64, device=dev)
            want_t, m, v = fc.adam(pt, gg, m, v, step, lr)
            want = want_t.cpu().numpy()
        wp = worst(p_gpu, want)
        assert wp <= 1e-4, (name, step, "params", wp)
        if oracle is not None and step == 1:
            from oracle_ffi import Hyper, Segments, Shape
            segs = [Segments(b.obs.astype(np.float64), b.action.astype(np.uint32),
                             b.reward.astype(np.float64), b.behavior_logp.astype(np.float64),
                             b.value_est.astype(np.float64), b.done.astype(np.uint8),
                             b.bootstrap.astype(np.float64), b.valid_steps.astype(np.uint32))
                    for b in shards]
            _, og, ost, _ = oracle.learner_step(Shape(2, D, A, hidden), p_prev, Hyper(**hp),
                                                ALGO[algo], segs)
            assert np.max(np.abs(og - g)) <= 1e-10 * max(gscale, 1e-30)
            assert abs(ost[0]["loss"] - stats[0]["loss"]) <= 1e-10 * max(1, abs(ost[0]["loss"]))
            wo = float(np.max(np.abs(g_gpu - og))) / max(gscale, 1e-30)
            rec["worst_grad_vs_oracle"] = wo
            assert wo <= 1e-4
        rec["worst_returns"] = max(rec["worst_returns"], wr)
        rec["worst_stats"] = max(rec["worst_stats"], ws)
        rec["worst_grad"] = max(rec["worst_grad"], wg)
        rec["worst_params"] = max(rec["worst_params"], wp)
        rec.setdefault("loss", []).append(sts[0]["loss"])
    _log(rec)
    del lrn
    torch.cuda.empty_cache()


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_c1_ppo_mlp256_b64(tlg, oracle, optimizer):
    """C1: PPO, MLP 64-256-256-(6,1), GAE, T=32, B=64 (also against the oracle itself)."""
    run_config(tlg, "C1", D=64, A=6, hidden=(256, 256), S=64, T=32, algo="ppo",
               optimizer=optimizer, steps=3, lr=3e-3 if optimizer == "adam" else 0.05, seed=1,
               oracle=oracle)


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_c2_vtrace_mlp512_t80_b256(tlg, optimizer):
    """C2: V-trace learner, MLP 64-512-512-(6,1), T=80, B=256."""
    run_config(tlg, "C2", D=64, A=6, hidden=(512, 512), S=256, T=80, algo="vtrace",
               optimizer=optimizer, steps=3, lr=3e-4 if optimizer == "adam" else 0.02, seed=2)


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_c3_bit_planes_full_4096x32_shard(tlg, optimizer):
    """C3: Pommerman-shaped 11x11x16 binary planes (bit-packed, int8 layer-1 tensor-core
    path incl. the 9-split int8 dW1 and the split-K dW2 over 131,072 frames), PPO,
    MLP 1936-256-256-(6,1), the full per-GPU shard B=4096 x T=32."""
    run_config(tlg, "C3", D=1936, A=6, hidden=(256, 256), S=4096, T=32, algo="ppo",
               optimizer=optimizer, steps=3, lr=3e-4 if optimizer == "adam" else 0.02,
               obs_kind="binary", seed=3)


def test_c5_ppo_vtrace_4x2048_s64(tlg):
    """C5 net at S=64 x T=64: PPO surrogate over V-trace targets, 64-2048^4-(6,1)."""
    run_config(tlg, "C5-S64", D=64, A=6, hidden=(2048,) * 4, S=64, T=64, algo="ppo_vtrace",
               optimizer="adam", steps=3, lr=3e-4, seed=5)


def test_c5_ppo_vtrace_4x2048_full_shard(tlg):
    """C5: one full per-GPU shard at 8 GPUs, B=16384/8=2048 segments x T=64 (131,072
    frames), 12.7M parameters, SGD so the update is checked end to end."""
    run_config(tlg, "C5-S2048", D=64, A=6, hidden=(2048,) * 4, S=2048, T=64,
               algo="ppo_vtrace", optimizer="sgd", steps=2, lr=0.01, seed=6)


def test_c3_two_local_shards_strong_split(tlg):
    """C3's 4096-segment draw split over 2 shards (the 2-GPU strong-scaling shard size,
    here as local shards: per-shard adv-norm and 1/n, rank-ordered mean)."""
    run_config(tlg, "C3-2x2048", D=1936, A=6, hidden=(256, 256), S=2048, T=32, algo="ppo",
               optimizer="adam", steps=2, lr=3e-4, obs_kind="binary", seed=7, n_shards=2)
