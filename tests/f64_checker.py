"""TEST INFRASTRUCTURE ONLY -- a batched torch-float64 restatement of the fp64 oracle.

oracle/tlg_oracle.cpp evaluates the learner step sample by sample (its MLP backward
scatters into the full flat gradient per frame), which is exact but far too slow at the
BASELINE shapes (C3: 131,072 frames x 563K parameters; C5: 12.7M parameters).  This
module restates the same arithmetic with whole-batch float64 GEMMs so that it runs on
the GPU box's device in seconds:

* BuildMinibatch (learner.cpp:56-102): segment-major, t-minor, padding skipped,
  segments with valid_steps == 0 contribute nothing
* GaeAdvantages / LambdaReturn / VtraceTargets (rlmath.cpp:45-114) as reverse
  recursions over t, vectorised over segments
* EffectiveAdvantages (rlmath.cpp:18-34): per-shard mean / population std, floor 1e-8
* PpoLossAndGrad / PgLossAndGrad (rlmath.cpp:116-222): analytic dlogits and dvalue per
  sample (gradient through the ratio only when t1 <= t2), x 1/n
* the MLP family's forward / chain rule exactly as oracle Forward / Backward
  (tlg_oracle.cpp:142-263), linear family as policy.cpp:82-104
* rank-ordered shard mean (learner.cpp:138-149), SgdStep (rlmath.cpp:224-232) and
  torch.optim.Adam semantics (tlg_oracle.cpp orc_adam_step)

It is pinned to tlg_oracle at small shapes by tests/test_f64_checker.py (CPU, 1e-10);
only tests/ import it.  Nothing here is on the product path.
"""
from __future__ import annotations

import numpy as np
import torch

F64 = torch.float64


class Net:
    """Flat layout of oracle MakeLayout (tlg_oracle.cpp:55-98): mlp
    [W_1 (h1 x d), b_1, ..., W_L, b_L | W_pi (A x hL), b_pi | w_v (hL), b_v]; linear
    [W (A x d) | v (d)]."""

    def __init__(self, family, obs_dim, n_actions, hidden=()):
        assert family in (1, 2), "tabular is checked by the oracle itself"
        self.family, self.d, self.a = family, obs_dim, n_actions
        self.hidden = tuple(hidden) if family == 2 else ()
        dims = [obs_dim] + list(self.hidden)
        self.dims = dims
        off = 0
        self.w_off, self.b_off = [], []
        for l in range(len(self.hidden)):
            self.w_off.append(off)
            off += dims[l + 1] * dims[l]
            self.b_off.append(off)
            off += dims[l + 1]
        hl = dims[-1]
        if family == 2:
            self.wpi = off; off += n_actions * hl
            self.bpi = off; off += n_actions
            self.wv = off; off += hl
            self.bv = off; off += 1
        else:
            self.wpi = 0
            self.wv = n_actions * obs_dim
            self.bpi = self.bv = None
            off = self.wv + obs_dim
        self.P = off

    def views(self, p):
        L = len(self.hidden)
        Ws = [p[self.w_off[l]:self.w_off[l] + self.dims[l + 1] * self.dims[l]].view(
            self.dims[l + 1], self.dims[l]) for l in range(L)]
        bs = [p[self.b_off[l]:self.b_off[l] + self.dims[l + 1]] for l in range(L)]
        hl = self.dims[-1]
        Wpi = p[self.wpi:self.wpi + self.a * hl].view(self.a, hl)
        wv = p[self.wv:self.wv + hl]
        bpi = p[self.bpi:self.bpi + self.a] if self.bpi is not None else None
        bv = p[self.bv] if self.bv is not None else None
        return Ws, bs, Wpi, bpi, wv, bv

    def forward(self, p, x):
        """Distribution + ValueEstimate for a batch: logits [N,A], value [N], trunk acts."""
        Ws, bs, Wpi, bpi, wv, bv = self.views(p)
        acts = []
        h = x
        for W, b in zip(Ws, bs):
            h = torch.tanh(h @ W.T + b)
            acts.append(h)
        z = h @ Wpi.T
        v = h @ wv
        if bpi is not None:
            z = z + bpi
            v = v + bv
        return z, v, acts

    def backward(self, p, x, acts, dz, dv):
        """Chain rule of oracle Backward (tlg_oracle.cpp:195-263), summed over the batch."""
        Ws, bs, Wpi, bpi, wv, bv = self.views(p)
        g = torch.zeros(self.P, dtype=F64, device=p.device)
        hL = acts[-1] if acts else x
        g[self.wpi:self.wpi + self.a * hL.shape[1]] = (dz.T @ hL).reshape(-1)
        g[self.wv:self.wv + hL.shape[1]] = dv @ hL
        if self.family == 1:
            return g
        g[self.bpi:self.bpi + self.a] = dz.sum(0)
        g[self.bv] = dv.sum()
        dh = dz @ Wpi + dv[:, None] * wv[None, :]
        for l in range(len(Ws) - 1, -1, -1):
            h = acts[l]
            hin = x if l == 0 else acts[l - 1]
            dpre = dh * (1.0 - h * h)
            n_w = Ws[l].numel()
            g[self.w_off[l]:self.w_off[l] + n_w] = (dpre.T @ hin).reshape(-1)
            g[self.b_off[l]:self.b_off[l] + Ws[l].shape[0]] = dpre.sum(0)
            if l > 0:
                dh = dpre @ Ws[l]
            del dpre
        return g


def _t(a, dev, dtype=F64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def returns(algo, hp, reward, value, done, boot, valid, blogp=None, tlogp=None):
    """[S,T] tensors -> (adv, target) [S,T], padding 0.  algo 0: GAE + lambda-return
    (rlmath.cpp:45-78); 1/2: V-trace pg_adv + vs (rlmath.cpp:80-114)."""
    S, T = reward.shape
    dev = reward.device
    gamma, lam = hp["gamma"], hp["lam"]
    adv = torch.zeros(S, T, dtype=F64, device=dev)
    tgt = torch.zeros(S, T, dtype=F64, device=dev)
    nt = 1.0 - done.to(F64)
    tix = torch.arange(T, device=dev)
    active = tix[None, :] < valid[:, None]
    if algo == 0:
        nv = boot.clone(); na = torch.zeros(S, dtype=F64, device=dev); ng = boot.clone()
        for t in range(T - 1, -1, -1):
            a = active[:, t]
            delta = reward[:, t] + gamma * nt[:, t] * nv - value[:, t]
            A = delta + gamma * lam * nt[:, t] * na
            G = reward[:, t] + gamma * nt[:, t] * ((1.0 - lam) * nv + lam * ng)
            adv[:, t] = torch.where(a, A, 0.0)
            tgt[:, t] = torch.where(a, G, 0.0)
            na = torch.where(a, A, na)
            ng = torch.where(a, G, ng)
            nv = torch.where(a, value[:, t], nv)
        return adv, tgt
    w = torch.exp(tlogp - blogp)
    rho = torch.clamp(w, max=hp["rho_bar"])
    c = torch.clamp(w, max=hp["c_bar"])
    nvs = boot.clone(); nv = boot.clone()
    vs = torch.zeros(S, T, dtype=F64, device=dev)
    for t in range(T - 1, -1, -1):
        a = active[:, t]
        delta = rho[:, t] * (reward[:, t] + gamma * nt[:, t] * nv - value[:, t])
        x = value[:, t] + delta + gamma * nt[:, t] * c[:, t] * (nvs - nv)
        vs[:, t] = torch.where(a, x, 0.0)
        nvs = torch.where(a, x, nvs)
        nv = torch.where(a, value[:, t], nv)
    # vs_{t+1}, with vs_n := bootstrap
    vs_next = torch.cat([vs[:, 1:], torch.zeros(S, 1, dtype=F64, device=dev)], 1)
    last = tix[None, :] == (valid[:, None] - 1)
    vs_next = torch.where(last, boot[:, None], vs_next)
    pg = rho * (reward + gamma * nt * vs_next - value)
    adv = torch.where(active, pg, 0.0)
    return adv, torch.where(active, vs, 0.0)


def shard_step(net: Net, p, hp, algo, b, dev, chunk=1 << 15):
    """One shard: BuildMinibatch + loss/grad (learner.cpp:117-128).  b is a synth
    SegmentBatch (fp32-representable arrays; obs may be uint8 planes).  Returns
    (stats dict, grad [P] f64 tensor, adv [S,T], target [S,T], target logp [S,T] | None)."""
    S, T = b.action.shape
    D = net.d
    obs = _t(np.asarray(b.obs).reshape(S * T, D), dev)
    act = _t(b.action.reshape(-1), dev, torch.int64)
    blogp = _t(b.behavior_logp, dev)
    valid = _t(b.valid_steps, dev, torch.int64)
    r, v, dn = _t(b.reward, dev), _t(b.value_est, dev), _t(b.done, dev)
    boot = _t(b.bootstrap, dev)
    mask = (torch.arange(T, device=dev)[None, :] < valid[:, None]).reshape(-1)
    idx = torch.nonzero(mask).squeeze(1)  # segment-major, t-minor valid frames
    n = int(idx.numel())
    if n == 0:
        raise ValueError("empty minibatch")
    tlogp = None
    if algo != 0:
        # target log-probs under the current parameters (learner.cpp:80-84)
        tl = torch.zeros(S * T, dtype=F64, device=dev)
        for lo in range(0, n, chunk):
            sel = idx[lo:lo + chunk]
            z, _, _ = net.forward(p, obs[sel])
            lp = torch.log_softmax(z, 1)
            tl[sel] = lp.gather(1, act[sel, None]).squeeze(1)
        tlogp = tl.view(S, T)
    adv, tgt = returns(algo, hp, r, v, dn, boot, valid, blogp, tlogp)
    a_all = adv.reshape(-1)[idx]
    if hp.get("adv_norm", True) and n >= 2:  # EffectiveAdvantages (rlmath.cpp:18-34)
        mean = a_all.mean()
        sd = torch.clamp(torch.sqrt(((a_all - mean) ** 2).mean()), min=1e-8)
        a_eff = (a_all - mean) / sd
    else:
        a_eff = a_all
    y_all = tgt.reshape(-1)[idx]
    bl_all = blogp.reshape(-1)[idx]
    inv_n = 1.0 / n
    eps, vf, ent = hp["clip_eps"], hp["vf_coef"], hp["ent_coef"]
    grad = torch.zeros(net.P, dtype=F64, device=dev)
    st = dict(loss=0.0, clip_fraction=0.0, mean_ratio=0.0, entropy=0.0, value_loss=0.0)
    clip = 0.0
    for lo in range(0, n, chunk):
        sel = idx[lo:lo + chunk]
        x = obs[sel]
        a = act[sel]
        A = a_eff[lo:lo + chunk]
        y = y_all[lo:lo + chunk]
        bl = bl_all[lo:lo + chunk]
        z, val, acts = net.forward(p, x)
        zm = z - z.max(1, keepdim=True).values
        e = torch.exp(zm)
        pr = e / e.sum(1, keepdim=True)          # Softmax (policy.cpp:45-55)
        lpr = torch.where(pr > 0, torch.log(pr), torch.zeros_like(pr))
        H = -(pr * lpr).sum(1)                     # Entropy (rlmath.cpp:36-41)
        logp = torch.log(pr.gather(1, a[:, None]).squeeze(1))
        verr = val - y
        onehot = torch.nn.functional.one_hot(a, net.a).to(F64)
        ratio = torch.exp(logp - bl)
        if algo == 1:  # PgLossAndGrad (rlmath.cpp:196-220)
            st["loss"] += float((inv_n * (-A * logp + vf * verr * verr - ent * H)).sum())
            dz = (-A[:, None] * (onehot - pr) + ent * pr * (lpr + H[:, None])) * inv_n
        else:          # PpoLossAndGrad (rlmath.cpp:129-182)
            t1 = ratio * A
            t2 = torch.clamp(ratio, 1.0 - eps, 1.0 + eps) * A
            surr = torch.minimum(t1, t2)
            st["loss"] += float((inv_n * (-surr + vf * verr * verr - ent * H)).sum())
            clip += float((t2 < t1).sum())
            through = (t1 <= t2).to(F64)
            dz = (through * -A * ratio)[:, None] * (onehot - pr) * inv_n
            dz = dz + ent * pr * (lpr + H[:, None]) * inv_n
        st["mean_ratio"] += float((inv_n * ratio).sum())
        st["entropy"] += float((inv_n * H).sum())
        st["value_loss"] += float((inv_n * verr * verr).sum())
        dv = 2.0 * vf * verr * inv_n
        grad += net.backward(p, x, acts, dz, dv)
        del acts, z
    st["clip_fraction"] = clip * inv_n if algo != 1 else 0.0
    st["n_samples"] = n
    return st, grad, adv, tgt, tlogp


def learner_step(net: Net, p, hp, algo, shards, dev):
    """Rank-ordered shard mean (learner.cpp:138-149): (stats list, avg grad,
    (adv, target, target logp) of the last shard)."""
    avg = torch.zeros(net.P, dtype=F64, device=dev)
    stats = []
    ret = None
    for b in shards:
        st, g, adv, tgt, tl = shard_step(net, p, hp, algo, b, dev)
        if not np.isfinite(st["loss"]):
            raise RuntimeError("non-finite loss")
        avg += g
        stats.append(st)
        ret = (adv, tgt, tl)
    avg *= 1.0 / len(shards)
    return stats, avg, ret


def sgd(p, g, lr):
    return p - lr * g


def adam(p, g, m, v, step, lr, b1=0.9, b2=0.999, eps=1e-8):
    """torch.optim.Adam semantics (orc_adam_step)."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    bc1 = 1 - b1 ** step
    bc2 = 1 - b2 ** step
    p = p - (lr / bc1) * m / (torch.sqrt(v) / np.sqrt(bc2) + eps)
    return p, m, v
