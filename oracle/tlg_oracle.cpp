// TEST INFRASTRUCTURE ONLY -- fp64 CPU oracle (checker) for the B200 learner path.
// See tlg_oracle.h for what is pinned against what.  Every function cites the
// reference routine it restates (paths relative to /root/reference/proj).
#include "tlg_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

template <typename F>
int Guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// Fixed-work parallel loop over [0, n) on std::thread (no OpenMP in this image).
template <typename F>
void ParallelFor(size_t n, F&& fn) {
  const size_t hw = std::max<unsigned>(1, std::thread::hardware_concurrency());
  const size_t nt = std::min(n, hw);
  if (nt <= 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> th;
  for (size_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t i = t; i < n; i += nt) fn(i);
    });
  for (auto& x : th) x.join();
}

// ---------------------------------------------------------------------------
// Flat parameter layout.
//  tabular (policy.cpp:78-80,96-105):  [T: obs_dim x A row-major | v: obs_dim]
//  linear  (policy.cpp:82-88,96-104):  [W: A x obs_dim row-major | v: obs_dim]
//  mlp (appended family):
//     [W_1 (h1 x d), b_1, ..., W_L (hL x h_{L-1}), b_L | W_pi (A x hL), b_pi | w_v (hL), b_v]
struct Layout {
  uint32_t family, d, a, L;
  std::vector<uint32_t> dims;      // dims[0] = d, dims[l] = hidden[l-1]
  std::vector<size_t> w_off, b_off;  // per trunk layer
  size_t wpi, bpi, wv, bv, total;
};

Layout MakeLayout(const orc_shape* s) {
  if (s->obs_dim == 0 || s->n_actions == 0)  // policy.cpp:11-14
    throw std::invalid_argument("policy shape dimensions must be positive");
  Layout lay;
  lay.family = s->family;
  lay.d = s->obs_dim;
  lay.a = s->n_actions;
  lay.L = s->family == 2 ? s->n_hidden : 0;
  if (s->family > 2) throw std::invalid_argument("unknown policy family");
  if (lay.L > 8) throw std::invalid_argument("at most 8 hidden layers");
  lay.dims.push_back(lay.d);
  size_t off = 0;
  for (uint32_t l = 0; l < lay.L; ++l) {
    if (s->hidden[l] == 0) throw std::invalid_argument("hidden width must be positive");
    lay.dims.push_back(s->hidden[l]);
    lay.w_off.push_back(off);
    off += size_t(s->hidden[l]) * lay.dims[l];
    lay.b_off.push_back(off);
    off += s->hidden[l];
  }
  const size_t hl = lay.dims.back();
  if (s->family == 2) {
    lay.wpi = off; off += size_t(lay.a) * hl;
    lay.bpi = off; off += lay.a;
    lay.wv = off;  off += hl;
    lay.bv = off;  off += 1;
  } else {
    // ParamCount: obs_dim * n_actions + obs_dim (policy.cpp:23-27)
    lay.wpi = 0;
    lay.wv = size_t(lay.d) * lay.a;
    lay.bpi = lay.bv = size_t(-1);
    off = lay.wv + lay.d;
  }
  lay.total = off;
  return lay;
}

// OneHotIndex (policy.cpp:57-71)
size_t OneHotIndex(const double* obs, size_t n) {
  size_t idx = n;
  for (size_t i = 0; i < n; ++i) {
    if (obs[i] == 1.0) {
      if (idx != n) throw std::invalid_argument("tabular observation must be one-hot");
      idx = i;
    } else if (obs[i] != 0.0) {
      throw std::invalid_argument("tabular observation must be one-hot");
    }
  }
  if (idx == n) throw std::invalid_argument("tabular observation must be one-hot");
  return idx;
}

// Softmax (policy.cpp:45-55): max-shifted, divide by the sum.
void Softmax(const double* z, size_t a, double* p) {
  double mx = *std::max_element(z, z + a);
  double sum = 0.0;
  for (size_t i = 0; i < a; ++i) {
    p[i] = std::exp(z[i] - mx);
    sum += p[i];
  }
  for (size_t i = 0; i < a; ++i) p[i] /= sum;
}

// Entropy (rlmath.cpp:36-41)
double Entropy(const double* p, size_t a) {
  double h = 0.0;
  for (size_t i = 0; i < a; ++i)
    if (p[i] > 0.0) h -= p[i] * std::log(p[i]);
  return h;
}

// Per-sample forward.  acts holds the trunk activations h_1..h_L (mlp) for
// the backward pass.  Distribution (policy.cpp:73-92) + ValueEstimate (:94-105).
struct Fwd {
  std::vector<double> z, p, acts;
  double v = 0.0;
  size_t row = 0;  // tabular
};

void Forward(const Layout& lay, const double* w, const double* obs, Fwd& f) {
  const size_t a = lay.a;
  f.z.assign(a, 0.0);
  f.p.assign(a, 0.0);
  if (lay.family == 0) {
    f.row = OneHotIndex(obs, lay.d);
    for (size_t k = 0; k < a; ++k) f.z[k] = w[f.row * a + k];
    f.v = w[lay.wv + f.row];
  } else if (lay.family == 1) {
    for (size_t k = 0; k < a; ++k) {
      double z = 0.0;
      for (size_t j = 0; j < lay.d; ++j) z += w[k * lay.d + j] * obs[j];
      f.z[k] = z;
    }
    double v = 0.0;
    for (size_t j = 0; j < lay.d; ++j) v += w[lay.wv + j] * obs[j];
    f.v = v;
  } else {
    size_t tot = 0;
    for (uint32_t l = 1; l <= lay.L; ++l) tot += lay.dims[l];
    f.acts.assign(tot, 0.0);
    const double* in = obs;
    size_t aoff = 0;
    for (uint32_t l = 0; l < lay.L; ++l) {
      const size_t ni = lay.dims[l], no = lay.dims[l + 1];
      const double* W = w + lay.w_off[l];
      const double* b = w + lay.b_off[l];
      double* out = f.acts.data() + aoff;
      for (size_t o = 0; o < no; ++o) {
        double s = 0.0;
        const double* row = W + o * ni;
        for (size_t i = 0; i < ni; ++i) s += row[i] * in[i];
        out[o] = std::tanh(s + b[o]);
      }
      in = out;
      aoff += no;
    }
    const size_t hl = lay.dims[lay.L];
    for (size_t k = 0; k < a; ++k) {
      double z = 0.0;
      const double* row = w + lay.wpi + k * hl;
      for (size_t j = 0; j < hl; ++j) z += row[j] * in[j];
      f.z[k] = z + w[lay.bpi + k];
    }
    double v = 0.0;
    for (size_t j = 0; j < hl; ++j) v += w[lay.wv + j] * in[j];
    f.v = v + w[lay.bv];
  }
  Softmax(f.z.data(), a, f.p.data());
}

// Chain rule into the flat gradient.  AccumulateGrad (policy.cpp:122-141) for
// tabular/linear; the mlp family back-propagates through the tanh trunk.
void Backward(const Layout& lay, const double* w, const double* obs, const Fwd& f,
              const double* dz, double dv, double* g, std::vector<double>& scratch) {
  const size_t a = lay.a;
  if (lay.family == 0) {
    for (size_t k = 0; k < a; ++k) g[f.row * a + k] += dz[k];
    g[lay.wv + f.row] += dv;
    return;
  }
  if (lay.family == 1) {
    for (size_t k = 0; k < a; ++k)
      for (size_t j = 0; j < lay.d; ++j) g[k * lay.d + j] += dz[k] * obs[j];
    for (size_t j = 0; j < lay.d; ++j) g[lay.wv + j] += dv * obs[j];
    return;
  }
  const size_t hl = lay.dims[lay.L];
  size_t aoff = f.acts.size() - hl;
  const double* hL = f.acts.data() + aoff;
  // heads
  scratch.assign(hl, 0.0);
  for (size_t k = 0; k < a; ++k) {
    double* gw = g + lay.wpi + k * hl;
    const double* W = w + lay.wpi + k * hl;
    for (size_t j = 0; j < hl; ++j) {
      gw[j] += dz[k] * hL[j];
      scratch[j] += dz[k] * W[j];
    }
    g[lay.bpi + k] += dz[k];
  }
  for (size_t j = 0; j < hl; ++j) {
    g[lay.wv + j] += dv * hL[j];
    scratch[j] += dv * w[lay.wv + j];
  }
  g[lay.bv] += dv;
  // trunk, l = L..1: dpre = dh * (1 - h^2); dW += dpre (x) h_{l-1}; dh_{l-1} = W^T dpre
  std::vector<double> dpre;
  for (int l = int(lay.L) - 1; l >= 0; --l) {
    const size_t ni = lay.dims[l], no = lay.dims[l + 1];
    const double* h = f.acts.data() + aoff;
    const double* hin;
    size_t ain = 0;
    if (l == 0) {
      hin = obs;
    } else {
      ain = aoff - ni;
      hin = f.acts.data() + ain;
    }
    dpre.assign(no, 0.0);
    for (size_t o = 0; o < no; ++o) dpre[o] = scratch[o] * (1.0 - h[o] * h[o]);
    double* gW = g + lay.w_off[l];
    double* gb = g + lay.b_off[l];
    const double* W = w + lay.w_off[l];
    for (size_t o = 0; o < no; ++o) {
      const double d = dpre[o];
      double* row = gW + o * ni;
      for (size_t i = 0; i < ni; ++i) row[i] += d * hin[i];
      gb[o] += d;
    }
    if (l > 0) {
      scratch.assign(ni, 0.0);
      for (size_t o = 0; o < no; ++o) {
        const double d = dpre[o];
        const double* row = W + o * ni;
        for (size_t i = 0; i < ni; ++i) scratch[i] += d * row[i];
      }
      aoff = ain;
    }
  }
}

// EffectiveAdvantages (rlmath.cpp:18-34): per-minibatch normalisation.
std::vector<double> EffectiveAdvantages(const double* adv_in, size_t n, bool normalize) {
  std::vector<double> adv(adv_in, adv_in + n);
  for (double a : adv)
    if (!std::isfinite(a)) throw std::invalid_argument("non-finite advantage");
  if (!normalize || n < 2) return adv;
  double mean = 0.0;
  for (double a : adv) mean += a;
  mean /= double(n);
  double var = 0.0;
  for (double a : adv) var += (a - mean) * (a - mean);
  var /= double(n);
  const double sd = std::max(std::sqrt(var), 1e-8);
  for (double& a : adv) a = (a - mean) / sd;
  return adv;
}

// Samples are processed in fixed chunks whose partial gradients are summed in
// chunk order, so the result does not depend on the OpenMP thread count.
size_t NumChunks(size_t n) { return std::min<size_t>(16, std::max<size_t>(1, n / 64)); }

enum LossKind { kPpo, kPg };

void LossAndGrad(LossKind kind, const orc_shape* s, const double* params, const double* teacher,
                 size_t n, const double* obs, const uint32_t* action, const double* blogp,
                 const double* adv_in, const double* vtarget, const orc_hyper* hp, double* grad,
                 orc_stats* stats) {
  if (n == 0) throw std::invalid_argument("empty minibatch");  // rlmath.cpp:118,189
  if (kind == kPpo && hp->kl_teacher_coef > 0.0 && teacher == nullptr)
    throw std::invalid_argument("teacher params required when kl_teacher_coef > 0");
  const Layout lay = MakeLayout(s);
  const double inv_n = 1.0 / double(n);
  const std::vector<double> adv = EffectiveAdvantages(adv_in, n, hp->adv_norm != 0);
  const size_t P = lay.total;
  const size_t nc = NumChunks(n);
  std::vector<double> part(nc * P, 0.0);
  struct Acc { double loss = 0, clip = 0, ratio = 0, ent = 0, vl = 0; };
  std::vector<Acc> acc(nc);
  std::vector<std::string> errs(nc);
  const size_t a = lay.a;
  ParallelFor(nc, [&](size_t c) {
    try {
      const size_t lo = n * c / nc, hi = n * (c + 1) / nc;
      Fwd f, tf;
      std::vector<double> dz(a), tlogp(a), scratch;
      double* g = part.data() + c * P;
      Acc& A = acc[c];
      for (size_t i = lo; i < hi; ++i) {
        const double* o = obs + i * lay.d;
        Forward(lay, params, o, f);
        if (action[i] >= a) throw std::invalid_argument("action out of range");
        const double logp = std::log(f.p[action[i]]);
        const double verr = f.v - vtarget[i];
        const double h = Entropy(f.p.data(), a);
        std::fill(dz.begin(), dz.end(), 0.0);
        if (kind == kPpo) {
          // PpoLossAndGrad per-sample body (rlmath.cpp:129-182)
          const double ratio = std::exp(logp - blogp[i]);
          const double clipped = std::clamp(ratio, 1.0 - hp->clip_eps, 1.0 + hp->clip_eps);
          const double t1 = ratio * adv[i];
          const double t2 = clipped * adv[i];
          const double surr = std::min(t1, t2);
          double kl = 0.0;
          if (teacher) {
            Forward(lay, teacher, o, tf);
            for (size_t k = 0; k < a; ++k) {
              tlogp[k] = std::log(std::max(tf.p[k], 1e-300));
              if (f.p[k] > 0.0) kl += f.p[k] * (std::log(f.p[k]) - tlogp[k]);
            }
          }
          A.loss += inv_n * (-surr + hp->vf_coef * verr * verr - hp->ent_coef * h +
                             hp->kl_teacher_coef * kl);
          A.ratio += inv_n * ratio;
          A.ent += inv_n * h;
          A.vl += inv_n * verr * verr;
          if (t2 < t1) A.clip += 1.0;
          if (t1 <= t2) {
            for (size_t k = 0; k < a; ++k) {
              const double ind = k == action[i] ? 1.0 : 0.0;
              dz[k] += -adv[i] * ratio * (ind - f.p[k]) * inv_n;
            }
          }
          for (size_t k = 0; k < a; ++k) {
            const double p = f.p[k];
            const double lpk = p > 0.0 ? std::log(p) : 0.0;
            dz[k] += hp->ent_coef * p * (lpk + h) * inv_n;
            if (teacher) dz[k] += hp->kl_teacher_coef * p * (lpk - tlogp[k] - kl) * inv_n;
          }
        } else {
          // PgLossAndGrad per-sample body (rlmath.cpp:196-220)
          A.loss += inv_n * (-adv[i] * logp + hp->vf_coef * verr * verr - hp->ent_coef * h);
          A.ent += inv_n * h;
          A.vl += inv_n * verr * verr;
          A.ratio += inv_n * std::exp(logp - blogp[i]);
          for (size_t k = 0; k < a; ++k) {
            const double ind = k == action[i] ? 1.0 : 0.0;
            const double p = f.p[k];
            const double lpk = p > 0.0 ? std::log(p) : 0.0;
            dz[k] += (-adv[i] * (ind - p) + hp->ent_coef * p * (lpk + h)) * inv_n;
          }
        }
        const double dv = 2.0 * hp->vf_coef * verr * inv_n;
        Backward(lay, params, o, f, dz.data(), dv, g, scratch);
      }
    } catch (const std::exception& e) {
      errs[c] = e.what();
    }
  });
  for (const auto& e : errs)
    if (!e.empty()) throw std::invalid_argument(e);
  std::memset(grad, 0, P * sizeof(double));
  orc_stats st{};
  double clip = 0.0;
  for (size_t c = 0; c < nc; ++c) {
    const double* g = part.data() + c * P;
    for (size_t p = 0; p < P; ++p) grad[p] += g[p];
    st.loss += acc[c].loss;
    clip += acc[c].clip;
    st.mean_ratio += acc[c].ratio;
    st.entropy += acc[c].ent;
    st.value_loss += acc[c].vl;
  }
  st.clip_fraction = kind == kPpo ? clip * inv_n : 0.0;
  st.n_samples = n;
  if (stats) *stats = st;
}

// GaeAdvantages (rlmath.cpp:62-78)
void Gae(const double* r, const double* v, const uint8_t* done, size_t n, double boot,
         double gamma, double lam, double* adv) {
  if (n == 0) throw std::invalid_argument("segment length must be >= 1");
  double next_value = boot, next_adv = 0.0;
  for (size_t i = n; i-- > 0;) {
    const double nt = done[i] ? 0.0 : 1.0;
    const double delta = r[i] + gamma * nt * next_value - v[i];
    adv[i] = delta + gamma * lam * nt * next_adv;
    next_value = v[i];
    next_adv = adv[i];
  }
}

// LambdaReturn (rlmath.cpp:45-60)
void LambdaRet(const double* r, const double* v, const uint8_t* done, size_t n, double boot,
               double gamma, double lam, double* ret) {
  if (n == 0) throw std::invalid_argument("segment length must be >= 1");
  double next_value = boot, next_ret = boot;
  for (size_t i = n; i-- > 0;) {
    const double nt = done[i] ? 0.0 : 1.0;
    ret[i] = r[i] + gamma * nt * ((1.0 - lam) * next_value + lam * next_ret);
    next_value = v[i];
    next_ret = ret[i];
  }
}

// VtraceTargets (rlmath.cpp:80-114)
void Vtrace(const double* bl, const double* tl, const double* r, const double* v,
            const uint8_t* done, size_t n, double boot, double gamma, double rho_bar,
            double c_bar, double* vs, double* pg) {
  if (n == 0) throw std::invalid_argument("segment length must be >= 1");
  std::vector<double> rho(n), c(n);
  for (size_t i = 0; i < n; ++i) {
    if (!std::isfinite(bl[i]) || !std::isfinite(tl[i]))
      throw std::invalid_argument("non-finite log probability");
    const double w = std::exp(tl[i] - bl[i]);
    rho[i] = std::min(rho_bar, w);
    c[i] = std::min(c_bar, w);
  }
  double next_vs = boot, next_value = boot;
  for (size_t i = n; i-- > 0;) {
    const double nt = done[i] ? 0.0 : 1.0;
    const double delta = rho[i] * (r[i] + gamma * nt * next_value - v[i]);
    vs[i] = v[i] + delta + gamma * nt * c[i] * (next_vs - next_value);
    next_vs = vs[i];
    next_value = v[i];
  }
  for (size_t i = 0; i < n; ++i) {
    const double nt = done[i] ? 0.0 : 1.0;
    const double vs_next = (i + 1 < n) ? vs[i + 1] : boot;
    pg[i] = rho[i] * (r[i] + gamma * nt * vs_next - v[i]);
  }
}

// BuildMinibatch (learner.cpp:56-102): segment-major, t-minor, padding skipped.
struct Batch {
  std::vector<double> obs, blogp, adv, tgt;
  std::vector<uint32_t> action;
  std::vector<size_t> frame;  // source frame index s*T + t
  size_t n = 0;
};

Batch BuildBatch(const orc_shape* s, const double* params, const orc_hyper* hp, uint32_t algo,
                 const orc_segments* sg) {
  if (sg->obs_dim != s->obs_dim) throw std::invalid_argument("observation size does not match policy shape");
  const Layout lay = MakeLayout(s);
  Batch b;
  const size_t T = sg->unroll_len, d = sg->obs_dim;
  Fwd f;
  std::vector<double> adv(T), tgt(T), tl(T);
  for (size_t si = 0; si < sg->n_segments; ++si) {
    const size_t n = sg->valid_steps[si];
    if (n == 0) continue;
    if (n > T) throw std::invalid_argument("valid_steps exceeds unroll_len");
    const size_t f0 = si * T;
    const double* r = sg->reward + f0;
    const double* v = sg->value_est + f0;
    const double* bl = sg->behavior_logp + f0;
    const uint8_t* dn = sg->done + f0;
    if (algo == 0) {
      Gae(r, v, dn, n, sg->bootstrap[si], hp->gamma, hp->lam, adv.data());
      LambdaRet(r, v, dn, n, sg->bootstrap[si], hp->gamma, hp->lam, tgt.data());
    } else {
      for (size_t t = 0; t < n; ++t) {
        Forward(lay, params, sg->obs + (f0 + t) * d, f);
        const uint32_t act = sg->action[f0 + t];
        if (act >= lay.a) throw std::invalid_argument("action out of range");
        tl[t] = std::log(f.p[act]);
      }
      Vtrace(bl, tl.data(), r, v, dn, n, sg->bootstrap[si], hp->gamma, hp->rho_bar, hp->c_bar,
             tgt.data(), adv.data());
    }
    for (size_t t = 0; t < n; ++t) {
      b.obs.insert(b.obs.end(), sg->obs + (f0 + t) * d, sg->obs + (f0 + t + 1) * d);
      b.action.push_back(sg->action[f0 + t]);
      b.blogp.push_back(bl[t]);
      b.adv.push_back(adv[t]);
      b.tgt.push_back(tgt[t]);
      b.frame.push_back(f0 + t);
    }
  }
  b.n = b.action.size();
  return b;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

size_t orc_param_count(const orc_shape* s) {
  size_t n = 0;
  if (Guard([&] { n = MakeLayout(s).total; }) != 0) return 0;
  return n;
}

// InitParams (policy.cpp:29-43): i.i.d. U[-s, s] from mt19937_64(seed) in flat order.
int orc_init_params(const orc_shape* s, double scale, uint64_t seed, double* out) {
  return Guard([&] {
    if (scale < 0.0) throw std::invalid_argument("init_scale must be >= 0");
    const size_t n = MakeLayout(s).total;
    std::fill(out, out + n, 0.0);
    if (scale > 0.0) {
      std::mt19937_64 rng(seed);
      std::uniform_real_distribution<double> u(-scale, scale);
      for (size_t i = 0; i < n; ++i) out[i] = u(rng);
    }
  });
}

int orc_forward(const orc_shape* s, const double* params, const double* obs, size_t n,
                double* logits, double* probs, double* value) {
  return Guard([&] {
    const Layout lay = MakeLayout(s);
    const size_t nc = std::min<size_t>(64, std::max<size_t>(1, n));
    std::vector<std::string> errs(nc);
    ParallelFor(nc, [&](size_t c) {
      Fwd f;
      try {
        for (size_t i = n * c / nc; i < n * (c + 1) / nc; ++i) {
          Forward(lay, params, obs + i * lay.d, f);
          for (size_t k = 0; k < lay.a; ++k) {
            if (logits) logits[i * lay.a + k] = f.z[k];
            if (probs) probs[i * lay.a + k] = f.p[k];
          }
          if (value) value[i] = f.v;
        }
      } catch (const std::exception& e) {
        errs[c] = e.what();
      }
    });
    for (const auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
  });
}

int orc_gae(const double* r, const double* v, const uint8_t* done, size_t n, double boot,
            double gamma, double lam, double* adv) {
  return Guard([&] { Gae(r, v, done, n, boot, gamma, lam, adv); });
}

int orc_lambda_return(const double* r, const double* v, const uint8_t* done, size_t n,
                      double boot, double gamma, double lam, double* ret) {
  return Guard([&] { LambdaRet(r, v, done, n, boot, gamma, lam, ret); });
}

int orc_vtrace(const double* bl, const double* tl, const double* r, const double* v,
               const uint8_t* done, size_t n, double boot, double gamma, double rho_bar,
               double c_bar, double* vs, double* pg_adv) {
  return Guard([&] { Vtrace(bl, tl, r, v, done, n, boot, gamma, rho_bar, c_bar, vs, pg_adv); });
}

int orc_ppo_loss_grad(const orc_shape* s, const double* params, const double* teacher,
                      size_t n, const double* obs, const uint32_t* action, const double* blogp,
                      const double* adv, const double* vtarget, const orc_hyper* hp,
                      double* grad, orc_stats* stats) {
  return Guard([&] {
    LossAndGrad(kPpo, s, params, teacher, n, obs, action, blogp, adv, vtarget, hp, grad, stats);
  });
}

int orc_pg_loss_grad(const orc_shape* s, const double* params, size_t n, const double* obs,
                     const uint32_t* action, const double* blogp, const double* adv,
                     const double* vtarget, const orc_hyper* hp, double* grad,
                     orc_stats* stats) {
  return Guard([&] {
    LossAndGrad(kPg, s, params, nullptr, n, obs, action, blogp, adv, vtarget, hp, grad, stats);
  });
}

int orc_shard_loss_grad(const orc_shape* s, const double* params, const orc_hyper* hp,
                        uint32_t algo, const orc_segments* segs, double* grad,
                        orc_stats* stats) {
  return Guard([&] {
    if (algo > 2) throw std::invalid_argument("unknown algo");
    Batch b = BuildBatch(s, params, hp, algo, segs);
    // Learner::TrainStep loss choice (learner.cpp:126-128); algo 2 = PPO surrogate
    // over V-trace targets.
    LossAndGrad(algo == 1 ? kPg : kPpo, s, params, nullptr, b.n, b.obs.data(), b.action.data(),
                b.blogp.data(), b.adv.data(), b.tgt.data(), hp, grad, stats);
  });
}

int orc_shard_returns(const orc_shape* s, const double* params, const orc_hyper* hp,
                      uint32_t algo, const orc_segments* segs, double* adv, double* target) {
  return Guard([&] {
    if (algo > 2) throw std::invalid_argument("unknown algo");
    Batch b = BuildBatch(s, params, hp, algo, segs);
    const size_t F = size_t(segs->n_segments) * segs->unroll_len;
    std::fill(adv, adv + F, 0.0);
    std::fill(target, target + F, 0.0);
    for (size_t i = 0; i < b.n; ++i) {
      adv[b.frame[i]] = b.adv[i];
      target[b.frame[i]] = b.tgt[i];
    }
  });
}

// SgdStep (rlmath.cpp:224-232)
int orc_sgd_step(const double* params, const double* grad, size_t n, double lr, double* out) {
  return Guard([&] {
    for (size_t i = 0; i < n; ++i) out[i] = params[i] - lr * grad[i];
  });
}

// torch.optim.Adam single-tensor semantics (no amsgrad, weight_decay 0):
//   m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2
//   p -= (lr / (1 - b1^t)) * m / (sqrt(v) / sqrt(1 - b2^t) + eps)
int orc_adam_step(double* params, const double* grad, double* m, double* v, size_t n,
                  uint64_t step, double lr, double beta1, double beta2, double eps) {
  return Guard([&] {
    if (step == 0) throw std::invalid_argument("adam step is 1-based");
    const double bc1 = 1.0 - std::pow(beta1, double(step));
    const double bc2 = 1.0 - std::pow(beta2, double(step));
    const double step_size = lr / bc1;
    const double bc2_sqrt = std::sqrt(bc2);
    for (size_t i = 0; i < n; ++i) {
      m[i] = beta1 * m[i] + (1.0 - beta1) * grad[i];
      v[i] = beta2 * v[i] + (1.0 - beta2) * grad[i] * grad[i];
      const double denom = std::sqrt(v[i]) / bc2_sqrt + eps;
      params[i] -= step_size * m[i] / denom;
    }
  });
}

}  // extern "C"
