// PolicyFamily::kMlp on the host (see tleague/policy/policy_mlp.hpp).
#include "tleague/policy/policy_mlp.hpp"

#include <cmath>
#include <stdexcept>
#include <vector>

namespace tleague::policy::mlp {

namespace {

struct Layout {
  std::vector<std::size_t> dims, w, b;  // dims[0] = obs_dim; per layer W and b offsets
  std::size_t wpi = 0, bpi = 0, wv = 0, bv = 0, total = 0;
};

Layout Plan(const PolicyShape& s) {
  if (s.hidden.empty()) throw std::invalid_argument("mlp policy needs at least one hidden layer");
  if (s.hidden.size() > 8) throw std::invalid_argument("mlp policy: at most 8 hidden layers");
  Layout L;
  L.dims.push_back(s.obs_dim);
  std::size_t off = 0;
  for (std::uint32_t h : s.hidden) {
    if (h == 0) throw std::invalid_argument("mlp hidden width must be positive");
    L.w.push_back(off);
    off += std::size_t(h) * L.dims.back();
    L.b.push_back(off);
    off += h;
    L.dims.push_back(h);
  }
  const std::size_t top = L.dims.back();
  L.wpi = off;
  off += std::size_t(s.n_actions) * top;
  L.bpi = off;
  off += s.n_actions;
  L.wv = off;
  off += top;
  L.bv = off;
  L.total = off + 1;
  return L;
}

// Trunk activations h_1..h_L, concatenated.
std::vector<double> Trunk(const Layout& L, const double* p, std::span<const double> obs) {
  std::size_t n = 0;
  for (std::size_t l = 1; l < L.dims.size(); ++l) n += L.dims[l];
  std::vector<double> acts(n);
  const double* x = obs.data();
  double* y = acts.data();
  for (std::size_t l = 0; l + 1 < L.dims.size(); ++l) {
    const std::size_t in = L.dims[l], out = L.dims[l + 1];
    for (std::size_t o = 0; o < out; ++o) {
      const double* row = p + L.w[l] + o * in;
      double z = p[L.b[l] + o];
      for (std::size_t i = 0; i < in; ++i) z += row[i] * x[i];
      y[o] = std::tanh(z);
    }
    x = y;
    y += out;
  }
  return acts;
}

void Check(const ParamBlob& params, const Layout& L) {
  if (params.values.size() != L.total)
    throw std::invalid_argument("mlp parameter count does not match its shape");
}

}  // namespace

std::size_t ParamCount(const PolicyShape& shape) { return Plan(shape).total; }

ActionDistribution Distribution(const ParamBlob& params, std::span<const double> obs) {
  const Layout L = Plan(params.shape);
  Check(params, L);
  const double* p = params.values.data();
  const std::vector<double> acts = Trunk(L, p, obs);
  const std::size_t top = L.dims.back(), A = params.shape.n_actions;
  const double* h = acts.data() + acts.size() - top;
  ActionDistribution dist;
  dist.logits.assign(A, 0.0);
  for (std::size_t k = 0; k < A; ++k) {
    double z = p[L.bpi + k];
    for (std::size_t j = 0; j < top; ++j) z += p[L.wpi + k * top + j] * h[j];
    dist.logits[k] = z;
  }
  dist.probs = Softmax(dist.logits);
  return dist;
}

double ValueEstimate(const ParamBlob& params, std::span<const double> obs) {
  const Layout L = Plan(params.shape);
  Check(params, L);
  const double* p = params.values.data();
  const std::vector<double> acts = Trunk(L, p, obs);
  const std::size_t top = L.dims.back();
  const double* h = acts.data() + acts.size() - top;
  double v = p[L.bv];
  for (std::size_t j = 0; j < top; ++j) v += p[L.wv + j] * h[j];
  return v;
}

void AccumulateGrad(const ParamBlob& params, std::span<const double> obs,
                    std::span<const double> dlogits, double dvalue, std::span<double> grad) {
  const Layout L = Plan(params.shape);
  Check(params, L);
  const double* p = params.values.data();
  const std::vector<double> acts = Trunk(L, p, obs);
  const std::size_t A = params.shape.n_actions, depth = L.dims.size() - 1;
  std::vector<std::size_t> aoff(depth);  // offset of h_{l+1} in acts
  for (std::size_t l = 0, o = 0; l < depth; o += L.dims[l + 1], ++l) aoff[l] = o;
  // heads: logits = W_pi h_L + b_pi, value = w_v . h_L + b_v
  const std::size_t top = L.dims.back();
  const double* hL = acts.data() + aoff[depth - 1];
  std::vector<double> dh(top, 0.0);
  for (std::size_t k = 0; k < A; ++k) {
    const double g = dlogits[k];
    grad[L.bpi + k] += g;
    for (std::size_t j = 0; j < top; ++j) {
      grad[L.wpi + k * top + j] += g * hL[j];
      dh[j] += g * p[L.wpi + k * top + j];
    }
  }
  grad[L.bv] += dvalue;
  for (std::size_t j = 0; j < top; ++j) {
    grad[L.wv + j] += dvalue * hL[j];
    dh[j] += dvalue * p[L.wv + j];
  }
  // trunk, top down: dz = dh (1 - h^2); dW += dz x h_in; db += dz; dh_in = W^T dz
  for (std::size_t l = depth; l-- > 0;) {
    const std::size_t in = L.dims[l], out = L.dims[l + 1];
    const double* h = acts.data() + aoff[l];
    const double* x = l == 0 ? obs.data() : acts.data() + aoff[l - 1];
    std::vector<double> dx(l > 0 ? in : 0, 0.0);
    for (std::size_t o = 0; o < out; ++o) {
      const double dz = dh[o] * (1.0 - h[o] * h[o]);
      grad[L.b[l] + o] += dz;
      double* gw = grad.data() + L.w[l] + o * in;
      const double* w = p + L.w[l] + o * in;
      for (std::size_t i = 0; i < in; ++i) gw[i] += dz * x[i];
      if (l > 0)
        for (std::size_t i = 0; i < in; ++i) dx[i] += dz * w[i];
    }
    dh.swap(dx);
  }
}

}  // namespace tleague::policy::mlp
