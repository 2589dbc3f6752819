// The MLP policy family (PolicyFamily::kMlp, wire tag 2) on the host, in fp64: what the
// reference's policy.cpp delegates to for kMlp once the family is registered at its
// extension seam (proj/docs/extending.md:23-37; integration/patches/mlp_family.py).
// Actors evaluate frozen MLP opponents with it (actor_loop.cpp:81-84), the reference's
// rlmath losses back-propagate through it, and it is the fp64 reference the B200
// learner / InfServer are checked against in integration/tests/dropin_test.cpp.
//
// Flat layout: [W_1 (h_1 x d), b_1, ..., W_L (h_L x h_{L-1}), b_L |
// W_pi (A x h_L), b_pi | w_v (h_L), b_v], W row-major [out x in]; h_l = tanh(W_l h_{l-1}
// + b_l), logits = W_pi h_L + b_pi, value = w_v . h_L + b_v.
#pragma once

#include <cstddef>
#include <span>

#include "tleague/policy/policy.hpp"
#include "tleague/types.hpp"

namespace tleague::policy::mlp {

// Parameter count of the layout above; throws std::invalid_argument on an empty trunk,
// a zero width or more than 8 trunk layers.
std::size_t ParamCount(const PolicyShape& shape);

ActionDistribution Distribution(const ParamBlob& params, std::span<const double> obs);
double ValueEstimate(const ParamBlob& params, std::span<const double> obs);

// grad += d(loss)/d(params) given d(loss)/d(logits) and d(loss)/d(value) for one sample
// (the forward is recomputed; the trunk is back-propagated through tanh).
void AccumulateGrad(const ParamBlob& params, std::span<const double> obs,
                    std::span<const double> dlogits, double dvalue, std::span<double> grad);

}  // namespace tleague::policy::mlp
