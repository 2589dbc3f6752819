#!/usr/bin/env python3
"""Registers the MLP policy family at the reference's extension seam
(proj/docs/extending.md:23-37), the way a maintainer would edit the reference tree:

  1. types.hpp   PolicyFamily::kMlp = 2 (appended) and PolicyShape::hidden (the tanh
                 trunk widths; empty for the reference's two families)
  2. policy.cpp  sizing / evaluation / chain rule of kMlp delegated to
                 integration/policy_mlp.cpp (tleague::policy::mlp); InitParams and
                 PolicyGradLogp are generic over ParamCount / AccumulateGrad already
  3. codec.cpp   wire tag 2 with the trunk widths as family-conditional fields after
                 n_actions (tags 0 and 1 encode exactly as before, so the reference's
                 golden frames stay valid)
  4. config.cpp  `family: mlp` and `hidden: w1,w2,...` group keys
  5. local_run.cpp  keeps the configured trunk widths when the env fixes the shape

rlmath.cpp needs no edit: PpoLossAndGrad / PgLossAndGrad reach the family only through
policy::Distribution / ValueEstimate / AccumulateGrad (rlmath.cpp:131-181,198-219).

The patched copies are build outputs written under oracle/_ref/dropin/patched/ (git-
ignored); nothing of the reference is committed here.  Each edit is anchored on an
exact line of the reference and fails loudly if the anchor is missing.

    python integration/patches/mlp_family.py <reference proj dir> <out dir>
"""
import os
import sys


def patch(src, dst, edits):
    with open(src) as f:
        text = f.read()
    for anchor, replacement in edits:
        n = text.count(anchor)
        if n != 1:
            raise SystemExit(f"{src}: anchor found {n} times: {anchor!r}")
        text = text.replace(anchor, replacement)
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    old = open(dst).read() if os.path.exists(dst) else None
    if old != text:  # keep the timestamp when nothing changed (make stays incremental)
        with open(dst, "w") as f:
            f.write(text)


def main(ref, out):
    patch(f"{ref}/include/tleague/types.hpp", f"{out}/include/tleague/types.hpp", [
        ("enum class PolicyFamily : std::uint8_t { kTabularSoftmax = 0, kLinearSoftmax = 1 };",
         "enum class PolicyFamily : std::uint8_t { kTabularSoftmax = 0, kLinearSoftmax = 1,"
         " kMlp = 2 };"),
        ("  std::uint32_t n_actions = 0;\n",
         "  std::uint32_t n_actions = 0;\n"
         "  // kMlp: widths of the tanh trunk layers (flat layout [W_1, b_1, ..., W_L, b_L |\n"
         "  // W_pi, b_pi | w_v, b_v], W row-major [out x in]); empty for the other families.\n"
         "  std::vector<std::uint32_t> hidden;\n"),
    ])
    mlp_hook = '#include "tleague/policy/policy_mlp.hpp"\n'
    patch(f"{ref}/src/policy/policy.cpp", f"{out}/src/policy/policy.cpp", [
        ('#include "tleague/policy/policy.hpp"\n',
         '#include "tleague/policy/policy.hpp"\n' + mlp_hook),
        ("  CheckShape(shape);\n  (void)family;",
         "  CheckShape(shape);\n  if (family == PolicyFamily::kMlp) return mlp::ParamCount(shape);\n"
         "  (void)family;"),
        ("  CheckObs(params, obs);\n  const std::uint32_t a = params.shape.n_actions;\n"
         "  ActionDistribution dist;",
         "  CheckObs(params, obs);\n"
         "  if (params.family == PolicyFamily::kMlp) return mlp::Distribution(params, obs);\n"
         "  const std::uint32_t a = params.shape.n_actions;\n  ActionDistribution dist;"),
        ("  CheckObs(params, obs);\n  const std::size_t value_off =",
         "  CheckObs(params, obs);\n"
         "  if (params.family == PolicyFamily::kMlp) return mlp::ValueEstimate(params, obs);\n"
         "  const std::size_t value_off ="),
        ("  if (grad.size() != params.values.size()) throw std::invalid_argument(\"grad size mismatch\");\n",
         "  if (grad.size() != params.values.size()) throw std::invalid_argument(\"grad size mismatch\");\n"
         "  if (params.family == PolicyFamily::kMlp) {\n"
         "    mlp::AccumulateGrad(params, obs, dlogits, dvalue, grad);\n"
         "    return;\n"
         "  }\n"),
    ])
    patch(f"{ref}/src/proto/codec.cpp", f"{out}/src/proto/codec.cpp", [
        ("  w.U32(b.shape.n_actions);\n  w.F64Vec(b.values);",
         "  w.U32(b.shape.n_actions);\n"
         "  if (b.family == PolicyFamily::kMlp) {  // wire tag 2: trunk widths\n"
         "    w.U32(static_cast<std::uint32_t>(b.shape.hidden.size()));\n"
         "    for (std::uint32_t h : b.shape.hidden) w.U32(h);\n"
         "  }\n"
         "  w.F64Vec(b.values);"),
        ("  if (fam > 1) throw DecodeError(\"unknown policy family\");",
         "  if (fam > 2) throw DecodeError(\"unknown policy family\");"),
        ("  b.shape.n_actions = r.U32();\n  b.values = r.F64Vec();",
         "  b.shape.n_actions = r.U32();\n"
         "  if (b.family == PolicyFamily::kMlp) {\n"
         "    const std::uint32_t n = r.U32();\n"
         "    if (n == 0 || n > 8) throw DecodeError(\"bad mlp trunk depth\");\n"
         "    b.shape.hidden.resize(n);\n"
         "    for (std::uint32_t& h : b.shape.hidden) h = r.U32();\n"
         "  }\n"
         "  b.values = r.F64Vec();"),
    ])
    # 4. run configs: `family: mlp` and `hidden: 256,256` in a [group] section
    patch(f"{ref}/src/run/config.cpp", f"{out}/src/run/config.cpp", [
        ("    else if (value == \"linear\") g.family = PolicyFamily::kLinearSoftmax;\n",
         "    else if (value == \"linear\") g.family = PolicyFamily::kLinearSoftmax;\n"
         "    else if (value == \"mlp\") g.family = PolicyFamily::kMlp;\n"),
        ("  else if (key == \"init_scale\") g.init_scale = ctx.Double(value);\n",
         "  else if (key == \"init_scale\") g.init_scale = ctx.Double(value);\n"
         "  else if (key == \"hidden\") {  // kMlp trunk widths, comma separated\n"
         "    g.shape.hidden.clear();\n"
         "    std::size_t pos = 0;\n"
         "    while (pos <= value.size()) {\n"
         "      const std::size_t comma = std::min(value.find(',', pos), value.size());\n"
         "      g.shape.hidden.push_back(ctx.U32(value.substr(pos, comma - pos)));\n"
         "      pos = comma + 1;\n"
         "    }\n"
         "  }\n"),
    ])
    # 5. the env fixes obs_dim / n_actions; the configured trunk widths survive
    keep = ("  for (auto& g : groups) {\n"
            "    const std::vector<std::uint32_t> hidden = g.shape.hidden;\n"
            "    g.shape = shape;\n"
            "    g.shape.hidden = hidden;\n"
            "  }\n")
    patch(f"{ref}/src/run/local_run.cpp", f"{out}/src/run/local_run.cpp", [
        ("  for (auto& g : groups) g.shape = shape;\n", keep),
    ])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
