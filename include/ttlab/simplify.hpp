// Drop-in ttlab/simplify.hpp on the B200: simplify(MPS) (/root/reference/proj/include/ttlab/simplify.hpp:182-195),
// combine (:151-179) and simplify(MPSSum) (:198-215), plus the batched extension simplify_batch
// (no reference counterpart).
#pragma once

#include <optional>

#include "ttlab/gpu.hpp"

namespace ttlab {

inline CanonicalMPS simplify(const MPS& target, const Strategy& strategy = DEFAULT_STRATEGY,
                             std::optional<MPS> guess = std::nullopt) {
  auto t = gpu::upload(target);
  std::optional<gpu::DMps> g;
  if (guess) g.emplace(gpu::upload(*guess));
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_simplify(gpu::ctx(), t.h, &s, g ? g->h : nullptr, &out, nullptr));
  gpu::DMps o(out);
  return gpu::canonical_from(o.h, 0);
}

/// Compress a lazy sum (simplify.hpp:198-215); guess defaults to default_guess (:133-144).
inline CanonicalMPS simplify(const MPSSum& target, const Strategy& strategy = DEFAULT_STRATEGY,
                             std::optional<MPS> guess = std::nullopt) {
  gpu::SumArgs a(target);
  std::optional<gpu::DMps> g;
  if (guess) g.emplace(gpu::upload(*guess));
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_simplify_sum(gpu::ctx(), a.n(), a.wr.data(), a.wi.data(), a.handles.data(), &s,
                                          g ? g->h : nullptr, &out, nullptr));
  gpu::DMps o(out);
  return gpu::canonical_from(o.h, 0);
}

/// Closest MPS under `strategy` to sum_l weights[l] states[l] (simplify.hpp:151-179).
inline CanonicalMPS combine(const std::vector<cplx>& weights, const std::vector<MPS>& states,
                            const Strategy& strategy = DEFAULT_STRATEGY) {
  if (weights.empty() || weights.size() != states.size())
    throw shape_error("combine: weights and states must be non-empty and match");
  const auto dims = states.front().physical_dimensions();
  for (const auto& s : states)
    if (s.physical_dimensions() != dims) throw shape_error("combine: states must share physical dimensions");
  return simplify(MPSSum(weights, states), strategy);
}

/// Batched simplify of independent, identically shaped chains (one device call).
inline std::vector<CanonicalMPS> simplify_batch(const std::vector<MPS>& targets,
                                                const Strategy& strategy = DEFAULT_STRATEGY) {
  if (targets.empty()) return {};
  std::vector<const MPS*> ptrs;
  bool real = true;
  for (const auto& m : targets) {
    ptrs.push_back(&m);
    real = real && gpu::all_real(m.tensors());
  }
  auto t = gpu::upload(ptrs, real);
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_simplify(gpu::ctx(), t.h, &s, nullptr, &out, nullptr));
  gpu::DMps o(out);
  std::vector<CanonicalMPS> res;
  for (size_t c = 0; c < targets.size(); ++c) res.push_back(gpu::canonical_from(o.h, static_cast<int>(c)));
  return res;
}

}  // namespace ttlab
