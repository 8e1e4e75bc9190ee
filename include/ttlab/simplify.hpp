// Drop-in ttlab/simplify.hpp: simplify(MPS) (/root/reference/proj/include/ttlab/simplify.hpp:182-195)
// on the B200, plus the batched extension simplify_batch (no reference counterpart).
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
