// Drop-in ttlab/simplify.hpp on the B200: simplify(MPS) (/root/reference/proj/include/ttlab/simplify.hpp:182-195),
// combine (:151-179) and simplify(MPSSum) (:198-215), plus the batched extension simplify_batch
// (no reference counterpart).
#pragma once

#include <optional>

#include "ttlab/forms.hpp"
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

namespace detail {
/// MPO -> MPS with the (out, in) pair fused into one physical index, and back (simplify.hpp:219-237).
inline MPS flatten_mpo(const MPO& op) {
  std::vector<Tensor3> ts;
  for (index_t n = 0; n < op.size(); ++n) ts.push_back(op[n].fuse_physical());
  return MPS(std::move(ts), 0.0);
}
inline MPO unflatten_mpo(const MPS& state, const std::vector<index_t>& out_dims, const std::vector<index_t>& in_dims) {
  std::vector<Tensor4> ts;
  for (index_t n = 0; n < state.size(); ++n)
    ts.push_back(Tensor4::split_physical(state[n], out_dims[static_cast<size_t>(n)], in_dims[static_cast<size_t>(n)]));
  return MPO(std::move(ts));
}
}  // namespace detail

/// Compress an MPO: flatten, simplify the state on the device, unflatten (simplify.hpp:241-245).
inline MPO simplify_mpo(const MPO& op, const Strategy& strategy = DEFAULT_STRATEGY) {
  const CanonicalMPS compact = simplify(detail::flatten_mpo(op), strategy.with_normalize(false));
  return detail::unflatten_mpo(compact, op.out_dimensions(), op.in_dimensions());
}

/// Compress a weighted sum of MPOs the same way (simplify.hpp:248-260).
inline MPO simplify_mpo(const std::vector<cplx>& weights, const std::vector<MPO>& terms,
                        const Strategy& strategy = DEFAULT_STRATEGY) {
  if (weights.empty() || weights.size() != terms.size())
    throw shape_error("simplify_mpo: weights and terms must be non-empty and match");
  std::vector<MPS> flats;
  for (const auto& t : terms) flats.push_back(detail::flatten_mpo(t));
  const CanonicalMPS compact = simplify(MPSSum(weights, flats), strategy.with_normalize(false));
  return detail::unflatten_mpo(compact, terms.front().out_dimensions(), terms.front().in_dimensions());
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
