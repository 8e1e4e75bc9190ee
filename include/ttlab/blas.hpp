// Drop-in ttlab/blas.hpp hot-path entries on the B200:
// apply(MPO, MPS, Strategy) (/root/reference/proj/include/ttlab/blas.hpp:8-11), apply(MPO, MPSSum)
// (:13-20), apply(MPOList, MPS | MPSSum) (:24-42), hadamard(MPS, MPS) (:45-67) and
// expectation_mpo (:128-138).
#pragma once

#include "ttlab/simplify.hpp"

namespace ttlab {

inline CanonicalMPS apply(const MPO& op, const MPS& v, const Strategy& strategy = DEFAULT_STRATEGY) {
  if (op.size() != v.size()) throw shape_error("apply: operator and state sizes differ");
  auto w = gpu::upload(op);
  auto d = gpu::upload(v);
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_apply(gpu::ctx(), w.h, d.h, &s, &out, nullptr));
  gpu::DMps o(out);
  return gpu::canonical_from(o.h, 0);
}

inline CanonicalMPS apply(const MPO& op, const MPSSum& v, const Strategy& strategy = DEFAULT_STRATEGY) {
  std::vector<MPS> applied;
  applied.reserve(static_cast<size_t>(v.terms()));
  for (const auto& s : v.states()) applied.push_back(detail::apply_raw(op, s));
  return simplify(MPSSum(v.weights(), applied), strategy);
}

inline CanonicalMPS apply(const MPOList& ops, const MPS& v, const Strategy& strategy = DEFAULT_STRATEGY) {
  if (ops.terms() == 0) throw shape_error("apply: empty MPO list");
  CanonicalMPS state = apply(ops[ops.terms() - 1], v, strategy);
  for (index_t k = ops.terms() - 2; k >= 0; --k) state = apply(ops[k], state, strategy);
  return state;
}

inline CanonicalMPS apply(const MPOList& ops, const MPSSum& v, const Strategy& strategy = DEFAULT_STRATEGY) {
  if (ops.terms() == 0) throw shape_error("apply: empty MPO list");
  CanonicalMPS state = apply(ops[ops.terms() - 1], v, strategy);
  for (index_t k = ops.terms() - 2; k >= 0; --k) state = apply(ops[k], state, strategy);
  return state;
}

/// <u, op v> (blas.hpp:128-138); `v` defaults to `u`.
inline cplx expectation_mpo(const MPO& op, const MPS& u, std::optional<MPS> v = std::nullopt) {
  const MPS& ket = v ? *v : u;
  if (op.size() != u.size() || ket.size() != u.size()) throw shape_error("expectation_mpo: size mismatch");
  auto w = gpu::upload(op);
  auto du = gpu::upload(u);
  std::optional<gpu::DMps> dv;
  if (v) dv.emplace(gpu::upload(*v));
  double re = 0.0, im = 0.0;
  gpu::check(gpu::ctx(), ttg_expectation_mpo(gpu::ctx(), w.h, du.h, dv ? dv->h : nullptr, &re, &im));
  return cplx(re, im);
}

inline MPS hadamard(const MPS& u, const MPS& v) {
  if (u.size() != v.size()) throw shape_error("hadamard: states of different length");
  auto du = gpu::upload(u);
  auto dv = gpu::upload(v);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_hadamard(gpu::ctx(), du.h, dv.h, &out));
  gpu::DMps o(out);
  double err = 0.0;
  auto ts = gpu::download(o.h, 0, &err, nullptr);
  return MPS(std::move(ts), err);
}

}  // namespace ttlab
