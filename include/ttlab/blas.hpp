// Drop-in ttlab/blas.hpp hot-path entries on the B200:
// apply(MPO, MPS, Strategy) (/root/reference/proj/include/ttlab/blas.hpp:8-11), apply(MPO, MPSSum)
// (:13-20), apply(MPOList, MPS | MPSSum) (:24-42), hadamard(MPS, MPS) (:45-67),
// mpo_from_diagonal_mps (:70-83), expectation_local (:100-125) and expectation_mpo (:128-138).
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

/// diag(v) as an MPO: B[b, j, i, b'] = delta_ji A[b, j, b'] (blas.hpp:70-83).
inline MPO mpo_from_diagonal_mps(const MPS& v) {
  std::vector<Tensor4> out;
  out.reserve(static_cast<size_t>(v.size()));
  for (index_t n = 0; n < v.size(); ++n) {
    const Tensor3& a = v[n];
    Tensor4 t(a.left_dim(), a.phys_dim(), a.phys_dim(), a.right_dim());
    for (index_t al = 0; al < a.left_dim(); ++al)
      for (index_t s = 0; s < a.phys_dim(); ++s)
        for (index_t ar = 0; ar < a.right_dim(); ++ar) t(al, s, s, ar) = a(al, s, ar);
    out.push_back(std::move(t));
  }
  return MPO(std::move(out));
}

/// <v, O_site v> or <v, O_site O2_site2 v> (blas.hpp:100-125), evaluated on the device as the
/// expectation of the bond-1 MPO with `op` (and `op2`) at their sites and identities elsewhere.
inline cplx expectation_local(const MPS& v, const Matrix& op, index_t site, std::optional<Matrix> op2 = std::nullopt,
                              std::optional<index_t> site2 = std::nullopt) {
  if (site < 0 || site >= v.size()) throw shape_error("expectation_local: site out of range");
  if (op2.has_value() != site2.has_value())
    throw shape_error("expectation_local: two-point value needs both operator and site");
  if (op2 && (*site2 < 0 || *site2 >= v.size() || *site2 == site))
    throw shape_error("expectation_local: second site out of range");
  std::vector<Tensor4> ts;
  for (index_t n = 0; n < v.size(); ++n) {
    const index_t d = v[n].phys_dim();
    const Matrix* o = n == site ? &op : (op2 && n == *site2 ? &*op2 : nullptr);
    if (o && (o->rows() != d || o->cols() != d)) throw shape_error("local operator dimension mismatch");
    Tensor4 t(1, d, d, 1);
    for (index_t j = 0; j < d; ++j)
      for (index_t i = 0; i < d; ++i) t(0, j, i, 0) = o ? (*o)(j, i) : cplx(i == j ? 1.0 : 0.0);
    ts.push_back(std::move(t));
  }
  return expectation_mpo(MPO(std::move(ts)), v);
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
