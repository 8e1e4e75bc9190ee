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

/// blas.hpp:13-20.  The applied terms stay on the device: one MPO upload, `ttg_apply_raw` per term, then the
/// sum is compressed by `ttg_simplify_sum` on the device handles (no host round trip of the expanded terms).
inline CanonicalMPS apply(const MPO& op, const MPSSum& v, const Strategy& strategy = DEFAULT_STRATEGY) {
  auto w = gpu::upload(op);
  gpu::SumArgs a(v);
  std::vector<gpu::DMps> applied;
  std::vector<const ttg_dmps*> handles;
  applied.reserve(static_cast<size_t>(a.n()));
  for (int l = 0; l < a.n(); ++l) {
    if (op.size() != v.states()[static_cast<size_t>(l)].size())
      throw shape_error("apply: operator and state sizes differ");
    ttg_dmps* t = nullptr;
    gpu::check(gpu::ctx(), ttg_apply_raw(gpu::ctx(), w.h, a.handles[static_cast<size_t>(l)], &t));
    applied.emplace_back(t);
    handles.push_back(t);
  }
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_simplify_sum(gpu::ctx(), a.n(), a.wr.data(), a.wi.data(), handles.data(), &s, nullptr,
                                          &out, nullptr));
  gpu::DMps o(out);
  return gpu::canonical_from(o.h, 0);
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

/// Register layout of a tensor product: A concatenates the registers, B interleaves them scale by scale
/// (blas.hpp:140).
enum class TensorOrder { A, B };

namespace detail {
/// Order B: output site (j, m) carries state m's tensor at scale j and the identity on the open bonds of the
/// other states — those before m have already advanced to bond j + 1, those after m are still at bond j
/// (blas.hpp:144-196).  The joint bond index is the mixed-radix number of the per-state indices, state 0
/// most significant.
inline MPS interleaved_product(const std::vector<MPS>& states) {
  const index_t L = states.front().size(), M = static_cast<index_t>(states.size());
  for (const auto& s : states)
    if (s.size() != L) throw shape_error("order B requires states of equal length");
  std::vector<Tensor3> out;
  for (index_t j = 0; j < L; ++j)
    for (index_t m = 0; m < M; ++m) {
      std::vector<index_t> ld(static_cast<size_t>(M)), rd(static_cast<size_t>(M));
      index_t left = 1, right = 1;
      for (index_t k = 0; k < M; ++k) {
        const Tensor3& t = states[static_cast<size_t>(k)][j];
        ld[static_cast<size_t>(k)] = k < m ? t.right_dim() : t.left_dim();
        rd[static_cast<size_t>(k)] = k <= m ? t.right_dim() : t.left_dim();
        left *= ld[static_cast<size_t>(k)];
        right *= rd[static_cast<size_t>(k)];
      }
      // strides of slot m and of the slots around it in the joint left / right index
      index_t lo = 1;  // product of the dims of the slots after m (equal on both sides)
      for (index_t k = m + 1; k < M; ++k) lo *= ld[static_cast<size_t>(k)];
      index_t hi = 1;  // product of the dims of the slots before m (equal on both sides)
      for (index_t k = 0; k < m; ++k) hi *= ld[static_cast<size_t>(k)];
      const Tensor3& a = states[static_cast<size_t>(m)][j];
      const index_t dl = a.left_dim(), dr = a.right_dim();
      Tensor3 t(left, a.phys_dim(), right);
      for (index_t h = 0; h < hi; ++h)
        for (index_t x = 0; x < dl; ++x)
          for (index_t y = 0; y < dr; ++y)
            for (index_t s = 0; s < a.phys_dim(); ++s) {
              const cplx v = a(x, s, y);
              if (v == cplx(0)) continue;
              for (index_t w = 0; w < lo; ++w) t((h * dl + x) * lo + w, s, (h * dr + y) * lo + w) = v;
            }
      out.push_back(std::move(t));
    }
  return MPS(std::move(out), 0.0);
}
}  // namespace detail

/// Tensor product of several states (blas.hpp:200-216).  Exact host-side restructuring.
inline MPS mps_tensor_product(const std::vector<MPS>& states, TensorOrder order = TensorOrder::A) {
  if (states.empty()) throw shape_error("mps_tensor_product: no states");
  double err = 0.0;
  for (const auto& s : states) err += s.error();
  if (order == TensorOrder::A) {
    std::vector<Tensor3> out;
    for (const auto& s : states)
      for (index_t n = 0; n < s.size(); ++n) out.push_back(s[n]);
    return MPS(std::move(out), err);
  }
  MPS out = detail::interleaved_product(states);
  out.set_error(err);
  return out;
}

/// Sum of mutually extended vectors: term k holds state k against all-ones registers for the others; the
/// block sum is exact and built on the device by MPSSum::join (blas.hpp:220-246).
inline MPS mps_tensor_sum(const std::vector<MPS>& states, TensorOrder order = TensorOrder::A) {
  if (states.empty()) throw shape_error("mps_tensor_sum: no states");
  const size_t M = states.size();
  if (M == 1) return states.front();
  std::vector<MPS> terms;
  for (size_t k = 0; k < M; ++k) {
    std::vector<MPS> factors;
    for (size_t m = 0; m < M; ++m) {
      if (m == k) {
        factors.push_back(states[m]);
        continue;
      }
      std::vector<Tensor3> ones;
      for (index_t n = 0; n < states[m].size(); ++n) {
        Tensor3 t(1, states[m][n].phys_dim(), 1);
        std::fill(t.data(), t.data() + t.size(), cplx(1));
        ones.push_back(std::move(t));
      }
      factors.emplace_back(std::move(ones), 0.0);
    }
    terms.push_back(mps_tensor_product(factors, order));
  }
  return MPSSum(std::vector<cplx>(M, cplx(1)), terms).join();
}

}  // namespace ttlab
