// Drop-in restatement of the MPO container of ttlab/mpo.hpp
// (/root/reference/proj/include/ttlab/mpo.hpp:14-155), MPOList (:109-129) and
// detail::apply_raw (:213-238, device).
#pragma once

#include <algorithm>
#include <cmath>
#include <vector>

#include "ttlab/mps.hpp"
#include "ttlab/tensor.hpp"

namespace ttlab {

inline constexpr index_t DENSE_OPERATOR_GUARD = index_t(1) << 13;  // mpo.hpp:10

class MPO {
public:
  MPO() = default;
  explicit MPO(std::vector<Tensor4> tensors) : tensors_(std::move(tensors)) {
    if (tensors_.empty()) return;
    if (tensors_.front().left_dim() != 1 || tensors_.back().right_dim() != 1)
      throw shape_error("MPO boundary bonds must have size one");
    for (size_t n = 0; n + 1 < tensors_.size(); ++n)
      if (tensors_[n].right_dim() != tensors_[n + 1].left_dim())
        throw shape_error("MPO bond mismatch between neighboring tensors");
  }
  index_t size() const { return static_cast<index_t>(tensors_.size()); }
  const Tensor4& operator[](index_t n) const { return tensors_[static_cast<size_t>(n)]; }
  Tensor4& operator[](index_t n) { return tensors_[static_cast<size_t>(n)]; }
  const std::vector<Tensor4>& tensors() const { return tensors_; }
  std::vector<index_t> bond_dimensions() const {
    std::vector<index_t> d{tensors_.empty() ? 1 : tensors_.front().left_dim()};
    for (const auto& t : tensors_) d.push_back(t.right_dim());
    return d;
  }
  index_t max_bond_dimension() const {  // mpo.hpp:35-40
    index_t chi = 1;
    for (const auto& t : tensors_) chi = std::max(chi, std::max(t.left_dim(), t.right_dim()));
    return chi;
  }
  std::vector<index_t> in_dimensions() const {  // mpo.hpp:42-47
    std::vector<index_t> d;
    for (const auto& t : tensors_) d.push_back(t.in_dim());
    return d;
  }
  std::vector<index_t> out_dimensions() const {  // mpo.hpp:48-53
    std::vector<index_t> d;
    for (const auto& t : tensors_) d.push_back(t.out_dim());
    return d;
  }
  /// mpo.hpp:54-74: |f|^(1/L) on every tensor, the phase on the first.
  MPO scaled(cplx factor) const {
    std::vector<Tensor4> out = tensors_;
    const double mag = std::abs(factor);
    if (mag == 0.0) {
      for (auto& t : out) std::fill(t.data(), t.data() + t.size(), cplx(0));
      return MPO(std::move(out));
    }
    const double root = std::pow(mag, 1.0 / static_cast<double>(size()));
    const cplx phase = factor / mag;
    for (size_t n = 0; n < out.size(); ++n) {
      const cplx f = n == 0 ? root * phase : cplx(root);
      for (index_t i = 0; i < out[n].size(); ++i) out[n].data()[i] *= f;
    }
    return MPO(std::move(out));
  }
  /// Hermitian adjoint: swap in/out indices and conjugate (mpo.hpp:77-92).
  MPO adjoint() const {
    std::vector<Tensor4> out;
    out.reserve(tensors_.size());
    for (const auto& t : tensors_) {
      Tensor4 a(t.left_dim(), t.in_dim(), t.out_dim(), t.right_dim());
      for (index_t c = 0; c < t.left_dim(); ++c)
        for (index_t j = 0; j < t.out_dim(); ++j)
          for (index_t i = 0; i < t.in_dim(); ++i)
            for (index_t cp = 0; cp < t.right_dim(); ++cp) a(c, i, j, cp) = std::conj(t(c, j, i, cp));
      out.push_back(std::move(a));
    }
    return MPO(std::move(out));
  }

private:
  std::vector<Tensor4> tensors_;
};

/// Product of MPO factors; the last entry is applied first (mpo.hpp:109-129).
class MPOList {
public:
  MPOList() = default;
  explicit MPOList(std::vector<MPO> factors) : factors_(std::move(factors)) {}
  index_t terms() const { return static_cast<index_t>(factors_.size()); }
  const MPO& operator[](index_t k) const { return factors_[static_cast<size_t>(k)]; }
  const std::vector<MPO>& factors() const { return factors_; }
  void push_back(MPO op) { factors_.push_back(std::move(op)); }
  MPOList concatenated(const MPOList& other) const {
    MPOList out = *this;
    for (const auto& f : other.factors_) out.push_back(f);
    return out;
  }

private:
  std::vector<MPO> factors_;
};

inline MPO mpo_identity(index_t L, index_t d) {
  std::vector<Tensor4> ts;
  for (index_t n = 0; n < L; ++n) {
    Tensor4 t(1, d, d, 1);
    for (index_t s = 0; s < d; ++s) t(0, s, s, 0) = 1.0;
    ts.push_back(std::move(t));
  }
  return MPO(std::move(ts));
}

/// Identity with per-site physical dimensions (mpo.hpp:145-155).
inline MPO mpo_identity(const std::vector<index_t>& dims) {
  std::vector<Tensor4> ts;
  for (index_t d : dims) {
    Tensor4 t(1, d, d, 1);
    for (index_t s = 0; s < d; ++s) t(0, s, s, 0) = 1.0;
    ts.push_back(std::move(t));
  }
  return MPO(std::move(ts));
}

/// Product of single-site operators, unit bonds (mpo.hpp:158-169).  Host helper.
inline MPO mpo_from_local_operators(const std::vector<Matrix>& ops) {
  std::vector<Tensor4> ts;
  for (const auto& m : ops) {
    Tensor4 t(1, m.rows(), m.cols(), 1);
    for (index_t j = 0; j < m.rows(); ++j)
      for (index_t i = 0; i < m.cols(); ++i) t(0, j, i, 0) = m(j, i);
    ts.push_back(std::move(t));
  }
  return MPO(std::move(ts));
}

/// Dense matrix of an MPO, row index = output, earlier sites most significant (mpo.hpp:172-197).
/// Host helper for small operators (tests, guards): one (J x I) block per open bond value, grown site by site.
inline Matrix mpo_to_dense(const MPO& op, index_t guard = DENSE_OPERATOR_GUARD) {
  index_t J = 1, I = 1;
  for (const auto& t : op.tensors()) {
    J *= t.out_dim();
    I *= t.in_dim();
    if (J > guard || I > guard) throw capacity_error("mpo_to_dense: dimension exceeds guard");
  }
  std::vector<std::vector<cplx>> acc(1, std::vector<cplx>(1, cplx(1)));  // [bond][j * I + i]
  index_t jd = 1, id = 1;
  for (const auto& t : op.tensors()) {
    const index_t jo = t.out_dim(), io = t.in_dim(), nj = jd * jo, ni = id * io;
    std::vector<std::vector<cplx>> next(static_cast<size_t>(t.right_dim()),
                                        std::vector<cplx>(static_cast<size_t>(nj * ni), cplx(0)));
    for (index_t b = 0; b < t.right_dim(); ++b)
      for (index_t a = 0; a < t.left_dim(); ++a)
        for (index_t j0 = 0; j0 < jd; ++j0)
          for (index_t i0 = 0; i0 < id; ++i0) {
            const cplx x = acc[static_cast<size_t>(a)][static_cast<size_t>(j0 * id + i0)];
            if (x == cplx(0)) continue;
            for (index_t j = 0; j < jo; ++j)
              for (index_t i = 0; i < io; ++i)
                next[static_cast<size_t>(b)][static_cast<size_t>((j0 * jo + j) * ni + i0 * io + i)] += x * t(a, j, i, b);
          }
    acc = std::move(next);
    jd = nj;
    id = ni;
  }
  if (acc.size() != 1) throw shape_error("mpo_to_dense: unclosed bond");
  Matrix out(jd, id);
  for (index_t j = 0; j < jd; ++j)
    for (index_t i = 0; i < id; ++i) out(j, i) = acc[0][static_cast<size_t>(j * id + i)];
  return out;
}

/// Dense matrix of an MPOList: product of the factor matrices (mpo.hpp:200-207).
inline Matrix mpo_to_dense(const MPOList& ops, index_t guard = DENSE_OPERATOR_GUARD) {
  if (ops.terms() == 0) throw shape_error("mpo_to_dense: empty MPO list");
  Matrix out = mpo_to_dense(ops[0], guard);
  for (index_t k = 1; k < ops.terms(); ++k) out = out * mpo_to_dense(ops[k], guard);
  return out;
}

/// Weighted sum of MPOs by block concatenation of the scaled terms; exact, bonds add (mpo.hpp:273-312).
inline MPO mpo_sum(const std::vector<cplx>& weights, const std::vector<MPO>& terms) {
  if (weights.empty() || weights.size() != terms.size())
    throw shape_error("mpo_sum: weights and terms must be non-empty and match");
  if (terms.size() == 1) return terms.front().scaled(weights.front());
  const index_t L = terms.front().size();
  std::vector<MPO> parts;
  for (size_t k = 0; k < terms.size(); ++k) {
    if (terms[k].size() != L) throw shape_error("mpo_sum: operator sizes differ");
    parts.push_back(terms[k].scaled(weights[k]));
  }
  std::vector<Tensor4> out;
  for (index_t n = 0; n < L; ++n) {
    const bool first = n == 0, last = n == L - 1;
    index_t dl = 0, dr = 0;
    for (const auto& p : parts) {
      dl += p[n].left_dim();
      dr += p[n].right_dim();
    }
    const Tensor4& f = parts.front()[n];
    Tensor4 t(first ? 1 : dl, f.out_dim(), f.in_dim(), last ? 1 : dr);
    index_t ol = 0, orr = 0;
    for (const auto& p : parts) {  // block (ol.., orr..) of the joint bonds holds this term
      const Tensor4& b = p[n];
      for (index_t a = 0; a < b.left_dim(); ++a)
        for (index_t j = 0; j < b.out_dim(); ++j)
          for (index_t i = 0; i < b.in_dim(); ++i)
            for (index_t c = 0; c < b.right_dim(); ++c) t(first ? 0 : ol + a, j, i, last ? 0 : orr + c) += b(a, j, i, c);
      ol += b.left_dim();
      orr += b.right_dim();
    }
    out.push_back(std::move(t));
  }
  return MPO(std::move(out));
}

namespace detail {
MPS apply_raw(const MPO& op, const MPS& v);  // mpo.hpp:213-238 (device)
}

}  // namespace ttlab

// definitions of the functions declared above that run on the device (schmidt_split, CanonicalMPS, scprod, apply_raw): like the reference, including mps.hpp / mpo.hpp alone is enough
#include "ttlab/gpu.hpp"
