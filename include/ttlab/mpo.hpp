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

namespace detail {
MPS apply_raw(const MPO& op, const MPS& v);  // mpo.hpp:213-238 (device)
}

}  // namespace ttlab
