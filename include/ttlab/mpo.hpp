// Drop-in restatement of the MPO container of ttlab/mpo.hpp
// (/root/reference/proj/include/ttlab/mpo.hpp:14-155), MPOList (:109-129) and
// detail::apply_raw (:213-238, device).
#pragma once

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
