// Drop-in restatement of the MPS containers of ttlab/mps.hpp
// (/root/reference/proj/include/ttlab/mps.hpp:21-143, 180-323, 326-412, 416-449, 493-544).
// Containers keep the reference's value semantics and host storage; every
// numerical operation on the hot path (canonical form, norms, overlaps)
// executes on the B200 through the C ABI (include/ttgpu.h, see gpu.hpp).
#pragma once

#include <algorithm>
#include <random>
#include <vector>

#include "ttlab/tensor.hpp"
#include "ttlab/types.hpp"

namespace ttlab {

inline constexpr index_t DENSE_VECTOR_GUARD = index_t(1) << 26;

class MPS {
public:
  MPS() = default;
  explicit MPS(std::vector<Tensor3> tensors, double error = 0.0) : tensors_(std::move(tensors)), error_(error) {
    check_shape();
  }
  index_t size() const { return static_cast<index_t>(tensors_.size()); }
  const Tensor3& operator[](index_t n) const { return tensors_[static_cast<size_t>(n)]; }
  Tensor3& operator[](index_t n) { return tensors_[static_cast<size_t>(n)]; }
  const std::vector<Tensor3>& tensors() const { return tensors_; }
  std::vector<index_t> physical_dimensions() const {
    std::vector<index_t> d;
    for (const auto& t : tensors_) d.push_back(t.phys_dim());
    return d;
  }
  std::vector<index_t> bond_dimensions() const {
    std::vector<index_t> d{tensors_.empty() ? 1 : tensors_.front().left_dim()};
    for (const auto& t : tensors_) d.push_back(t.right_dim());
    return d;
  }
  index_t max_bond_dimension() const {
    index_t chi = 1;
    for (const auto& t : tensors_) chi = std::max({chi, t.left_dim(), t.right_dim()});
    return chi;
  }
  index_t dimension(index_t guard = DENSE_VECTOR_GUARD) const {
    index_t dim = 1;
    for (const auto& t : tensors_) {
      dim *= t.phys_dim();
      if (dim > guard) throw capacity_error("MPS dimension exceeds guard");
    }
    return dim;
  }
  double error() const { return error_; }
  void set_error(double e) { error_ = e; }
  double update_error(double delta) { return error_ += delta; }
  double norm_squared() const;  // <v,v> on the device (gpu.hpp)
  double norm() const { return std::sqrt(std::max(0.0, norm_squared())); }
  /// mps.hpp:98-117 (host container operation): |f|^(1/L) on every tensor, phase on the first.
  MPS scaled(cplx factor) const {
    const double mag = std::abs(factor);
    if (mag == 0.0) return zero_like();
    std::vector<Tensor3> out = tensors_;
    const double root = std::pow(mag, 1.0 / static_cast<double>(size()));
    const cplx phase = factor / mag;
    for (size_t n = 0; n < out.size(); ++n) {
      const cplx f = n == 0 ? root * phase : cplx(root);
      for (index_t i = 0; i < out[n].size(); ++i) out[n].data()[i] *= f;
    }
    return MPS(std::move(out), error_ * mag);
  }
  /// mps.hpp:88-94
  MPS conj() const {
    std::vector<Tensor3> out;
    out.reserve(tensors_.size());
    for (const auto& t : tensors_) out.push_back(t.conj());
    return MPS(std::move(out), error_);
  }
  /// mps.hpp:120-126
  MPS zero_like() const {
    std::vector<Tensor3> out;
    for (const auto& t : tensors_) out.emplace_back(1, t.phys_dim(), 1);
    return MPS(std::move(out), 0.0);
  }

protected:
  void check_shape() const {
    if (tensors_.empty()) return;
    if (tensors_.front().left_dim() != 1 || tensors_.back().right_dim() != 1)
      throw shape_error("MPS boundary bonds must have size one");
    for (size_t n = 0; n + 1 < tensors_.size(); ++n)
      if (tensors_[n].right_dim() != tensors_[n + 1].left_dim())
        throw shape_error("MPS bond mismatch between neighboring tensors");
    if (error_ < 0) throw shape_error("MPS error bound must be non-negative");
  }
  std::vector<Tensor3> tensors_;
  double error_ = 0.0;
};

/// Truncated two-factor split theta ~= a b (schmidt.hpp:62-89), computed on the
/// device (ttg_schmidt_split); LEFT_TO_RIGHT: a is an isometry, RIGHT_TO_LEFT: b is.
struct SchmidtSplit {
  Matrix a;  // rows x rank
  Matrix b;  // rank x cols
  double error;
};
SchmidtSplit schmidt_split(const Matrix& theta, const Strategy& strategy,
                           SweepDirection direction = SweepDirection::LEFT_TO_RIGHT);
/// Schmidt coefficients across a bipartition (schmidt.hpp:92-94), descending.
RealVector schmidt_values(const Matrix& theta);

namespace detail {
/// Join neighbouring tensors into one with fused physical index (s1, s2) (mps.hpp:148-155).
inline Tensor3 join_pair(const Tensor3& a, const Tensor3& b) {
  if (a.right_dim() != b.left_dim()) throw shape_error("join_pair: bond mismatch");
  Tensor3 out(a.left_dim(), a.phys_dim() * b.phys_dim(), b.right_dim());
  const index_t rows = a.left_dim() * a.phys_dim(), inner = a.right_dim(), cols = b.phys_dim() * b.right_dim();
  for (index_t i = 0; i < rows; ++i)
    for (index_t k = 0; k < inner; ++k) {
      const cplx x = a.data()[i * inner + k];
      if (x == cplx(0)) continue;
      for (index_t j = 0; j < cols; ++j) out.data()[i * cols + j] += x * b.data()[k * cols + j];
    }
  return out;
}

struct PairSplit {  // mps.hpp:157-161
  Tensor3 left;
  Tensor3 right;
  double error;
};
/// Split a joined two-site tensor, truncating per `strategy` (mps.hpp:164-173, device).
PairSplit split_pair(const Tensor3& joined, index_t d1, index_t d2, const Strategy& strategy,
                     SweepDirection direction);
}  // namespace detail

/// MPS in canonical form around `center` (off-centre tensors are isometries).
class CanonicalMPS : public MPS {
public:
  CanonicalMPS() = default;
  CanonicalMPS(std::vector<Tensor3> tensors, index_t center, double error)
      : MPS(std::move(tensors), error), center_(center) {}
  /// mps.hpp:188-218 on the device (QR pass + truncating right-to-left pass).
  CanonicalMPS(const MPS& state, index_t center, const Strategy& strategy);
  index_t center() const { return center_; }
  double norm_squared() const {
    const double n = tensors_[static_cast<size_t>(center_)].frobenius_norm();
    return n * n;
  }
  double norm() const { return tensors_[static_cast<size_t>(center_)].frobenius_norm(); }
  /// mps.hpp:227-235
  void normalize_in_place() {
    const double n = norm();
    if (n == 0.0) return;
    auto& t = tensors_[static_cast<size_t>(center_)];
    for (index_t i = 0; i < t.size(); ++i) t.data()[i] /= n;
    error_ /= n;
  }
  /// Move the centre one site right / left, truncating per `strategy`; returns the
  /// dropped weight (mps.hpp:238-265; device, ttg_recenter).
  double move_center_right(const Strategy& strategy);
  double move_center_left(const Strategy& strategy);
  /// Recenter at `target`, accounting truncation in the error ledger (mps.hpp:268-279; device).
  CanonicalMPS& recenter(index_t target, const Strategy& strategy);
  /// Replace the (centre, neighbour) pair by the truncated split of `joined` and move the
  /// centre in `direction` (mps.hpp:283-297; device split).
  double update_two_site(const Tensor3& joined, SweepDirection direction, const Strategy& strategy) {
    const index_t n = center_;
    const bool to_right = direction == SweepDirection::LEFT_TO_RIGHT;
    if ((to_right && n + 1 >= size()) || (!to_right && n == 0))
      throw shape_error("update_two_site: no neighboring pair in that direction");
    const index_t lo = to_right ? n : n - 1;
    const index_t d1 = tensors_[static_cast<size_t>(lo)].phys_dim();
    const index_t d2 = tensors_[static_cast<size_t>(lo + 1)].phys_dim();
    auto split = detail::split_pair(joined, d1, d2, strategy, direction);
    tensors_[static_cast<size_t>(lo)] = std::move(split.left);
    tensors_[static_cast<size_t>(lo + 1)] = std::move(split.right);
    center_ = to_right ? lo + 1 : lo;
    return split.error;
  }
  /// Raw tensor write for sweep kernels; the caller maintains the isometry invariants (mps.hpp:301-302).
  void set_tensor(index_t n, Tensor3 t) { tensors_[static_cast<size_t>(n)] = std::move(t); }
  void set_center(index_t c) { center_ = c; }

private:
  void move_to(index_t target, const Strategy& strategy, double* err);  // device moves (gpu.hpp)
  index_t center_ = 0;
};

inline CanonicalMPS canonicalize(const MPS& state, index_t center = 0, const Strategy& strategy = DEFAULT_STRATEGY) {
  return CanonicalMPS(state, center, strategy);
}

/// Already-canonical input: just move the centre (mps.hpp:316-323).
inline CanonicalMPS canonicalize(const CanonicalMPS& state, index_t center = 0,
                                 const Strategy& strategy = DEFAULT_STRATEGY) {
  CanonicalMPS out = state;
  out.recenter(center, strategy);
  if (strategy.normalize) out.normalize_in_place();
  return out;
}

/// Lazy weighted sum of MPS with equal physical dimensions (mps.hpp:326-412).
class MPSSum {
public:
  MPSSum(std::vector<cplx> weights, std::vector<MPS> states)
      : weights_(std::move(weights)), states_(std::move(states)) {
    if (weights_.empty() || weights_.size() != states_.size())
      throw shape_error("MPSSum: weights and states must be non-empty and match");
    const auto dims = states_.front().physical_dimensions();
    for (const auto& s : states_)
      if (s.physical_dimensions() != dims) throw shape_error("MPSSum: states must share physical dimensions");
  }
  const std::vector<cplx>& weights() const { return weights_; }
  const std::vector<MPS>& states() const { return states_; }
  index_t terms() const { return static_cast<index_t>(states_.size()); }
  index_t size() const { return states_.front().size(); }
  double error() const {  // mps.hpp:344-349
    double acc = 0.0;
    for (size_t l = 0; l < states_.size(); ++l) acc += std::abs(weights_[l]) * states_[l].error();
    return acc;
  }
  MPS join() const;  // mps.hpp:352-405 (device block concatenation, gpu.hpp)

private:
  std::vector<cplx> weights_;
  std::vector<MPS> states_;
};

cplx scprod(const MPS& u, const MPS& v);  // mps.hpp:416-423 (device)
inline double norm(const MPS& s) { return s.norm(); }
inline double norm(const CanonicalMPS& s) { return s.norm(); }

/// Dense vector (mps.hpp:438-449), most significant site first.
inline Vector mps_to_dense(const MPS& state, index_t guard = DENSE_VECTOR_GUARD) {
  const index_t dim = state.dimension(guard);
  std::vector<cplx> acc{cplx(1)};
  index_t rows = 1;
  for (index_t n = 0; n < state.size(); ++n) {
    const Tensor3& t = state[n];
    const index_t a = t.left_dim(), w = t.phys_dim() * t.right_dim();
    std::vector<cplx> next(static_cast<size_t>(rows * w), cplx(0));
    for (index_t r = 0; r < rows; ++r)
      for (index_t k = 0; k < a; ++k) {
        const cplx x = acc[static_cast<size_t>(r * a + k)];
        if (x == cplx(0)) continue;
        for (index_t j = 0; j < w; ++j) next[static_cast<size_t>(r * w + j)] += x * t.data()[k * w + j];
      }
    rows *= t.phys_dim();
    acc = std::move(next);
  }
  if (rows != dim) throw shape_error("mps_to_dense: inconsistent contraction");
#if TTLAB_HAS_EIGEN
  return Eigen::Map<const Vector>(acc.data(), static_cast<index_t>(acc.size()));
#else
  return acc;
#endif
}

/// random_uniform_mps (mps.hpp:493-514): entries cplx(U(-1,1), U(-1,1)) from
/// std::mt19937_64(seed), interior bonds min(bond, d^k, d^(L-k)).
inline MPS random_uniform_mps(index_t L, index_t d, index_t bond, uint64_t seed) {
  if (L < 1 || d < 1 || bond < 1) throw shape_error("random_uniform_mps: L, d, bond must be >= 1");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  auto cap = [&](index_t cut) {
    const double c = std::min({static_cast<double>(bond), std::pow(static_cast<double>(d), static_cast<double>(cut)),
                               std::pow(static_cast<double>(d), static_cast<double>(L - cut))});
    return static_cast<index_t>(std::max(1.0, c));
  };
  std::vector<Tensor3> ts;
  for (index_t n = 0; n < L; ++n) {
    Tensor3 t(cap(n), d, cap(n + 1));
    for (index_t i = 0; i < t.size(); ++i) t.data()[i] = cplx(dist(rng), dist(rng));
    ts.push_back(std::move(t));
  }
  return MPS(std::move(ts), 0.0);
}

inline MPS basis_state(index_t L, index_t d, index_t idx) {
  std::vector<Tensor3> ts(static_cast<size_t>(L));
  index_t rem = idx;
  for (index_t n = L - 1; n >= 0; --n) {
    Tensor3 t(1, d, 1);
    t(0, rem % d, 0) = 1.0;
    ts[static_cast<size_t>(n)] = std::move(t);
    rem /= d;
  }
  return MPS(std::move(ts), 0.0);
}

/// Product state with the same single-site vector at every site (mps.hpp:517-528).
inline MPS product_state(index_t L, const Vector& site) {
  const index_t d = static_cast<index_t>(site.size());
  std::vector<Tensor3> ts;
  for (index_t n = 0; n < L; ++n) {
    Tensor3 t(1, d, 1);
    for (index_t s = 0; s < d; ++s) t(0, s, 0) = site[s];
    ts.push_back(std::move(t));
  }
  return MPS(std::move(ts), 0.0);
}

/// Dense vector -> CanonicalMPS at centre 0 (mps.hpp:453-486): the index is split per `dims` (most
/// significant first) by right-to-left truncated splits (device `schmidt_split`), whose errors are mutually
/// orthogonal; ledger = sqrt(sum err^2) + fp_error_floor(|v|).
inline CanonicalMPS mps_from_dense(const Vector& v, const std::vector<index_t>& dims,
                                   const Strategy& strategy = DEFAULT_STRATEGY) {
  index_t total = 1;
  for (index_t d : dims) {
    if (d < 1) throw shape_error("mps_from_dense: physical dimensions must be >= 1");
    total *= d;
  }
  const index_t nv = static_cast<index_t>(v.size());
  if (total != nv) throw shape_error("mps_from_dense: vector length does not match dimensions");
  const index_t L = static_cast<index_t>(dims.size());
  std::vector<Tensor3> ts(static_cast<size_t>(L));
  std::vector<cplx> rest(static_cast<size_t>(nv));  // row-major (rows x cols) remainder, rows * cols = rest.size()
  double vnorm2 = 0.0;
  for (index_t i = 0; i < nv; ++i) {
    rest[static_cast<size_t>(i)] = v[i];
    vnorm2 += std::norm(rest[static_cast<size_t>(i)]);
  }
  double err2 = 0.0;
  index_t right = 1;
  for (index_t n = L - 1; n > 0; --n) {
    const index_t d = dims[static_cast<size_t>(n)], cols = d * right;
    const index_t rows = static_cast<index_t>(rest.size()) / cols;
    Matrix theta(rows, cols);
    for (index_t i = 0; i < rows; ++i)
      for (index_t j = 0; j < cols; ++j) theta(i, j) = rest[static_cast<size_t>(i * cols + j)];
    const SchmidtSplit sp = schmidt_split(theta, strategy, SweepDirection::RIGHT_TO_LEFT);
    err2 += sp.error * sp.error;
    const index_t rank = sp.b.rows();
    Tensor3 t(rank, d, right);
    for (index_t i = 0; i < rank; ++i)
      for (index_t j = 0; j < cols; ++j) t.data()[i * cols + j] = sp.b(i, j);
    ts[static_cast<size_t>(n)] = std::move(t);
    rest.assign(static_cast<size_t>(rows * rank), cplx(0));
    for (index_t i = 0; i < rows; ++i)
      for (index_t j = 0; j < rank; ++j) rest[static_cast<size_t>(i * rank + j)] = sp.a(i, j);
    right = rank;
  }
  Tensor3 first(1, dims[0], right);
  std::copy(rest.begin(), rest.end(), first.data());
  ts[0] = std::move(first);
  MPS out(std::move(ts), std::sqrt(err2) + detail::fp_error_floor(std::sqrt(vnorm2)));
  CanonicalMPS result(out, 0, NO_TRUNCATION);
  result.set_error(out.error());
  if (strategy.normalize) result.normalize_in_place();
  return result;
}

}  // namespace ttlab

// the device definitions (ttlab/gpu.hpp, pulled in at the end of mpo.hpp) need the MPO container
#include "ttlab/mpo.hpp"
