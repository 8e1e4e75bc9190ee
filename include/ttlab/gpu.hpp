// Bridge from the drop-in ttlab containers to the B200 C ABI (include/ttgpu.h).
//
// Each host thread owns one device context (device from $TTLAB_DEVICE, default
// 0).  States whose entries are all real are uploaded as float64 (the
// reference promotes them to complex128, types.hpp:12-16; gauge-invariant
// results are the same), everything else as complex128.  ttg status codes are
// rethrown as the reference's exception types (types.hpp:22-37).
#pragma once

#include <cstdlib>
#include <memory>
#include <optional>
#include <vector>

#include "ttgpu.h"
#include "ttlab/mpo.hpp"
#include "ttlab/mps.hpp"

namespace ttlab {
namespace gpu {

inline void check(ttg_ctx* c, ttg_status s) {
  if (s == TTG_OK) return;
  const std::string msg = ttg_last_error(c);
  switch (s) {
    case TTG_SHAPE: throw shape_error(msg);
    case TTG_CAPACITY: throw capacity_error(msg);
    case TTG_NUMERIC: throw numeric_error(msg);
    default: throw std::runtime_error("ttgpu: " + msg);
  }
}

struct Context {
  ttg_ctx* h = nullptr;
  Context() {
    const char* e = std::getenv("TTLAB_DEVICE");
    if (ttg_create(e ? std::atoi(e) : 0, &h) != TTG_OK) throw std::runtime_error("ttgpu: no usable CUDA device");
  }
  ~Context() { ttg_destroy(h); }
};

inline ttg_ctx* ctx() {
  thread_local Context c;
  return c.h;
}

struct DMps {
  ttg_dmps* h = nullptr;
  DMps() = default;
  explicit DMps(ttg_dmps* p) : h(p) {}
  DMps(const DMps&) = delete;
  DMps(DMps&& o) noexcept : h(o.h) { o.h = nullptr; }
  ~DMps() { ttg_mps_free(h); }
};

struct DMpo {
  ttg_dmpo* h = nullptr;
  ~DMpo() { ttg_mpo_free(h); }
};

template <typename T> inline bool all_real(const T& tensors) {
  for (const auto& t : tensors)
    for (index_t i = 0; i < t.size(); ++i)
      if (t.data()[i].imag() != 0.0) return false;
  return true;
}

inline DMps upload(const std::vector<const MPS*>& chains, bool real) {
  const int n = static_cast<int>(chains.front()->size());
  std::vector<std::vector<int64_t>> bonds, phys;
  std::vector<std::vector<std::vector<double>>> reals;
  std::vector<std::vector<const void*>> ptrs;
  std::vector<ttg_mps_view> views;
  bonds.reserve(chains.size());
  phys.reserve(chains.size());
  reals.reserve(chains.size());
  ptrs.reserve(chains.size());
  for (const MPS* m : chains) {
    if (m->size() != n) throw shape_error("batch chains differ in length");
    bonds.emplace_back();
    phys.emplace_back();
    reals.emplace_back();
    ptrs.emplace_back();
    for (auto b : m->bond_dimensions()) bonds.back().push_back(b);
    for (auto d : m->physical_dimensions()) phys.back().push_back(d);
    for (index_t k = 0; k < n; ++k) {
      const Tensor3& t = (*m)[k];
      if (real) {
        reals.back().emplace_back(static_cast<size_t>(t.size()));
        for (index_t i = 0; i < t.size(); ++i) reals.back().back()[static_cast<size_t>(i)] = t.data()[i].real();
      }
    }
    for (index_t k = 0; k < n; ++k)
      ptrs.back().push_back(real ? static_cast<const void*>(reals.back()[static_cast<size_t>(k)].data())
                                 : static_cast<const void*>((*m)[k].data()));
    views.push_back(ttg_mps_view{n, real ? TTG_F64 : TTG_C128, bonds.back().data(), phys.back().data(),
                                 ptrs.back().data(), m->error()});
  }
  ttg_dmps* h = nullptr;
  check(ctx(), ttg_mps_upload(ctx(), views.data(), static_cast<int>(views.size()), &h));
  return DMps(h);
}

inline DMps upload(const MPS& m) { return upload({&m}, all_real(m.tensors())); }

inline std::vector<Tensor3> download(ttg_dmps* h, int chain, double* error, int* center) {
  int n = 0, dtype = 0, count = 0;
  check(ctx(), ttg_mps_info(h, chain, &n, &dtype, &count, nullptr, nullptr, nullptr, nullptr));
  std::vector<int64_t> bonds(static_cast<size_t>(n + 1)), phys(static_cast<size_t>(n));
  check(ctx(), ttg_mps_info(h, chain, nullptr, nullptr, nullptr, bonds.data(), phys.data(), error, center));
  std::vector<Tensor3> ts;
  std::vector<std::vector<double>> reals(static_cast<size_t>(n));
  std::vector<void*> ptrs;
  for (int k = 0; k < n; ++k) {
    ts.emplace_back(bonds[k], phys[k], bonds[k + 1]);
    if (dtype == TTG_F64) {
      reals[k].resize(static_cast<size_t>(ts.back().size()));
      ptrs.push_back(reals[k].data());
    } else {
      ptrs.push_back(ts.back().data());
    }
  }
  check(ctx(), ttg_mps_download(ctx(), h, chain, ptrs.data()));
  if (dtype == TTG_F64)
    for (int k = 0; k < n; ++k)
      for (index_t i = 0; i < ts[k].size(); ++i) ts[k].data()[i] = cplx(reals[k][static_cast<size_t>(i)], 0.0);
  return ts;
}

inline ttg_strategy to_c(const Strategy& s) {
  ttg_strategy c{};
  c.method = s.method == Truncation::SVD_TRUNCATE ? TTG_SVD_TRUNCATE : TTG_VARIATIONAL;
  c.tolerance = s.tolerance;
  c.simplification_tolerance = s.simplification_tolerance;
  c.max_bond = (s.max_bond == UNBOUNDED_BOND || s.max_bond >= (index_t(1) << 31)) ? 0 : s.max_bond;
  c.max_sweeps = s.max_sweeps;
  c.normalize = s.normalize ? 1 : 0;
  return c;
}

inline CanonicalMPS canonical_from(ttg_dmps* h, int chain) {
  double err = 0.0;
  int center = 0;
  auto ts = download(h, chain, &err, &center);
  return CanonicalMPS(std::move(ts), center < 0 ? 0 : center, err);
}

inline DMpo upload(const MPO& op) {
  const int n = static_cast<int>(op.size());
  const bool real = all_real(op.tensors());
  std::vector<int64_t> bonds, dout, din;
  for (auto b : op.bond_dimensions()) bonds.push_back(b);
  std::vector<std::vector<double>> reals;
  std::vector<const void*> ptrs;
  for (int k = 0; k < n; ++k) {
    dout.push_back(op[k].out_dim());
    din.push_back(op[k].in_dim());
    if (real) {
      reals.emplace_back(static_cast<size_t>(op[k].size()));
      for (index_t i = 0; i < op[k].size(); ++i) reals.back()[static_cast<size_t>(i)] = op[k].data()[i].real();
      ptrs.push_back(reals.back().data());
    } else {
      ptrs.push_back(op[k].data());
    }
  }
  ttg_mpo_view v{n, real ? TTG_F64 : TTG_C128, bonds.data(), dout.data(), din.data(), ptrs.data()};
  DMpo w;
  check(ctx(), ttg_mpo_upload(ctx(), &v, &w.h));
  return w;
}

/// Device handles of the summands plus the C arrays ttg_mps_join / ttg_simplify_sum take.
struct SumArgs {
  std::vector<DMps> states;
  std::vector<const ttg_dmps*> handles;
  std::vector<double> wr, wi;
  explicit SumArgs(const MPSSum& s) {
    states.reserve(s.states().size());
    for (size_t l = 0; l < s.states().size(); ++l) {
      states.push_back(upload(s.states()[l]));
      handles.push_back(states.back().h);
      wr.push_back(s.weights()[l].real());
      wi.push_back(s.weights()[l].imag());
    }
  }
  int n() const { return static_cast<int>(handles.size()); }
};

}  // namespace gpu

inline MPS MPSSum::join() const {
  gpu::SumArgs a(*this);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_mps_join(gpu::ctx(), a.n(), a.wr.data(), a.wi.data(), a.handles.data(), &out));
  gpu::DMps o(out);
  double err = 0.0;
  auto ts = gpu::download(o.h, 0, &err, nullptr);
  return MPS(std::move(ts), err);
}

// ---- hot-path entry points (definitions of the declarations in mps.hpp / mpo.hpp)

inline double MPS::norm_squared() const {
  if (tensors_.empty()) return 0.0;
  auto d = gpu::upload(*this);
  double re = 0.0, im = 0.0;
  gpu::check(gpu::ctx(), ttg_scprod(gpu::ctx(), d.h, d.h, &re, &im));
  return re;
}

inline CanonicalMPS::CanonicalMPS(const MPS& state, index_t center, const Strategy& strategy) {
  if (center < 0 || center >= state.size()) throw shape_error("canonical center out of range");
  auto d = gpu::upload(state);
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_canonicalize(gpu::ctx(), d.h, static_cast<int>(center), &s, &out, nullptr));
  gpu::DMps o(out);
  *this = gpu::canonical_from(o.h, 0);
}

inline void CanonicalMPS::move_to(index_t target, const Strategy& strategy, double* err) {
  *err = 0.0;
  if (target == center_) return;
  auto d = gpu::upload(*this);
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_recenter(gpu::ctx(), d.h, static_cast<int>(center_), static_cast<int>(target), &s, &out,
                                      err));
  gpu::DMps o(out);
  double e = 0.0;
  int c = 0;
  tensors_ = gpu::download(o.h, 0, &e, &c);
  center_ = target;
}

inline double CanonicalMPS::move_center_right(const Strategy& strategy) {  // mps.hpp:238-250
  if (center_ + 1 >= size()) throw shape_error("move_center_right: already at the last site");
  double e = 0.0;
  move_to(center_ + 1, strategy, &e);
  return e;
}

inline double CanonicalMPS::move_center_left(const Strategy& strategy) {  // mps.hpp:253-265
  if (center_ == 0) throw shape_error("move_center_left: already at the first site");
  double e = 0.0;
  move_to(center_ - 1, strategy, &e);
  return e;
}

inline CanonicalMPS& CanonicalMPS::recenter(index_t target, const Strategy& strategy) {  // mps.hpp:268-279
  if (target < 0 || target >= size()) throw shape_error("recenter: center out of range");
  double e = 0.0;
  move_to(target, strategy, &e);
  if (e > 0) update_error(e);
  return *this;
}

namespace gpu {
// Row-major host split through ttg_schmidt_split; a: m x r, b: r x n (row-major), returns r.
inline index_t split_rowmajor(const std::vector<cplx>& theta, index_t m, index_t n, const Strategy& strategy,
                              SweepDirection direction, std::vector<cplx>& a, std::vector<cplx>& b, double* err) {
  const index_t k = std::min(m, n);
  bool real = true;
  for (const auto& x : theta) real = real && x.imag() == 0.0;
  const ttg_strategy s = to_c(strategy);
  const int dir = direction == SweepDirection::LEFT_TO_RIGHT ? TTG_LEFT_TO_RIGHT : TTG_RIGHT_TO_LEFT;
  int64_t r = 0;
  if (real) {
    std::vector<double> th(theta.size()), ra(static_cast<size_t>(m * k)), rb(static_cast<size_t>(k * n));
    for (size_t i = 0; i < th.size(); ++i) th[i] = theta[i].real();
    check(ctx(), ttg_schmidt_split(ctx(), TTG_F64, m, n, th.data(), dir, &s, ra.data(), rb.data(), &r, err));
    a.assign(ra.begin(), ra.begin() + m * r);
    b.assign(rb.begin(), rb.begin() + r * n);
  } else {
    a.assign(static_cast<size_t>(m * k), cplx(0));
    b.assign(static_cast<size_t>(k * n), cplx(0));
    check(ctx(), ttg_schmidt_split(ctx(), TTG_C128, m, n, theta.data(), dir, &s, a.data(), b.data(), &r, err));
    a.resize(static_cast<size_t>(m * r));
    b.resize(static_cast<size_t>(r * n));
  }
  return r;
}
}  // namespace gpu

inline SchmidtSplit schmidt_split(const Matrix& theta, const Strategy& strategy, SweepDirection direction) {
  const index_t m = theta.rows(), n = theta.cols();
  std::vector<cplx> th(static_cast<size_t>(m * n)), a, b;
  for (index_t i = 0; i < m; ++i)
    for (index_t j = 0; j < n; ++j) th[static_cast<size_t>(i * n + j)] = theta(i, j);
  SchmidtSplit out;
  const index_t r = gpu::split_rowmajor(th, m, n, strategy, direction, a, b, &out.error);
  out.a = Matrix(m, r);
  out.b = Matrix(r, n);
  for (index_t i = 0; i < m; ++i)
    for (index_t j = 0; j < r; ++j) out.a(i, j) = a[static_cast<size_t>(i * r + j)];
  for (index_t i = 0; i < r; ++i)
    for (index_t j = 0; j < n; ++j) out.b(i, j) = b[static_cast<size_t>(i * n + j)];
  return out;
}

inline RealVector schmidt_values(const Matrix& theta) {
  // b = S V^H of the untruncated split: the row norms are the singular values (descending)
  const auto sp = schmidt_split(theta, NO_TRUNCATION, SweepDirection::LEFT_TO_RIGHT);
  const index_t k = std::min(theta.rows(), theta.cols());
  RealVector s(k);
  for (index_t i = 0; i < k; ++i) {
    double acc = 0.0;
    if (i < sp.b.rows())
      for (index_t j = 0; j < sp.b.cols(); ++j) acc += std::norm(sp.b(i, j));
    s[i] = std::sqrt(acc);
  }
  return s;
}

namespace detail {
inline PairSplit split_pair(const Tensor3& joined, index_t d1, index_t d2, const Strategy& strategy,
                            SweepDirection direction) {  // mps.hpp:164-173
  if (joined.phys_dim() != d1 * d2) throw shape_error("split_pair: fused physical dimension mismatch");
  const index_t al = joined.left_dim(), ar = joined.right_dim();
  std::vector<cplx> th(joined.data(), joined.data() + joined.size()), a, b;
  double err = 0.0;
  const index_t r = gpu::split_rowmajor(th, al * d1, d2 * ar, strategy, direction, a, b, &err);
  PairSplit out{Tensor3(al, d1, r), Tensor3(r, d2, ar), err};
  std::copy(a.begin(), a.end(), out.left.data());
  std::copy(b.begin(), b.end(), out.right.data());
  return out;
}
}  // namespace detail

inline cplx scprod(const MPS& u, const MPS& v) {
  if (u.size() != v.size()) throw shape_error("scprod: states of different length");
  auto du = gpu::upload(u);
  auto dv = gpu::upload(v);
  double re = 0.0, im = 0.0;
  gpu::check(gpu::ctx(), ttg_scprod(gpu::ctx(), du.h, dv.h, &re, &im));
  return cplx(re, im);
}

namespace detail {
inline MPS apply_raw(const MPO& op, const MPS& v) {
  if (op.size() != v.size()) throw shape_error("apply: operator and state sizes differ");
  auto w = gpu::upload(op);
  auto d = gpu::upload(v);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_apply_raw(gpu::ctx(), w.h, d.h, &out));
  gpu::DMps o(out);
  double err = 0.0;
  auto ts = gpu::download(o.h, 0, &err, nullptr);
  return MPS(std::move(ts), err);
}
}  // namespace detail

}  // namespace ttlab
