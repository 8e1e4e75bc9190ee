// Drop-in ttlab/forms.hpp: the two-site linear and quadratic forms
// (/root/reference/proj/include/ttlab/forms.hpp:91-192) and the plain environments they are built from
// (environments.hpp:13-89).  These are the small host-side helpers of the reference's solvers and tests
// (dense effective operators of dimension (a d1 d2 b)^2); the hot-path versions — environment chains,
// `project_pair` in the minimal contraction order, the two-site effective-operator matvec — run on the
// device inside ttg_simplify / ttg_apply / ttg_apply_effective_two_site.  Same values, same index order.
#pragma once

#include <vector>

#include "ttlab/mpo.hpp"
#include "ttlab/mps.hpp"

namespace ttlab {
namespace detail {

/// Row-major dense block used by the forms (host, small).
struct Dense {
  index_t r = 0, c = 0;
  std::vector<cplx> v;
  Dense() = default;
  Dense(index_t rows, index_t cols) : r(rows), c(cols), v(static_cast<size_t>(rows * cols), cplx(0)) {}
  cplx& operator()(index_t i, index_t j) { return v[static_cast<size_t>(i * c + j)]; }
  const cplx& operator()(index_t i, index_t j) const { return v[static_cast<size_t>(i * c + j)]; }
  static Dense one() {
    Dense d(1, 1);
    d(0, 0) = 1.0;
    return d;
  }
};

/// out[br, kr] = sum_s sum_{a,b} conj(bra[a,s,br]) env[a,b] ket[b,s,kr]   (environments.hpp:18-23)
inline Dense left_env_step(const Dense& env, const Tensor3& bra, const Tensor3& ket) {
  Dense out(bra.right_dim(), ket.right_dim());
  for (index_t s = 0; s < bra.phys_dim(); ++s)
    for (index_t a = 0; a < bra.left_dim(); ++a)
      for (index_t b = 0; b < ket.left_dim(); ++b) {
        const cplx e = env(a, b);
        if (e == cplx(0)) continue;
        for (index_t br = 0; br < bra.right_dim(); ++br) {
          const cplx x = std::conj(bra(a, s, br)) * e;
          for (index_t kr = 0; kr < ket.right_dim(); ++kr) out(br, kr) += x * ket(b, s, kr);
        }
      }
  return out;
}

/// out[bl, kl] = sum_s sum_{a,b} conj(bra[bl,s,a]) env[a,b] ket[kl,s,b]   (environments.hpp:25-30)
inline Dense right_env_step(const Dense& env, const Tensor3& bra, const Tensor3& ket) {
  Dense out(bra.left_dim(), ket.left_dim());
  for (index_t s = 0; s < bra.phys_dim(); ++s)
    for (index_t a = 0; a < bra.right_dim(); ++a)
      for (index_t b = 0; b < ket.right_dim(); ++b) {
        const cplx e = env(a, b);
        if (e == cplx(0)) continue;
        for (index_t bl = 0; bl < bra.left_dim(); ++bl) {
          const cplx x = std::conj(bra(bl, s, a)) * e;
          for (index_t kl = 0; kl < ket.left_dim(); ++kl) out(bl, kl) += x * ket(kl, s, b);
        }
      }
  return out;
}

/// Operator environments, one block per open MPO bond value (environments.hpp:42-83).
using DenseOpEnv = std::vector<Dense>;

inline DenseOpEnv left_op_env_step(const DenseOpEnv& env, const Tensor3& bra, const Tensor4& op, const Tensor3& ket) {
  DenseOpEnv out(static_cast<size_t>(op.right_dim()), Dense(bra.right_dim(), ket.right_dim()));
  for (index_t c = 0; c < op.left_dim(); ++c)
    for (index_t sp = 0; sp < op.out_dim(); ++sp)
      for (index_t s = 0; s < op.in_dim(); ++s)
        for (index_t cp = 0; cp < op.right_dim(); ++cp) {
          const cplx w = op(c, sp, s, cp);
          if (w == cplx(0)) continue;
          const Dense& e = env[static_cast<size_t>(c)];
          Dense& o = out[static_cast<size_t>(cp)];
          for (index_t a = 0; a < bra.left_dim(); ++a)
            for (index_t b = 0; b < ket.left_dim(); ++b) {
              const cplx x = w * e(a, b);
              if (x == cplx(0)) continue;
              for (index_t br = 0; br < bra.right_dim(); ++br) {
                const cplx y = std::conj(bra(a, sp, br)) * x;
                for (index_t kr = 0; kr < ket.right_dim(); ++kr) o(br, kr) += y * ket(b, s, kr);
              }
            }
        }
  return out;
}

inline DenseOpEnv right_op_env_step(const DenseOpEnv& env, const Tensor3& bra, const Tensor4& op, const Tensor3& ket) {
  DenseOpEnv out(static_cast<size_t>(op.left_dim()), Dense(bra.left_dim(), ket.left_dim()));
  for (index_t cp = 0; cp < op.right_dim(); ++cp)
    for (index_t sp = 0; sp < op.out_dim(); ++sp)
      for (index_t s = 0; s < op.in_dim(); ++s)
        for (index_t c = 0; c < op.left_dim(); ++c) {
          const cplx w = op(c, sp, s, cp);
          if (w == cplx(0)) continue;
          const Dense& e = env[static_cast<size_t>(cp)];
          Dense& o = out[static_cast<size_t>(c)];
          for (index_t a = 0; a < bra.right_dim(); ++a)
            for (index_t b = 0; b < ket.right_dim(); ++b) {
              const cplx x = w * e(a, b);
              if (x == cplx(0)) continue;
              for (index_t bl = 0; bl < bra.left_dim(); ++bl) {
                const cplx y = std::conj(bra(bl, sp, a)) * x;
                for (index_t kl = 0; kl < ket.left_dim(); ++kl) o(bl, kl) += y * ket(kl, s, b);
              }
            }
        }
  return out;
}

}  // namespace detail

/// <v| restricted to sites (site, site+1) applied to w: the projection is the two-site tensor the
/// simplification sweep splits (forms.hpp:91-136).
class TwoSiteLinearForm {
public:
  TwoSiteLinearForm(const MPS& v, const MPS& w, index_t site) : v_(v), w_(w), site_(site) {
    if (v.size() != w.size()) throw shape_error("TwoSiteLinearForm: states of different length");
    if (site < 0 || site + 1 >= v.size()) throw shape_error("TwoSiteLinearForm: site out of range");
    left_ = detail::Dense::one();
    for (index_t n = 0; n < site; ++n) left_ = detail::left_env_step(left_, v_[n], w_[n]);
    right_ = detail::Dense::one();
    for (index_t n = v.size() - 1; n > site + 1; --n) right_ = detail::right_env_step(right_, v_[n], w_[n]);
  }

  index_t site() const { return site_; }

  /// out[a, (i1, i2), b] = sum L[a, x] w1[x, i1, m] w2[m, i2, y] R[b, y]   (forms.hpp:13-32)
  Tensor3 projection() const {
    const Tensor3 &k1 = w_[site_], &k2 = w_[site_ + 1];
    const index_t d1 = k1.phys_dim(), d2 = k2.phys_dim(), al = left_.r, ar = right_.r;
    const Tensor3 pair = detail::join_pair(k1, k2);  // [x, (i1, i2), y]
    Tensor3 out(al, d1 * d2, ar);
    for (index_t a = 0; a < al; ++a)
      for (index_t x = 0; x < left_.c; ++x) {
        const cplx lx = left_(a, x);
        if (lx == cplx(0)) continue;
        for (index_t p = 0; p < d1 * d2; ++p)
          for (index_t y = 0; y < right_.c; ++y) {
            const cplx t = lx * pair(x, p, y);
            if (t == cplx(0)) continue;
            for (index_t b = 0; b < ar; ++b) out(a, p, b) += t * right_(b, y);
          }
      }
    return out;
  }

  /// <v, w> evaluated through the form (forms.hpp:128-132).
  cplx scalar() const {
    const Tensor3 f = projection();
    const Tensor3 pair = detail::join_pair(v_[site_], v_[site_ + 1]);
    cplx acc(0);
    for (index_t i = 0; i < f.size(); ++i) acc += std::conj(pair.data()[i]) * f.data()[i];
    return acc;
  }

private:
  MPS v_, w_;
  index_t site_;
  detail::Dense left_, right_;
};

/// <v| op |w> restricted to sites (site, site+1): dense effective two-site operator
/// H[(a, j1, j2, b), (a', i1, i2, b')] = sum L[c0][a, a'] W1[c0, j1, i1, c1] W2[c1, j2, i2, c2] R[c2][b, b']
/// (forms.hpp:34-50, 138-189).  The matrix-free product with the same operator is
/// `ttg_apply_effective_two_site` on the device.
class TwoSiteQuadraticForm {
public:
  TwoSiteQuadraticForm(const MPS& v, const MPO& op, const MPS& w, index_t site) : v_(v), op_(op), w_(w), site_(site) {
    if (v.size() != w.size() || op.size() != v.size()) throw shape_error("TwoSiteQuadraticForm: size mismatch");
    if (site < 0 || site + 1 >= v.size()) throw shape_error("TwoSiteQuadraticForm: site out of range");
    left_ = detail::DenseOpEnv{detail::Dense::one()};
    for (index_t n = 0; n < site; ++n) left_ = detail::left_op_env_step(left_, v_[n], op_[n], w_[n]);
    right_ = detail::DenseOpEnv{detail::Dense::one()};
    for (index_t n = v.size() - 1; n > site + 1; --n) right_ = detail::right_op_env_step(right_, v_[n], op_[n], w_[n]);
  }

  index_t site() const { return site_; }

  Matrix matrix() const {
    const Tensor4 &w1 = op_[site_], &w2 = op_[site_ + 1];
    const index_t al = left_[0].r, alp = left_[0].c, bl = right_[0].r, blp = right_[0].c;
    const index_t j1 = w1.out_dim(), i1 = w1.in_dim(), j2 = w2.out_dim(), i2 = w2.in_dim();
    Matrix out = Matrix::Zero(al * j1 * j2 * bl, alp * i1 * i2 * blp);
    for (index_t c0 = 0; c0 < w1.left_dim(); ++c0)
      for (index_t c1 = 0; c1 < w1.right_dim(); ++c1)
        for (index_t c2 = 0; c2 < w2.right_dim(); ++c2)
          for (index_t a = 0; a < al; ++a)
            for (index_t ap = 0; ap < alp; ++ap) {
              const cplx l = left_[static_cast<size_t>(c0)](a, ap);
              if (l == cplx(0)) continue;
              for (index_t p1 = 0; p1 < j1; ++p1)
                for (index_t q1 = 0; q1 < i1; ++q1) {
                  const cplx x1 = l * w1(c0, p1, q1, c1);
                  if (x1 == cplx(0)) continue;
                  for (index_t p2 = 0; p2 < j2; ++p2)
                    for (index_t q2 = 0; q2 < i2; ++q2) {
                      const cplx x2 = x1 * w2(c1, p2, q2, c2);
                      if (x2 == cplx(0)) continue;
                      for (index_t b = 0; b < bl; ++b)
                        for (index_t bp = 0; bp < blp; ++bp)
                          out(((a * j1 + p1) * j2 + p2) * bl + b, ((ap * i1 + q1) * i2 + q2) * blp + bp) +=
                              x2 * right_[static_cast<size_t>(c2)](b, bp);
                    }
                }
            }
    return out;
  }

  /// <v, op w> evaluated through the form (forms.hpp:183-187).
  cplx scalar() const {
    const Tensor3 vp = detail::join_pair(v_[site_], v_[site_ + 1]);
    const Tensor3 wp = detail::join_pair(w_[site_], w_[site_ + 1]);
    const Matrix h = matrix();
    cplx acc(0);
    for (index_t r = 0; r < h.rows(); ++r) {
      cplx row(0);
      for (index_t c = 0; c < h.cols(); ++c) row += h(r, c) * wp.data()[c];
      acc += std::conj(vp.data()[r]) * row;
    }
    return acc;
  }

private:
  MPS v_;
  MPO op_;
  MPS w_;
  index_t site_;
  detail::DenseOpEnv left_, right_;
};

}  // namespace ttlab
