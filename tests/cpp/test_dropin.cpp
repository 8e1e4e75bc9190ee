// The reference's hot-path test cases (proj/tests/test_core.cpp, test_blas.cpp),
// re-run through the drop-in headers, i.e. through the B200 path.  Dense
// checks use small hand-written helpers instead of Eigen.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>

#include "ttlab/blas.hpp"

using namespace ttlab;

static int failures = 0;
#define CHECK(cond)                                                             \
  do {                                                                          \
    if (!(cond)) {                                                              \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);             \
      ++failures;                                                               \
    }                                                                           \
  } while (0)

static double dist(const std::vector<cplx>& a, const std::vector<cplx>& b) {
  double acc = 0.0;
  for (size_t i = 0; i < a.size(); ++i) acc += std::norm(a[i] - b[i]);
  return std::sqrt(acc);
}
static double nrm(const std::vector<cplx>& a) {
  double acc = 0.0;
  for (auto x : a) acc += std::norm(x);
  return std::sqrt(acc);
}

template <typename F> static void section(const char* name, F&& f) {
  const int before = failures;
  try {
    f();
  } catch (const std::exception& e) {
    std::printf("EXCEPTION in %s: %s\n", name, e.what());
    ++failures;
  }
  std::printf("%s %s\n", failures == before ? "ok  " : "FAIL", name);
}

int main() {
  section("canonicalize: isometry invariants and dense state (test_core.cpp:120-129)", [] {
    MPS state = random_uniform_mps(6, 2, 5, 42);
    for (index_t center : {0, 2, 5}) {
      auto c = canonicalize(state, center, NO_TRUNCATION);
      CHECK(c.center() == center);
      CHECK(dist(mps_to_dense(c), mps_to_dense(state)) < 1e-12);
    }
  });
  section("canonicalize: truncation error equals dense distance (test_core.cpp:138-147)", [] {
    MPS state = random_uniform_mps(8, 2, 8, 3);
    auto exact = mps_to_dense(state);
    auto c = canonicalize(state, 3, NO_TRUNCATION.with_max_bond(4));
    const double d = dist(mps_to_dense(c), exact);
    CHECK(d <= c.error());
    CHECK(std::abs(d - c.error()) < 1e-10 * nrm(exact));
    CHECK(c.max_bond_dimension() <= 4);
  });
  section("norm against dense (test_core.cpp:169-174)", [] {
    MPS state = random_uniform_mps(6, 2, 4, 23);
    CHECK(std::abs(state.norm() - nrm(mps_to_dense(state))) < 1e-12 * state.norm());
  });
  section("apply_raw identity (test_core.cpp:201-205)", [] {
    MPS state = random_uniform_mps(5, 2, 3, 21);
    MPS applied = detail::apply_raw(mpo_identity(5, 2), state);
    CHECK(dist(mps_to_dense(applied), mps_to_dense(state)) < 1e-14);
  });
  section("simplify: exact-rank input reproduced (test_blas.cpp:41-45)", [] {
    MPS v = random_uniform_mps(6, 2, 4, 7);
    auto s = simplify(v, DEFAULT_STRATEGY.with_max_sweeps(6));
    CHECK(dist(mps_to_dense(s), mps_to_dense(v)) < 1e-10 * v.norm());
  });
  section("simplify: guess accepted (test_blas.cpp:72-76)", [] {
    MPS v = random_uniform_mps(5, 2, 3, 10);
    auto s = simplify(v, DEFAULT_STRATEGY.with_max_sweeps(8), basis_state(5, 2, 0));
    CHECK(dist(mps_to_dense(s), mps_to_dense(v)) < 1e-9 * v.norm());
  });
  section("apply: identity and shape errors (test_blas.cpp:109-129)", [] {
    MPS v = random_uniform_mps(5, 2, 3, 11);
    auto w = apply(mpo_identity(5, 2), v);
    CHECK(dist(mps_to_dense(w), mps_to_dense(v)) <= 1e-12 * v.norm());
    bool threw = false;
    try {
      apply(mpo_identity(3, 2), random_uniform_mps(4, 2, 1, 1));
    } catch (const shape_error&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      apply(mpo_identity(4, 3), random_uniform_mps(4, 2, 1, 1));
    } catch (const shape_error&) {
      threw = true;
    }
    CHECK(threw);
  });
  section("hadamard: dense oracle and exact bond product (test_blas.cpp:193-201)", [] {
    MPS u = random_uniform_mps(5, 2, 2, 20), v = random_uniform_mps(5, 2, 3, 21);
    MPS w = hadamard(u, v);
    auto du = mps_to_dense(u), dv = mps_to_dense(v), dw = mps_to_dense(w);
    double m = 0.0;
    for (size_t i = 0; i < dw.size(); ++i) m = std::max(m, std::abs(dw[i] - du[i] * dv[i]));
    CHECK(m < 1e-12);
    auto bu = u.bond_dimensions(), bv = v.bond_dimensions(), bw = w.bond_dimensions();
    for (size_t k = 0; k < bw.size(); ++k) CHECK(bw[k] == bu[k] * bv[k]);
  });
  section("scprod against dense (test_blas.cpp:146-151)", [] {
    MPS v = random_uniform_mps(5, 2, 3, 14), u = random_uniform_mps(5, 2, 2, 15);
    auto du = mps_to_dense(u), dv = mps_to_dense(v);
    cplx ref(0);
    for (size_t i = 0; i < du.size(); ++i) ref += std::conj(du[i]) * dv[i];
    CHECK(std::abs(scprod(u, v) - ref) < 1e-12);
  });
  section("simplify_batch equals per-chain simplify", [] {
    std::vector<MPS> chains;
    for (int i = 0; i < 4; ++i) chains.push_back(random_uniform_mps(8, 2, 8, 100 + i));
    auto strat = DEFAULT_STRATEGY.with_max_bond(4);
    auto batch = simplify_batch(chains, strat);
    for (int i = 0; i < 4; ++i) {
      auto one = simplify(chains[i], strat);
      CHECK(dist(mps_to_dense(batch[i]), mps_to_dense(one)) < 1e-10);
      CHECK(std::abs(batch[i].error() - one.error()) < 1e-12);
    }
  });
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
