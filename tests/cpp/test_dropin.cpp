// The reference's hot-path test cases (proj/tests/test_core.cpp, test_blas.cpp),
// re-run through the drop-in headers, i.e. through the B200 path.  Dense
// checks use small hand-written helpers instead of Eigen.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>

#include "ttlab/blas.hpp"
#include "ttlab/qft.hpp"
#include "ttlab/serialize.hpp"

#include <sstream>

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
  section("combine: v+v, v-v, 3-term dense sum, SVD route, errors (test_blas.cpp:8-36)", [] {
    MPS v = random_uniform_mps(4, 2, 2, 1);
    auto s = combine({1.0, 1.0}, {v, v});
    auto dv = mps_to_dense(v);
    for (auto& x : dv) x *= 2.0;
    CHECK(dist(mps_to_dense(s), dv) < 1e-12);
    MPS u = random_uniform_mps(4, 2, 2, 2);
    CHECK(combine({1.0, -1.0}, {u, u}).norm() <= 1e-12);
    std::vector<MPS> states = {random_uniform_mps(5, 2, 2, 3), random_uniform_mps(5, 2, 3, 4),
                               random_uniform_mps(5, 2, 2, 5)};
    std::vector<cplx> w = {cplx(0.3, -1.0), cplx(-2.0, 0.1), cplx(0.0, 0.7)};
    std::vector<cplx> expected(32, cplx(0));
    for (size_t l = 0; l < states.size(); ++l) {
      auto d = mps_to_dense(states[l]);
      for (size_t i = 0; i < d.size(); ++i) expected[i] += w[l] * d[i];
    }
    auto sum = combine(w, states, DEFAULT_STRATEGY.with_max_sweeps(8));
    CHECK(dist(mps_to_dense(sum), expected) < 1e-10);
    CHECK(dist(mps_to_dense(sum), expected) <= sum.error());
    auto svd_sum = combine(w, states, NO_TRUNCATION);
    CHECK(dist(mps_to_dense(svd_sum), expected) < 1e-10);
    CHECK(dist(mps_to_dense(MPSSum(w, states).join()), expected) < 1e-12);
    bool threw = false;
    try {
      combine({}, {});
    } catch (const shape_error&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      combine({1.0}, {random_uniform_mps(3, 2, 1, 1), random_uniform_mps(3, 2, 1, 2)});
    } catch (const shape_error&) {
      threw = true;
    }
    CHECK(threw);
  });
  section("simplify(MPSSum): v - v collapses to zero (test_blas.cpp:67-71)", [] {
    MPS v = random_uniform_mps(4, 2, 3, 9);
    auto s = simplify(MPSSum({1.0, -1.0}, {v, v}));
    CHECK(s.norm() <= 1e-12);
  });
  section("apply(MPOList) right to left, apply(MPO, MPSSum) (test_blas.cpp:132-141)", [] {
    auto local = [](cplx a, cplx b, cplx c, cplx d) {
      std::vector<Tensor4> ts;
      for (int n = 0; n < 3; ++n) {
        Tensor4 t(1, 2, 2, 1);
        if (n == 0) {
          t(0, 0, 0, 0) = a; t(0, 0, 1, 0) = b; t(0, 1, 0, 0) = c; t(0, 1, 1, 0) = d;
        } else {
          t(0, 0, 0, 0) = 1.0; t(0, 1, 1, 0) = 1.0;
        }
        ts.push_back(std::move(t));
      }
      return MPO(std::move(ts));
    };
    const cplx m1[4] = {0.3, -1.2, 0.7, 0.4}, m2[4] = {cplx(0.1, 1.0), 0.5, -0.8, 2.0};
    MPO a = local(m1[0], m1[1], m1[2], m1[3]), b = local(m2[0], m2[1], m2[2], m2[3]);
    MPS v = random_uniform_mps(3, 2, 2, 13);
    auto dv = mps_to_dense(v);  // index = s0 * 4 + rest: the local operator acts on s0
    auto act = [](const cplx* m, const std::vector<cplx>& x) {
      std::vector<cplx> y(x.size());
      for (size_t r = 0; r < 4; ++r)
        for (int j = 0; j < 2; ++j) y[j * 4 + r] = m[j * 2 + 0] * x[r] + m[j * 2 + 1] * x[4 + r];
      return y;
    };
    auto expected = act(m1, act(m2, dv));
    CHECK(dist(mps_to_dense(apply(MPOList({a, b}), v)), expected) < 1e-10);
    MPS u = random_uniform_mps(3, 2, 2, 14);
    auto du = mps_to_dense(u);
    std::vector<cplx> mix(dv.size());
    for (size_t i = 0; i < dv.size(); ++i) mix[i] = 0.5 * dv[i] + cplx(0, -1) * du[i];
    auto got = apply(b, MPSSum({0.5, cplx(0, -1)}, {v, u}), DEFAULT_STRATEGY.with_max_sweeps(8));
    CHECK(dist(mps_to_dense(got), act(m2, mix)) < 1e-10 * nrm(mix) + 1e-12);
  });
  section("qft: e_0 -> uniform, iqft(qft(v)) = v, qft_flip(qft(v)) = DFT (test_lapack.cpp:265-291)", [] {
    auto f = mps_to_dense(qft(basis_state(6, 2, 0)));
    double worst = 0.0;
    for (auto x : f) worst = std::max(worst, std::abs(x - cplx(1.0 / 8.0)));
    CHECK(worst < 1e-12);
    MPS v = random_uniform_mps(6, 2, 3, 23);
    CHECK(dist(mps_to_dense(iqft(qft(v))), mps_to_dense(v)) < 1e-12 * v.norm());
    MPS u = random_uniform_mps(6, 2, 3, 24);
    auto x = mps_to_dense(u);
    std::vector<cplx> expected(64);
    const double pi = std::acos(-1.0);
    for (int i = 0; i < 64; ++i) {
      cplx acc(0);
      for (int j = 0; j < 64; ++j) acc += std::polar(1.0, -2.0 * pi * i * j / 64.0) * x[static_cast<size_t>(j)];
      expected[static_cast<size_t>(i)] = acc / 8.0;
    }
    CHECK(dist(mps_to_dense(qft_flip(qft(u))), expected) < 1e-10);
    CHECK(dist(mps_to_dense(qft_flip(qft_flip(u))), x) == 0.0);
  });
  section("expectation_mpo: identity = scprod (test_blas.cpp:170-174)", [] {
    MPS u = random_uniform_mps(4, 2, 2, 17), v = random_uniform_mps(4, 2, 3, 18);
    CHECK(std::abs(expectation_mpo(mpo_identity(4, 2), u, v) - scprod(u, v)) < 1e-12);
    CHECK(std::abs(expectation_mpo(mpo_identity(4, 2), u) - u.norm_squared()) < 1e-12);
  });
  section("serialization round trip is bit exact; device loader reads the same file (test_core.cpp:229-256)", [] {
    MPS state = random_uniform_mps(5, 2, 4, 123);
    state.set_error(0.125);
    std::stringstream buffer;
    save_mps(buffer, state);
    MPS loaded = load_mps(buffer);
    CHECK(loaded.size() == state.size());
    CHECK(loaded.error() == state.error());
    for (index_t n = 0; n < state.size(); ++n)
      CHECK(std::memcmp(loaded[n].data(), state[n].data(), sizeof(cplx) * static_cast<size_t>(state[n].size())) == 0);
    MPO op = mpo_identity(3, 2);
    std::stringstream obuf;
    save_mpo(obuf, op);
    MPO oload = load_mpo(obuf);
    CHECK(oload.size() == op.size());
    bool threw = false;
    try {
      std::stringstream bad("garbage");
      load_mps(bad);
    } catch (const numeric_error&) {
      threw = true;
    }
    CHECK(threw);
    const std::string path = "/tmp/ttgpu_dropin_state.ttlab";
    save_mps(path, state);
    ttg_dmps* d = nullptr;
    gpu::check(gpu::ctx(), ttg_mps_load(gpu::ctx(), path.c_str(), 1, &d));
    gpu::DMps dm(d);
    double err = 0.0;
    auto ts = gpu::download(dm.h, 0, &err, nullptr);
    CHECK(err == 0.125);
    for (index_t n = 0; n < state.size(); ++n)
      CHECK(std::memcmp(ts[static_cast<size_t>(n)].data(), state[n].data(),
                        sizeof(cplx) * static_cast<size_t>(state[n].size())) == 0);
    std::remove(path.c_str());
  });
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
