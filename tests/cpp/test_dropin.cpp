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
    // sharded form on the context's communicator: one GPU here, so a world of one, first
    // without a communicator, then on a single-rank NCCL communicator (ncclCommInitRank + ncclAllGather)
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) gpu::comm_init(1, 0, gpu::comm_unique_id());
      BatchStats all;
      auto sharded = simplify_batch(chains, strat, &all, 4);
      CHECK(all.norm.size() == 4 && all.error.size() == 4 && all.sweeps.size() == 4);
      for (int i = 0; i < 4; ++i) {
        CHECK(std::abs(all.norm[static_cast<size_t>(i)] - batch[i].norm()) < 1e-12 * batch[i].norm());
        CHECK(std::abs(all.error[static_cast<size_t>(i)] - batch[i].error()) < 1e-12);
        CHECK(all.sweeps[static_cast<size_t>(i)] >= 1);
      }
    }
    CHECK(gpu::shard_range(1024, 8, 3).first == 384 && gpu::shard_range(1024, 8, 3).second == 512);
    CHECK(gpu::shard_range(10, 4, 1).first == 3 && gpu::shard_range(10, 4, 3).second == 10);
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
  section("schmidt_split KATs on the device (test_core.cpp:73-101)", [] {
    Matrix theta = Matrix::Identity(2, 2);
    theta(0, 0) = theta(1, 1) = 1.0 / std::sqrt(2.0);
    auto split = schmidt_split(theta, NO_TRUNCATION);
    CHECK(split.error == 0.0);
    CHECK((split.a * split.b - theta).norm() < 1e-14);
    auto sv = schmidt_values(theta);
    CHECK(std::abs(sv[0] - 1 / std::sqrt(2.0)) < 1e-15 && std::abs(sv[1] - 1 / std::sqrt(2.0)) < 1e-15);
    auto s1 = schmidt_split(theta, NO_TRUNCATION.with_max_bond(1));
    CHECK(std::abs(s1.error - 1 / std::sqrt(2.0)) < 1e-15);
    CHECK(s1.a.cols() == 1);
    Matrix r(4, 4);
    MPS rs = random_uniform_mps(2, 4, 4, 5);  // 4 x 4 complex entries from the reference generator
    for (index_t i = 0; i < 4; ++i)
      for (index_t j = 0; j < 4; ++j) r(i, j) = rs[0](0, i, j) + rs[1](j, 0, 0) * 0.5;
    auto s2 = schmidt_split(r, NO_TRUNCATION.with_max_bond(2));
    CHECK(std::abs((s2.a * s2.b - r).norm() - s2.error) < 1e-12);
    Matrix t6(6, 4);
    MPS r6 = random_uniform_mps(2, 6, 4, 9);
    for (index_t i = 0; i < 6; ++i)
      for (index_t j = 0; j < 4; ++j) t6(i, j) = r6[0](0, i, j);
    auto lr = schmidt_split(t6, NO_TRUNCATION, SweepDirection::LEFT_TO_RIGHT);
    CHECK((lr.a.adjoint() * lr.a - Matrix::Identity(4, 4)).norm() < 1e-12);
    auto rl = schmidt_split(t6, NO_TRUNCATION, SweepDirection::RIGHT_TO_LEFT);
    CHECK((rl.b * rl.b.adjoint() - Matrix::Identity(4, 4)).norm() < 1e-12);
    CHECK((rl.a * rl.b - t6).norm() < 1e-12);
  });
  auto isometries_ok = [](const CanonicalMPS& st) {
    for (index_t n = 0; n < st.size(); ++n) {
      const Tensor3& t = st[n];
      if (n < st.center()) {  // left unfolding a^H a = I
        const index_t rows = t.left_dim() * t.phys_dim(), c = t.right_dim();
        for (index_t i = 0; i < c; ++i)
          for (index_t j = 0; j < c; ++j) {
            cplx acc = 0;
            for (index_t k = 0; k < rows; ++k) acc += std::conj(t.data()[k * c + i]) * t.data()[k * c + j];
            if (std::abs(acc - cplx(i == j ? 1.0 : 0.0)) > 1e-12) return false;
          }
      } else if (n > st.center()) {  // right unfolding b b^H = I
        const index_t rows = t.left_dim(), c = t.phys_dim() * t.right_dim();
        for (index_t i = 0; i < rows; ++i)
          for (index_t j = 0; j < rows; ++j) {
            cplx acc = 0;
            for (index_t k = 0; k < c; ++k) acc += t.data()[i * c + k] * std::conj(t.data()[j * c + k]);
            if (std::abs(acc - cplx(i == j ? 1.0 : 0.0)) > 1e-12) return false;
          }
      }
    }
    return true;
  };
  section("canonicalize: isometries at every centre (test_core.cpp:105-129)", [&] {
    MPS state = random_uniform_mps(6, 2, 5, 42);
    for (index_t center : {0, 2, 5}) {
      auto c = canonicalize(state, center, NO_TRUNCATION);
      CHECK(isometries_ok(c));
    }
    auto c3 = canonicalize(random_uniform_mps(8, 2, 8, 3), 3, NO_TRUNCATION.with_max_bond(4));
    CHECK(isometries_ok(c3));
  });
  section("canonicalize(CanonicalMPS) at the same centre is unchanged (test_core.cpp:130-137)", [] {
    MPS state = random_uniform_mps(5, 2, 4, 7);
    auto c = canonicalize(state, 2, NO_TRUNCATION);
    auto c2 = canonicalize(c, 2, NO_TRUNCATION);
    CHECK(c2.center() == 2);
    for (index_t n = 0; n < c.size(); ++n)
      for (index_t i = 0; i < c[n].size(); ++i) CHECK(std::abs(c[n].data()[i] - c2[n].data()[i]) < 1e-14);
    CHECK(c2.error() == c.error());  // recenter, not a new canonical pass (no floor added)
  });
  section("recenter back and forth leaves the vector invariant (test_core.cpp:148-155)", [&] {
    MPS state = random_uniform_mps(6, 2, 4, 11);
    auto exact = mps_to_dense(state);
    auto c = canonicalize(state, 0, NO_TRUNCATION);
    c.recenter(5, NO_TRUNCATION);
    CHECK(c.center() == 5);
    CHECK(isometries_ok(c));
    c.recenter(0, NO_TRUNCATION);
    CHECK(c.center() == 0);
    CHECK(dist(mps_to_dense(c), exact) < 1e-12 * nrm(exact));
    bool threw = false;
    try {
      c.recenter(6, NO_TRUNCATION);
    } catch (const shape_error&) {
      threw = true;
    }
    CHECK(threw);
  });
  section("truncating moves: error ledger and single moves (mps.hpp:238-279)", [&] {
    MPS state = random_uniform_mps(8, 2, 8, 3);
    auto exact = mps_to_dense(state);
    auto c = canonicalize(state, 3, NO_TRUNCATION);
    const double e0 = c.error();
    const double w = c.move_center_right(NO_TRUNCATION.with_max_bond(4));  // bond 4: 8 -> 4
    CHECK(c.center() == 4 && w > 0.0 && c.error() == e0);  // single moves do not touch the ledger
    c.recenter(7, NO_TRUNCATION.with_max_bond(4));
    CHECK(c.error() > e0);
    CHECK(isometries_ok(c));
    CHECK(dist(mps_to_dense(c), exact) <= c.error() + w + 1e-12);
    const double wl = c.move_center_left(NO_TRUNCATION);
    CHECK(c.center() == 6 && wl < 1e-12);
    c.normalize_in_place();
    CHECK(std::abs(c.norm() - 1.0) < 1e-14);
  });
  section("update_two_site / split_pair on the device (mps.hpp:164-173, 283-297)", [&] {
    MPS state = random_uniform_mps(5, 2, 4, 17);
    auto exact = mps_to_dense(state);
    auto c = canonicalize(state, 1, NO_TRUNCATION);
    Tensor3 joined = detail::join_pair(c[1], c[2]);
    const double e = c.update_two_site(joined, SweepDirection::LEFT_TO_RIGHT, NO_TRUNCATION);
    CHECK(c.center() == 2 && e < 1e-12);
    CHECK(isometries_ok(c));
    CHECK(dist(mps_to_dense(c), exact) < 1e-12 * nrm(exact));
    joined = detail::join_pair(c[1], c[2]);
    c.update_two_site(joined, SweepDirection::RIGHT_TO_LEFT, NO_TRUNCATION);
    CHECK(c.center() == 1);
    CHECK(isometries_ok(c));
    CHECK(dist(mps_to_dense(c), exact) < 1e-12 * nrm(exact));
    c.set_center(1);
    c.set_tensor(1, c[1]);
    bool threw = false;
    try {
      detail::split_pair(joined, 3, 2, NO_TRUNCATION, SweepDirection::LEFT_TO_RIGHT);
    } catch (const shape_error&) {
      threw = true;
    }
    CHECK(threw);
  });
  section("diag(v) w = v .* w (test_core.cpp:183-188, blas.hpp:70-83)", [] {
    MPS v = random_uniform_mps(4, 2, 2, 22);
    MPS w = random_uniform_mps(4, 2, 3, 23);
    auto via_mpo = mps_to_dense(detail::apply_raw(mpo_from_diagonal_mps(v), w));
    auto via_hadamard = mps_to_dense(hadamard(v, w));
    CHECK(dist(via_mpo, via_hadamard) < 1e-12);
    MPS e0 = basis_state(2, 2, 0);
    MPO d = mpo_from_diagonal_mps(e0);
    CHECK(d[0](0, 0, 0, 0) == cplx(1) && d[0](0, 1, 1, 0) == cplx(0) && d[0](0, 0, 1, 0) == cplx(0));
  });
  section("expectation_local on the device (test_blas.cpp:155-178)", [] {
    Matrix sz(2, 2);
    sz(0, 0) = 1.0;
    sz(1, 1) = -1.0;
    CHECK(std::abs(expectation_local(basis_state(3, 2, 0), sz, 0) - cplx(1)) < 1e-15);
    CHECK(std::abs(expectation_local(basis_state(2, 2, 1), sz, 0, sz, 1) + cplx(1)) < 1e-15);
    MPS v = random_uniform_mps(4, 2, 3, 16);
    Matrix op(2, 2);
    op(0, 1) = cplx(0.5, -1.0);
    op(1, 0) = cplx(2.0, 0.25);
    op(1, 1) = 0.75;
    // dense reference: <v| op_2 |v>
    auto dv = mps_to_dense(v);
    cplx ref = 0;
    for (index_t i = 0; i < 16; ++i)
      for (index_t j = 0; j < 16; ++j) {
        bool same = true;
        for (int b = 0; b < 4; ++b)
          if (b != 2 && (((i >> (3 - b)) & 1) != ((j >> (3 - b)) & 1))) same = false;
        if (same) ref += std::conj(dv[i]) * op((i >> 1) & 1, (j >> 1) & 1) * dv[j];
      }
    CHECK(std::abs(expectation_local(v, op, 2) - ref) < 1e-12 * std::abs(ref));
    bool threw = false;
    try {
      expectation_local(v, op, 1, op, 1);
    } catch (const shape_error&) {
      threw = true;
    }
    CHECK(threw);
  });
  section("MPO / Tensor4 host algebra (mpo.hpp:42-92, tensor.hpp:113-142)", [] {
    MPS v = random_uniform_mps(3, 2, 2, 31);
    MPO a = mpo_from_diagonal_mps(v);
    MPO h = a.adjoint();
    CHECK(h.in_dimensions() == a.out_dimensions());
    CHECK(h[1](0, 1, 1, 1) == std::conj(a[1](0, 1, 1, 1)));
    MPO sc = a.scaled(cplx(0, 8.0));
    CHECK(std::abs(sc[0](0, 1, 1, 1) - a[0](0, 1, 1, 1) * cplx(0, 2.0)) < 1e-14);
    CHECK(std::abs(sc[2](1, 0, 0, 0) - a[2](1, 0, 0, 0) * 2.0) < 1e-14);
    Tensor3 f = a[1].fuse_physical();
    CHECK(f.phys_dim() == 4 && f(1, 3, 0) == a[1](1, 1, 1, 0));
    Tensor4 back = Tensor4::split_physical(f, 2, 2);
    CHECK(back(1, 1, 1, 0) == a[1](1, 1, 1, 0));
    CHECK(a[1].conj()(0, 1, 1, 1) == std::conj(a[1](0, 1, 1, 1)));
    Matrix blk = a[1].bond_block(0, 1);
    CHECK(blk(1, 1) == a[1](0, 1, 1, 1));
    MPS cj = v.conj();
    CHECK(cj[0](0, 1, 1) == std::conj(v[0](0, 1, 1)));
  });
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
