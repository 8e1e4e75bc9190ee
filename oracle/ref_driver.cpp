// TEST INFRASTRUCTURE — command-line driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/ttlab/*.hpp, compiled where they lie; Eigen replaced by
// oracle/eigen_standin, see its header).  Built by oracle/Makefile into oracle/_ref/ttlab_ref.
// It reads TTLAB1 containers (the reference's own serialize.hpp), runs one public entry point
// of the hot path and writes the result as TTLAB1 plus one JSON line on stdout.  Used only by
// tests/golden/make_ref_fixtures.py and tests/test_oracle_vs_ref.py to pin the oracle.
//
//   ttlab_ref <op> <out.ttlab> <strategy> <inputs...>
//     op = apply        <mpo> <mps>            ttlab::apply            blas.hpp:8-11
//          apply_raw    <mpo> <mps>            detail::apply_raw       mpo.hpp:213-238
//          hadamard     <mps> <mps>            ttlab::hadamard         blas.hpp:45-67
//          hadamard_simplify <mps> <mps>       hadamard + simplify
//          simplify     <mps> [guess]          ttlab::simplify         simplify.hpp:182-195
//          canonicalize <center> <mps>         ttlab::canonicalize     mps.hpp:310-313
//          simplify_sum <n> <w_re> <w_im> <mps> ...   simplify(MPSSum) simplify.hpp:198-215
//          apply_sum    <mpo> <n> <w_re> <w_im> <mps> ...   apply(MPO, MPSSum) blas.hpp:13-20
//          scprod       <mps> <mps>            ttlab::scprod           mps.hpp:416-423
//          expectation_mpo <mpo> <mps> <mps>   blas.hpp:128-138
//          qft | iqft   <mps>                  ttlab::qft / iqft (apply(MPOList)) qft.hpp:108-113, blas.hpp:24-32
//          qft_flip     <mps>                  ttlab::qft_flip         qft.hpp:117-128
//          heff <mpo> <bra> <ket> <site>       operator environments (environments.hpp:42-83) up to the pair
//                                              (site, site+1) and y = H_eff x for x = join_pair(ket pair)
//                                              (detail::apply_effective_two_site, eigensolvers.hpp:15-64);
//                                              <out> receives y as raw complex128
//          random_uniform <L> <d> <bond> <seed>  random_uniform_mps   mps.hpp:488-513
//     strategy = method:tolerance:simplification_tolerance:max_bond:max_sweeps:normalize
//                (method V|S, max_bond 0 = unbounded)
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "ttlab/blas.hpp"
#include "ttlab/eigensolvers.hpp"
#include "ttlab/qft.hpp"
#include "ttlab/serialize.hpp"

using namespace ttlab;

static Strategy parse_strategy(const std::string &s) {
  std::vector<std::string> f;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ':'))
    f.push_back(item);
  if (f.size() != 6)
    throw std::invalid_argument("strategy needs 6 fields");
  Strategy out;
  out.method = f[0] == "S" ? Truncation::SVD_TRUNCATE : Truncation::VARIATIONAL;
  out.tolerance = std::strtod(f[1].c_str(), nullptr);
  out.simplification_tolerance = std::strtod(f[2].c_str(), nullptr);
  const long long mb = std::atoll(f[3].c_str());
  out.max_bond = mb <= 0 ? UNBOUNDED_BOND : static_cast<index_t>(mb);
  out.max_sweeps = std::atoi(f[4].c_str());
  out.normalize = f[5] == "1";
  return out;
}

static void report(const MPS &out, const std::string &extra) {
  std::printf("{\"error\": %.17g, \"norm\": %.17g, \"bonds\": [", out.error(), out.norm());
  for (index_t n = 0; n < out.size(); ++n)
    std::printf("%s%lld", n ? ", " : "", static_cast<long long>(out[n].right_dim()));
  std::printf("]%s}\n", extra.c_str());
}

int main(int argc, char **argv) {
  try {
    if (argc < 4)
      throw std::invalid_argument("usage: ttlab_ref <op> <out> <strategy> <inputs...>");
    const std::string op = argv[1], outp = argv[2];
    const Strategy strat = parse_strategy(argv[3]);
    auto arg = [&](int k) -> std::string {
      if (4 + k >= argc)
        throw std::invalid_argument("missing argument");
      return argv[4 + k];
    };
    char buf[256];
    if (op == "apply") {
      CanonicalMPS out = apply(load_mpo(arg(0)), load_mps(arg(1)), strat);
      save_mps(outp, out);
      std::snprintf(buf, sizeof buf, ", \"center\": %lld", static_cast<long long>(out.center()));
      report(out, buf);
    } else if (op == "apply_raw") {
      MPS out = detail::apply_raw(load_mpo(arg(0)), load_mps(arg(1)));
      save_mps(outp, out);
      report(out, "");
    } else if (op == "hadamard") {
      MPS out = hadamard(load_mps(arg(0)), load_mps(arg(1)));
      save_mps(outp, out);
      report(out, "");
    } else if (op == "hadamard_simplify") {
      CanonicalMPS out = simplify(hadamard(load_mps(arg(0)), load_mps(arg(1))), strat);
      save_mps(outp, out);
      report(out, "");
    } else if (op == "simplify") {
      MPS target = load_mps(arg(0));
      std::optional<MPS> guess;
      if (argc > 5)
        guess = load_mps(arg(1));
      CanonicalMPS out = simplify(target, strat, guess);
      save_mps(outp, out);
      // the sweep count is internal to simplify(); run the same internal call once more to report it
      std::string extra;
      if (strat.method == Truncation::VARIATIONAL) {
        auto res = detail::variational_compress({cplx(1)}, {target}, guess ? *guess : MPS(target), strat);
        std::snprintf(buf, sizeof buf, ", \"sweeps\": %d, \"converged\": %s, \"residual\": %.17g", res.sweeps,
                      res.converged ? "true" : "false", res.residual);
        extra = buf;
      }
      report(out, extra);
    } else if (op == "canonicalize") {
      CanonicalMPS out = canonicalize(load_mps(arg(1)), static_cast<index_t>(std::atoll(arg(0).c_str())), strat);
      save_mps(outp, out);
      std::snprintf(buf, sizeof buf, ", \"center\": %lld", static_cast<long long>(out.center()));
      report(out, buf);
    } else if (op == "simplify_sum" || op == "apply_sum") {
      int k = 0;
      std::optional<MPO> W;
      if (op == "apply_sum")
        W = load_mpo(arg(k++));
      const int terms = std::atoi(arg(k++).c_str());
      std::vector<cplx> w;
      std::vector<MPS> states;
      for (int t = 0; t < terms; ++t) {
        const double re = std::strtod(arg(k++).c_str(), nullptr);
        const double im = std::strtod(arg(k++).c_str(), nullptr);
        w.emplace_back(re, im);
        states.push_back(load_mps(arg(k++)));
      }
      MPSSum sum(w, states);
      CanonicalMPS out = W ? apply(*W, sum, strat) : simplify(sum, strat);
      save_mps(outp, out);
      report(out, "");
    } else if (op == "scprod") {
      const cplx v = scprod(load_mps(arg(0)), load_mps(arg(1)));
      std::printf("{\"re\": %.17g, \"im\": %.17g}\n", v.real(), v.imag());
    } else if (op == "expectation_mpo") {
      const cplx v = expectation_mpo(load_mpo(arg(0)), load_mps(arg(1)), load_mps(arg(2)));
      std::printf("{\"re\": %.17g, \"im\": %.17g}\n", v.real(), v.imag());
    } else if (op == "qft" || op == "iqft") {
      MPS v = load_mps(arg(0));
      CanonicalMPS out = op == "qft" ? qft(v, strat) : iqft(v, strat);
      save_mps(outp, out);
      report(out, "");
    } else if (op == "qft_flip") {
      MPS out = qft_flip(load_mps(arg(0)));
      save_mps(outp, out);
      report(out, "");
    } else if (op == "heff") {
      const MPO W = load_mpo(arg(0));
      const MPS bra = load_mps(arg(1)), ket = load_mps(arg(2));
      const index_t site = std::atoll(arg(3).c_str());
      detail::OpEnv lenv = detail::begin_op_environment(), renv = detail::begin_op_environment();
      for (index_t n = 0; n < site; ++n)
        lenv = detail::update_left_op_environment(lenv, bra[n], W[n], ket[n]);
      for (index_t n = ket.size() - 1; n > site + 1; --n)
        renv = detail::update_right_op_environment(renv, bra[n], W[n], ket[n]);
      const Vector x = detail::tensor_to_vector(detail::join_pair(ket[site], ket[site + 1]));
      const Vector y = detail::apply_effective_two_site(lenv, W[site], W[site + 1], renv, x);
      // the same product through the dense effective operator (forms.hpp:34-50), as a self-check of the run
      const Vector yd = detail::effective_two_site_operator(lenv, W[site], W[site + 1], renv) * x;
      std::ofstream out(outp, std::ios::binary);
      out.write(reinterpret_cast<const char *>(y.data()), static_cast<std::streamsize>(sizeof(cplx) * y.size()));
      const Vector xb = detail::tensor_to_vector(detail::join_pair(bra[site], bra[site + 1]));
      const cplx q = xb.dot(y);
      std::printf("{\"size\": %lld, \"re\": %.17g, \"im\": %.17g, \"dense_diff\": %.3g, \"ynorm\": %.17g}\n",
                  static_cast<long long>(y.size()), q.real(), q.imag(), (y - yd).norm(), y.norm());
    } else if (op == "random_uniform") {
      MPS out = random_uniform_mps(std::atoll(arg(0).c_str()), std::atoll(arg(1).c_str()),
                                   std::atoll(arg(2).c_str()), std::strtoull(arg(3).c_str(), nullptr, 10));
      save_mps(outp, out);
      report(out, "");
    } else {
      throw std::invalid_argument("unknown op " + op);
    }
    return 0;
  } catch (const shape_error &e) {
    std::printf("{\"exception\": \"shape_error\", \"what\": \"%s\"}\n", e.what());
    return 3;
  } catch (const capacity_error &e) {
    std::printf("{\"exception\": \"capacity_error\", \"what\": \"%s\"}\n", e.what());
    return 4;
  } catch (const numeric_error &e) {
    std::printf("{\"exception\": \"numeric_error\", \"what\": \"%s\"}\n", e.what());
    return 5;
  } catch (const std::exception &e) {
    std::fprintf(stderr, "ttlab_ref: %s\n", e.what());
    return 2;
  }
}
