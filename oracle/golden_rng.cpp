// Golden-vector generator for the oracle's restatement of the reference's
// random inputs: ttlab::random_uniform_mps (mps.hpp:493-514) and
// oracle::random_matrix (tests/test_utils.hpp:31-39) both draw
// cplx(dist(rng), dist(rng)) from std::mt19937_64 + uniform_real_distribution(-1,1).
// This program uses the same libstdc++ facilities (no reference source) and
// prints the draws as hex doubles so tests/golden/ can pin oracle/rng.py.
// Build+run: g++ -O2 -std=c++20 golden_rng.cpp -o /tmp/golden_rng && /tmp/golden_rng
#include <complex>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <random>

static unsigned long long bits(double x) { unsigned long long u; std::memcpy(&u, &x, 8); return u; }

int main() {
  const unsigned long long seeds[] = {1, 3, 5, 9, 42, 99, 123, 0xDEADBEEFull};
  std::printf("{\n");
  for (size_t k = 0; k < sizeof(seeds) / sizeof(seeds[0]); ++k) {
    std::mt19937_64 rng(seeds[k]);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::printf("  \"%llu\": {\"raw\": [", seeds[k]);
    std::mt19937_64 raw(seeds[k]);
    for (int i = 0; i < 8; ++i) std::printf("%s\"%016llx\"", i ? ", " : "", (unsigned long long)raw());
    std::printf("], \"cplx\": [");
    for (int i = 0; i < 400; ++i) {
      std::complex<double> z(dist(rng), dist(rng));
      std::printf("%s[\"%016llx\", \"%016llx\"]", i ? ", " : "", bits(z.real()), bits(z.imag()));
    }
    std::printf("]}%s\n", k + 1 < sizeof(seeds) / sizeof(seeds[0]) ? "," : "");
  }
  std::printf("}\n");
  return 0;
}
