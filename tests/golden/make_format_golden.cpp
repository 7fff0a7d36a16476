// Golden vectors for format_double (io.hpp:13-16 / format.hpp:9-11: "shortest
// decimal representation that parses back to the same double (std::to_chars
// general form)"): libstdc++'s std::to_chars(..., std::chars_format::general)
// on a deterministic mix of random bit patterns, decimal-looking values,
// powers of two and the special values.  Output: "<hex bits> <text>" lines.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>

static void emit(double v) {
  char out[64];
  auto r = std::to_chars(out, out + sizeof out, v, std::chars_format::general);
  *r.ptr = 0;
  uint64_t b;
  std::memcpy(&b, &v, 8);
  std::printf("%016llx %s\n", static_cast<unsigned long long>(b), out);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 4000;
  const double specials[] = {0.0, -0.0, 1.0, -1.0, 100.0, 1e-4, 1e-5, 99999.5, 100000.0, 999999.0, 1000000.0,
                             0.1, 1.0 / 3, 36.787944117144235, 60.653065971263345, 13.533528323661271,
                             1e-300, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                             12345678901234567890.0, std::numeric_limits<double>::infinity(),
                             -std::numeric_limits<double>::infinity()};
  for (double v : specials) emit(v);
  std::mt19937_64 g(0x1309769);
  for (int i = 0; i < n; ++i) {
    double v;
    const uint64_t b = g();
    switch (i % 4) {
      case 0: std::memcpy(&v, &b, 8); if (std::isnan(v)) v = 0.5; break;
      case 1: v = static_cast<double>(b % 100000000000000000ULL) * std::pow(10.0, static_cast<int>(g() % 40) - 36); break;
      case 2: v = static_cast<double>(b % 10000000) * std::pow(10.0, static_cast<int>(g() % 30) - 15); break;
      default: v = std::ldexp(1.0 + static_cast<double>(b % 1000) / 1000.0, static_cast<int>(g() % 200) - 100); break;
    }
    emit(v);
  }
  return 0;
}
