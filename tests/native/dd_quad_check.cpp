// Host check: the device slow path's double-double log/cos (ig_noise.cuh) is
// correctly rounded -- compared against __float128 (libquadmath).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <quadmath.h>
#include "../../paper_2512_08309_b200/csrc/ig_noise.cuh"
int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 200000;
  uint64_t s = 0x243F6A8885A308D3ull;
  long bad_log = 0, bad_cos = 0;
  for (long i = 0; i < n; ++i) {
    s = ig::fin64(s + ig::kGamma);
    uint64_t k = s >> 32; if (!k) k = 1;
    double u1 = (double)k * 0x1p-32;
    if (ig::cr_log_u32(k) != (double)logq((__float128)u1)) ++bad_log;
    double a = 6.283185307179586 * ((double)(s & 0xFFFFFFFFu) * 0x1p-32);
    if (ig::cr_cos_small(a) != (double)cosq((__float128)a)) ++bad_cos;
  }
  printf("n=%ld bad_log=%ld bad_cos=%ld\n", n, bad_log, bad_cos);
  return (bad_log || bad_cos) ? 1 : 0;
}
