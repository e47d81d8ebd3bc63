// Host check of the device slow path (double-double log/cos) against glibc.
// Built and run by tests/test_noise_host.py; prints mismatch counts.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include "../../paper_2512_08309_b200/csrc/ig_noise.cuh"

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 200000;
  uint64_t s = 0x1234567;
  long bad_log = 0, bad_cos = 0, bad_bm = 0;
  for (long i = 0; i < n; ++i) {
    s = ig::fin64(s + ig::kGamma);
    uint64_t k = (s >> 32); if (!k) k = 1;
    double L = ig::cr_log_u32(k);
    if (L != log((double)k * 0x1p-32)) ++bad_log;
    double u2 = (double)(s & 0xFFFFFFFFu) * 0x1p-32;
    double a = 6.283185307179586 * u2;
    if (ig::cr_cos_small(a) != cos(a)) ++bad_cos;
    double zb = ig::box_muller_exact(k, u2);
    double zr = sqrt(-2.0 * log((double)k * 0x1p-32)) * cos(a);
    if (zb != zr) ++bad_bm;
  }
  printf("n=%ld bad_log=%ld bad_cos=%ld bad_bm=%ld\n", n, bad_log, bad_cos, bad_bm);
  return (bad_log || bad_cos || bad_bm) ? 1 : 0;
}
