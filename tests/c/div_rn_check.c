/* The count / N of the ECDF epilogue is computed as q = RN(c * RN(1/N)) followed by one
 * Markstein correction RN(q + RN(c - q N) * RN(1/N)) (common.cuh: div_rn).  This checks that it
 * equals the IEEE quotient c / N for every count c in [0, N] of the benchmark sizes (and a
 * sample for the largest), i.e. that the GPU epilogue is bitwise the reference's division.
 * Built with -ffp-contract=off so that fma() is the only fused operation. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

int main(void) {
  const double Ns[] = {1, 2, 3, 7, 500, 20000, 60000, 65536, 1000000, 1100000, 1200000,
                       10000000, 100000000, 12345677, 99999989};
  long bad = 0, tot = 0;
  for (size_t k = 0; k < sizeof Ns / sizeof Ns[0]; ++k) {
    const double b = Ns[k], rb = 1.0 / b;
    const long step = b > 2e7 ? 7 : 1; /* every 7th count of the largest sizes (speed) */
    for (long i = 0; i <= (long)b; i += step) {
      const double a = (double)i, q = a * rb, q2 = fma(fma(-q, b, a), rb, q);
      if (q2 != a / b) {
        if (bad < 5) printf("mismatch a=%ld b=%.0f\n", i, b);
        ++bad;
      }
      ++tot;
    }
  }
  /* random (c, N) with 1 <= N < 2^31 and 0 <= c <= N (splitmix64 stream, fixed seed) */
  unsigned long long st = 0x2005032460000001ull;
  for (long k = 0; k < 20000000; ++k) {
    unsigned long long z = (st += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const long nb = 1 + (long)(z & 0x7FFFFFFEull);
    const long c = (long)((z >> 32) % (unsigned long long)(nb + 1));
    const double a = (double)c, b = (double)nb, rb = 1.0 / b;
    const double q = a * rb, q2 = fma(fma(-q, b, a), rb, q);
    if (q2 != a / b) {
      if (bad < 5) printf("mismatch a=%ld b=%ld\n", c, nb);
      ++bad;
    }
    ++tot;
  }
  printf("checked %ld quotients, %ld mismatches\n", tot, bad);
  return bad != 0;
}
