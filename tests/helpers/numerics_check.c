/* Compares the glibc exp/log1p restatement (csrc/glibc_math.h, both
 * contractions) with this host's libm on n pseudo-random inputs spanning the
 * estimator's domain.  Prints the mismatch counts:
 *   "<plain exp> <plain log1p> <fma exp> <fma log1p>" */
#include <stdio.h>
#include <stdlib.h>

#include "glibc_math.h"

static uint64_t s = 88172645463325252ULL;
static uint64_t xr(void) {
  s ^= s << 13;
  s ^= s >> 7;
  s ^= s << 17;
  return s;
}

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  long bad[2][2] = {{0, 0}, {0, 0}};
  for (long i = 0; i < n; ++i) {
    double x = -25.0 + 35.0 * ((double)(xr() >> 11) / 9007199254740992.0);
    double y;
    switch (i % 4) {
      case 0: y = (double)(xr() % 5000000); break;                                 /* token counts */
      case 1: y = (double)(xr() % 2400000) * (double)(1 << (xr() % 17)); break;    /* kv bytes */
      case 2: y = ldexp((double)(xr() >> 11) / 9007199254740992.0, (int)(xr() % 80) - 40); break;
      default: {
        uint64_t u = xr() & 0x7fefffffffffffffULL;
        memcpy(&y, &u, 8);
      }
    }
    double e = exp(x), l = log1p(y);
    for (int v = 0; v < 2; ++v) {
      double a = ssg_exp(x, v), b = ssg_log1p(y, v);
      if (memcmp(&a, &e, 8)) bad[v][0]++;
      if (memcmp(&b, &l, 8)) bad[v][1]++;
    }
  }
  printf("%ld %ld %ld %ld\n", bad[0][0], bad[0][1], bad[1][0], bad[1][1]);
  return 0;
}
