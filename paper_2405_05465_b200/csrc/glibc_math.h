// glibc_math.h -- bit-exact restatements of the two glibc 2.39 libm routines
// that sit on the predictor hot path, usable from host C++ and sm_100a device
// code alike.
//
//   x = log1p(v)  per feature   (reference estimator.hpp:120)
//   y = exp(reg)  per query     (reference estimator.hpp:122)
//
// The reference is plain C++ linked against glibc, which dispatches both
// functions through an ifunc: on hosts with FMA+AVX2 the variant compiled with
// -mfma runs (GCC contracts a*b+c into fma), elsewhere the SSE2 variant.  The
// two differ in the last ulp for ~0.07% (exp) / ~0.001% (log1p) of inputs, so
// each routine exists here in both contractions; ssg_init() probes the host
// libm once and tells the device which one to use (SSG_MATH_FMA / _PLAIN).
//
// Compile-side contract: every translation unit that includes this header must
// be built without implicit contraction (host: -ffp-contract=off; nvcc:
// --fmad=false), so that the only fused operations are the explicit fma() calls
// below.  Division and sqrt are IEEE round-to-nearest on both sides.
//
// exp: glibc sysdeps/ieee754/dbl-64/e_exp.c (N = 2^7 table, degree-5 poly).
// log1p: glibc sysdeps/ieee754/dbl-64/s_log1p.c (fdlibm, Estrin-split poly).
// Contraction points of the FMA variants were read off the x86-64 code GCC
// emits for the same expressions with -mfma.
#pragma once
#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define SSG_HD __host__ __device__ __forceinline__
#else
#define SSG_HD static inline
#endif

#define SSG_MATH_PLAIN 0
#define SSG_MATH_FMA 1

// tab[2k]   = bits of T_k = RN((2^(k/128) - H_k) / H_k)
// tab[2k+1] = bits of H_k = RN(2^(k/128)), minus (k << 45)
#define SSG_EXP_TAB_BODY \
  0x0000000000000000ULL, 0x3ff0000000000000ULL, \
  0x3c9b3b4f1a88bf6eULL, 0x3feff63da9fb3335ULL, \
  0xbc7160139cd8dc5dULL, 0x3fefec9a3e778061ULL, \
  0xbc905e7a108766d1ULL, 0x3fefe315e86e7f85ULL, \
  0x3c8cd2523567f613ULL, 0x3fefd9b0d3158574ULL, \
  0xbc8bce8023f98efaULL, 0x3fefd06b29ddf6deULL, \
  0x3c60f74e61e6c861ULL, 0x3fefc74518759bc8ULL, \
  0x3c90a3e45b33d399ULL, 0x3fefbe3ecac6f383ULL, \
  0x3c979aa65d837b6dULL, 0x3fefb5586cf9890fULL, \
  0x3c8eb51a92fdeffcULL, 0x3fefac922b7247f7ULL, \
  0x3c3ebe3d702f9cd1ULL, 0x3fefa3ec32d3d1a2ULL, \
  0xbc6a033489906e0bULL, 0x3fef9b66affed31bULL, \
  0xbc9556522a2fbd0eULL, 0x3fef9301d0125b51ULL, \
  0xbc5080ef8c4eea55ULL, 0x3fef8abdc06c31ccULL, \
  0xbc91c923b9d5f416ULL, 0x3fef829aaea92de0ULL, \
  0x3c80d3e3e95c55afULL, 0x3fef7a98c8a58e51ULL, \
  0xbc801b15eaa59348ULL, 0x3fef72b83c7d517bULL, \
  0xbc8f1ff055de323dULL, 0x3fef6af9388c8deaULL, \
  0x3c8b898c3f1353bfULL, 0x3fef635beb6fcb75ULL, \
  0xbc96d99c7611eb26ULL, 0x3fef5be084045cd4ULL, \
  0x3c9aecf73e3a2f60ULL, 0x3fef54873168b9aaULL, \
  0xbc8fe782cb86389dULL, 0x3fef4d5022fcd91dULL, \
  0x3c8a6f4144a6c38dULL, 0x3fef463b88628cd6ULL, \
  0x3c807a05b0e4047dULL, 0x3fef3f49917ddc96ULL, \
  0x3c968efde3a8a894ULL, 0x3fef387a6e756238ULL, \
  0x3c875e18f274487dULL, 0x3fef31ce4fb2a63fULL, \
  0x3c80472b981fe7f2ULL, 0x3fef2b4565e27cddULL, \
  0xbc96b87b3f71085eULL, 0x3fef24dfe1f56381ULL, \
  0x3c82f7e16d09ab31ULL, 0x3fef1e9df51fdee1ULL, \
  0xbc3d219b1a6fbffaULL, 0x3fef187fd0dad990ULL, \
  0x3c8b3782720c0ab4ULL, 0x3fef1285a6e4030bULL, \
  0x3c6e149289cecb8fULL, 0x3fef0cafa93e2f56ULL, \
  0x3c834d754db0abb6ULL, 0x3fef06fe0a31b715ULL, \
  0x3c864201e2ac744cULL, 0x3fef0170fc4cd831ULL, \
  0x3c8fdd395dd3f84aULL, 0x3feefc08b26416ffULL, \
  0xbc86a3803b8e5b04ULL, 0x3feef6c55f929ff1ULL, \
  0xbc924aedcc4b5068ULL, 0x3feef1a7373aa9cbULL, \
  0xbc9907f81b512d8eULL, 0x3feeecae6d05d866ULL, \
  0xbc71d1e83e9436d2ULL, 0x3feee7db34e59ff7ULL, \
  0xbc991919b3ce1b15ULL, 0x3feee32dc313a8e5ULL, \
  0x3c859f48a72a4c6dULL, 0x3feedea64c123422ULL, \
  0xbc9312607a28698aULL, 0x3feeda4504ac801cULL, \
  0xbc58a78f4817895bULL, 0x3feed60a21f72e2aULL, \
  0xbc7c2c9b67499a1bULL, 0x3feed1f5d950a897ULL, \
  0x3c4363ed60c2ac11ULL, 0x3feece086061892dULL, \
  0x3c9666093b0664efULL, 0x3feeca41ed1d0057ULL, \
  0x3c6ecce1daa10379ULL, 0x3feec6a2b5c13cd0ULL, \
  0x3c93ff8e3f0f1230ULL, 0x3feec32af0d7d3deULL, \
  0x3c7690cebb7aafb0ULL, 0x3feebfdad5362a27ULL, \
  0x3c931dbdeb54e077ULL, 0x3feebcb299fddd0dULL, \
  0xbc8f94340071a38eULL, 0x3feeb9b2769d2ca7ULL, \
  0xbc87deccdc93a349ULL, 0x3feeb6daa2cf6642ULL, \
  0xbc78dec6bd0f385fULL, 0x3feeb42b569d4f82ULL, \
  0xbc861246ec7b5cf6ULL, 0x3feeb1a4ca5d920fULL, \
  0x3c93350518fdd78eULL, 0x3feeaf4736b527daULL, \
  0x3c7b98b72f8a9b05ULL, 0x3feead12d497c7fdULL, \
  0x3c9063e1e21c5409ULL, 0x3feeab07dd485429ULL, \
  0x3c34c7855019c6eaULL, 0x3feea9268a5946b7ULL, \
  0x3c9432e62b64c035ULL, 0x3feea76f15ad2148ULL, \
  0xbc8ce44a6199769fULL, 0x3feea5e1b976dc09ULL, \
  0xbc8c33c53bef4da8ULL, 0x3feea47eb03a5585ULL, \
  0xbc845378892be9aeULL, 0x3feea34634ccc320ULL, \
  0xbc93cedd78565858ULL, 0x3feea23882552225ULL, \
  0x3c5710aa807e1964ULL, 0x3feea155d44ca973ULL, \
  0xbc93b3efbf5e2228ULL, 0x3feea09e667f3bcdULL, \
  0xbc6a12ad8734b982ULL, 0x3feea012750bdabfULL, \
  0xbc6367efb86da9eeULL, 0x3fee9fb23c651a2fULL, \
  0xbc80dc3d54e08851ULL, 0x3fee9f7df9519484ULL, \
  0xbc781f647e5a3ecfULL, 0x3fee9f75e8ec5f74ULL, \
  0xbc86ee4ac08b7db0ULL, 0x3fee9f9a48a58174ULL, \
  0xbc8619321e55e68aULL, 0x3fee9feb564267c9ULL, \
  0x3c909ccb5e09d4d3ULL, 0x3feea0694fde5d3fULL, \
  0xbc7b32dcb94da51dULL, 0x3feea11473eb0187ULL, \
  0x3c94ecfd5467c06bULL, 0x3feea1ed0130c132ULL, \
  0x3c65ebe1abd66c55ULL, 0x3feea2f336cf4e62ULL, \
  0xbc88a1c52fb3cf42ULL, 0x3feea427543e1a12ULL, \
  0xbc9369b6f13b3734ULL, 0x3feea589994cce13ULL, \
  0xbc805e843a19ff1eULL, 0x3feea71a4623c7adULL, \
  0xbc94d450d872576eULL, 0x3feea8d99b4492edULL, \
  0x3c90ad675b0e8a00ULL, 0x3feeaac7d98a6699ULL, \
  0x3c8db72fc1f0eab4ULL, 0x3feeace5422aa0dbULL, \
  0xbc65b6609cc5e7ffULL, 0x3feeaf3216b5448cULL, \
  0x3c7bf68359f35f44ULL, 0x3feeb1ae99157736ULL, \
  0xbc93091fa71e3d83ULL, 0x3feeb45b0b91ffc6ULL, \
  0xbc5da9b88b6c1e29ULL, 0x3feeb737b0cdc5e5ULL, \
  0xbc6c23f97c90b959ULL, 0x3feeba44cbc8520fULL, \
  0xbc92434322f4f9aaULL, 0x3feebd829fde4e50ULL, \
  0xbc85ca6cd7668e4bULL, 0x3feec0f170ca07baULL, \
  0x3c71affc2b91ce27ULL, 0x3feec49182a3f090ULL, \
  0x3c6dd235e10a73bbULL, 0x3feec86319e32323ULL, \
  0xbc87c50422622263ULL, 0x3feecc667b5de565ULL, \
  0x3c8b1c86e3e231d5ULL, 0x3feed09bec4a2d33ULL, \
  0xbc91bbd1d3bcbb15ULL, 0x3feed503b23e255dULL, \
  0x3c90cc319cee31d2ULL, 0x3feed99e1330b358ULL, \
  0x3c8469846e735ab3ULL, 0x3feede6b5579fdbfULL, \
  0xbc82dfcd978e9db4ULL, 0x3feee36bbfd3f37aULL, \
  0x3c8c1a7792cb3387ULL, 0x3feee89f995ad3adULL, \
  0xbc907b8f4ad1d9faULL, 0x3feeee07298db666ULL, \
  0xbc55c3d956dcaebaULL, 0x3feef3a2b84f15fbULL, \
  0xbc90a40e3da6f640ULL, 0x3feef9728de5593aULL, \
  0xbc68d6f438ad9334ULL, 0x3feeff76f2fb5e47ULL, \
  0xbc91eee26b588a35ULL, 0x3fef05b030a1064aULL, \
  0x3c74ffd70a5fddcdULL, 0x3fef0c1e904bc1d2ULL, \
  0xbc91bdfbfa9298acULL, 0x3fef12c25bd71e09ULL, \
  0x3c736eae30af0cb3ULL, 0x3fef199bdd85529cULL, \
  0x3c8ee3325c9ffd94ULL, 0x3fef20ab5fffd07aULL, \
  0x3c84e08fd10959acULL, 0x3fef27f12e57d14bULL, \
  0x3c63cdaf384e1a67ULL, 0x3fef2f6d9406e7b5ULL, \
  0x3c676b2c6c921968ULL, 0x3fef3720dcef9069ULL, \
  0xbc808a1883ccb5d2ULL, 0x3fef3f0b555dc3faULL, \
  0xbc8fad5d3ffffa6fULL, 0x3fef472d4a07897cULL, \
  0xbc900dae3875a949ULL, 0x3fef4f87080d89f2ULL, \
  0x3c74a385a63d07a7ULL, 0x3fef5818dcfba487ULL, \
  0xbc82919e2040220fULL, 0x3fef60e316c98398ULL, \
  0x3c8e5a50d5c192acULL, 0x3fef69e603db3285ULL, \
  0x3c843a59ac016b4bULL, 0x3fef7321f301b460ULL, \
  0xbc82d52107b43e1fULL, 0x3fef7c97337b9b5fULL, \
  0xbc892ab93b470dc9ULL, 0x3fef864614f5a129ULL, \
  0x3c74b604603a88d3ULL, 0x3fef902ee78b3ff6ULL, \
  0x3c83c5ec519d7271ULL, 0x3fef9a51fbc74c83ULL, \
  0xbc8ff7128fd391f0ULL, 0x3fefa4afa2a490daULL, \
  0xbc8dae98e223747dULL, 0x3fefaf482d8e67f1ULL, \
  0x3c8ec3bc41aa2008ULL, 0x3fefba1bee615a27ULL, \
  0x3c842b94c3a9eb32ULL, 0x3fefc52b376bba97ULL, \
  0x3c8a64a931d185eeULL, 0x3fefd0765b6e4540ULL, \
  0xbc8e37bae43be3edULL, 0x3fefdbfdad9cbe14ULL, \
  0x3c77893b4d91cd9dULL, 0x3fefe7c1819e90d8ULL, \
  0x3c5305c14160cc89ULL, 0x3feff3c22b8f71f1ULL, \

static const uint64_t ssg_exp_tab_h[256] = {SSG_EXP_TAB_BODY};
#if defined(__CUDACC__)
// Plain global (not __constant__): lanes index it divergently, which would
// serialise on the constant cache; through L1 it is one 2 KB working set.
static __device__ const uint64_t ssg_exp_tab_d[256] = {SSG_EXP_TAB_BODY};
#endif

SSG_HD double ssg_asdouble(uint64_t u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}
SSG_HD uint64_t ssg_asuint64(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
}

SSG_HD const uint64_t* ssg_exp_table() {
#if defined(__CUDA_ARCH__)
  return ssg_exp_tab_d;
#else
  return ssg_exp_tab_h;
#endif
}

// exp(x) for the finite range the estimator produces (|x| < 512; log-runtimes
// of seconds live in about [-25, 10]).  Outside that range the caller must not
// get here: ssg_exp_in_range() guards it and the kernels report an internal
// error rather than guess.
SSG_HD int ssg_exp_in_range(double x) {
  uint32_t abstop = (uint32_t)(ssg_asuint64(x) >> 52) & 0x7ff;
  // glibc: abstop - top12(2^-54) >= top12(512) - top12(2^-54) is the slow path;
  // tiny |x| is handled (1.0 + x), large |x| is not.
  return abstop < 0x408;
}

SSG_HD double ssg_exp(double x, int fma_variant) {
  const double InvLn2N = 0x1.71547652b82fep0 * 128.0;
  const double NegLn2hiN = -0x1.62e42fefa0000p-8;
  const double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double Shift = 0x1.8p52;
  const double C2 = 0x1.ffffffffffdbdp-2;
  const double C3 = 0x1.555555555543cp-3;
  const double C4 = 0x1.55555cf172b91p-5;
  const double C5 = 0x1.1111167a4d017p-7;
  uint32_t abstop = (uint32_t)(ssg_asuint64(x) >> 52) & 0x7ff;
  if (abstop < 0x3c9) return 1.0 + x;  // |x| < 2^-54
  const uint64_t* T = ssg_exp_table();
  double kd, r, r2, tmp;
  uint64_t ki;
  if (fma_variant) {
    kd = fma(InvLn2N, x, Shift);
    ki = ssg_asuint64(kd);
    kd -= Shift;
    r = fma(kd, NegLn2loN, fma(kd, NegLn2hiN, x));
  } else {
    double z = InvLn2N * x;
    kd = z + Shift;
    ki = ssg_asuint64(kd);
    kd -= Shift;
    r = x + kd * NegLn2hiN + kd * NegLn2loN;
  }
  uint64_t idx = 2 * (ki % 128);
  uint64_t top = ki << 45;
  double tail = ssg_asdouble(T[idx]);
  uint64_t sbits = T[idx + 1] + top;
  r2 = r * r;
  double scale = ssg_asdouble(sbits);
  if (fma_variant) {
    tmp = fma(r2 * r2, fma(r, C5, C4), fma(r2, fma(r, C3, C2), tail + r));
    return fma(scale, tmp, scale);
  }
  tmp = tail + r + r2 * (C2 + r * C3) + r2 * r2 * (C4 + r * C5);
  return scale + scale * tmp;
}

SSG_HD int32_t ssg_hi_word(double x) { return (int32_t)(ssg_asuint64(x) >> 32); }
SSG_HD double ssg_with_hi_word(double x, int32_t hi) {
  uint64_t u = (ssg_asuint64(x) & 0xffffffffULL) | ((uint64_t)(uint32_t)hi << 32);
  return ssg_asdouble(u);
}

// log1p(x), fdlibm argument reduction to 1+x = 2^k (1+f), f in [sqrt2/2-1, sqrt2-1],
// then log(1+f) = f - hfsq + s (hfsq + R(z)), s = f/(2+f), z = s^2.
SSG_HD double ssg_log1p(double x, int fma_variant) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  int32_t hx = ssg_hi_word(x);
  int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {  // x < 0.41422
    if (ax >= 0x3ff00000) {  // x <= -1
      if (x == -1.0) return -INFINITY;
      return NAN;
    }
    if (ax < 0x3e200000) {  // |x| < 2^-29
      if (ax < 0x3c900000) return x;
      double xx = x * x;
      return fma_variant ? fma(xx, -0.5, x) : x - xx * 0.5;
    }
    if (ax > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = ssg_hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = ssg_hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = ssg_with_hi_word(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = ssg_with_hi_word(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double dk = (double)k;
  double hfsq = 0.5 * f * f;
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      if (fma_variant) {
        c = fma(dk, ln2_lo, c);
        return fma(dk, ln2_hi, c);
      }
      c += dk * ln2_lo;
      return dk * ln2_hi + c;
    }
    double R;
    if (fma_variant) {
      R = hfsq * fma(-0.66666666666666666, f, 1.0);
      if (k == 0) return f - R;
      double t = fma(dk, ln2_lo, c);
      return fma(dk, ln2_hi, -((R - t) - f));
    }
    R = hfsq * (1.0 - 0.66666666666666666 * f);
    if (k == 0) return f - R;
    return dk * ln2_hi - ((R - (dk * ln2_lo + c)) - f);
  }
  double s = f / (2.0 + f);
  double z = s * s;
  double R;
  if (fma_variant) {
    double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
    double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
    R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, z2 * R2)));
    double p = s * (hfsq + R);
    if (k == 0) return f - (hfsq - p);
    double t = fma(dk, ln2_lo, c);
    return fma(dk, ln2_hi, -((hfsq - (p + t)) - f));
  }
  double R1 = z * Lp1, z2 = z * z;
  double R2 = Lp2 + z * Lp3, z4 = z2 * z2;
  double R3 = Lp4 + z * Lp5, z6 = z4 * z2;
  double R4 = Lp6 + z * Lp7;
  R = R1 + z2 * R2 + z4 * R3 + z6 * R4;
  if (k == 0) return f - (hfsq - s * (hfsq + R));
  return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + (dk * ln2_lo + c))) - f);
}

// llround for the non-negative, finite arguments of equivalent_prefill_length
// (reference estimator.hpp:45): round half away from zero.
SSG_HD int64_t ssg_llround_nonneg(double x) {
  double t = trunc(x);
  if (x - t >= 0.5) t += 1.0;
  return (int64_t)t;
}
