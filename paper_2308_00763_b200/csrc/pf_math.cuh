// pf_math.cuh -- portable, IEEE-only transcendental functions.
//
// Every function here is a fixed sequence of correctly rounded +,-,*,/ (no
// FMA: explicit __d*_rn / __f*_rn intrinsics, and the library is built with
// -fmad=false), so it returns the same bits as its NumPy restatement in
// oracle/rng.py (exp64_np, exp32_np, log64, log1p64).  That is what makes the
// device RNG slow path and the fused FP32/FP64 weights bit-reproducible on
// the host.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace pfm {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }

// c_i = c_{i-1} / i  (oracle/rng.py EXP_COEF)
__constant__ double kExpC[14] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1,
    0x1.5555555555555p-3, 0x1.5555555555555p-5, 0x1.1111111111111p-7,
    0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16,
    0x1.71de3a556c734p-19, 0x1.27e4fb7789f5dp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d0ap-33};
// 1/(2i+1)  (oracle/rng.py LOG_COEF)
__constant__ double kLogC[12] = {
    0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3,
    0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4,
    0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
    0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
__constant__ float kExpCf[9] = {0x1.0000000000000p+0f, 0x1.0000000000000p+0f, 0x1.0000000000000p-1f,
                                0x1.5555560000000p-3f, 0x1.5555560000000p-5f, 0x1.1111120000000p-7f,
                                0x1.6c16c20000000p-10f, 0x1.a01a020000000p-13f, 0x1.a01a020000000p-16f};

constexpr double kLog2e = 0x1.71547652b82fep+0;
constexpr double kLn2Hi = 0x1.62e42fee00000p-1;
constexpr double kLn2Lo = 0x1.a39ef35793c76p-33;
constexpr double kSqrt2 = 0x1.6a09e667f3bcdp+0;
constexpr float kLog2ef = 0x1.7154760000000p+0f;
constexpr float kLn2Hif = 0x1.62e4000000000p-1f;
constexpr float kLn2Lof = 0x1.7f7d1c0000000p-20f;

// oracle/rng.py exp64 / exp64_np
__device__ __forceinline__ double exp64(double x) {
  if (x != x) return x;
  if (x < -708.0) return 0.0;
  if (x > 709.0) return __longlong_as_double(0x7ff0000000000000LL);
  double k = rint(dmul(x, kLog2e));
  double r = dsub(dsub(x, dmul(k, kLn2Hi)), dmul(k, kLn2Lo));
  double p = kExpC[13];
#pragma unroll
  for (int i = 12; i >= 0; --i) p = dadd(dmul(p, r), kExpC[i]);
  long long e = (long long)k + 1023;
  return dmul(p, __longlong_as_double(e << 52));
}

// oracle/rng.py exp32_np
__device__ __forceinline__ float exp32(float x) {
  if (x != x) return x;
  if (x < -87.0f) return 0.0f;
  if (x > 88.0f) return __int_as_float(0x7f800000);
  float k = rintf(fmul(x, kLog2ef));
  float r = fsub(fsub(x, fmul(k, kLn2Hif)), fmul(k, kLn2Lof));
  float p = kExpCf[8];
#pragma unroll
  for (int i = 7; i >= 0; --i) p = fadd(fmul(p, r), kExpCf[i]);
  int e = (int)k + 127;
  return fmul(p, __int_as_float(e << 23));
}

// oracle/rng.py log64 (finite u > 0, normal range)
__device__ __forceinline__ double log64(double u) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(u);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((long long)((bits & 0xfffffffffffffULL) | (1023ULL << 52)));
  if (m > kSqrt2) {
    m = dmul(m, 0.5);
    e += 1;
  }
  double f = dsub(m, 1.0);
  double s = __ddiv_rn(f, dadd(2.0, f));
  double z = dmul(s, s);
  double p = kLogC[11];
#pragma unroll
  for (int i = 10; i >= 0; --i) p = dadd(dmul(p, z), kLogC[i]);
  double logm = dmul(dadd(s, s), p);
  double ef = (double)e;
  return dadd(dmul(ef, kLn2Hi), dadd(dmul(ef, kLn2Lo), logm));
}

// oracle/rng.py log1p64
__device__ __forceinline__ double log1p64(double x) {
  double u = dadd(1.0, x);
  if (u == 1.0) return x;
  return dmul(log64(u), __ddiv_rn(x, dsub(u, 1.0)));
}

}  // namespace pfm
