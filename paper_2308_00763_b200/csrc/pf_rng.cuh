// pf_rng.cuh -- counter-based LCG stream + ziggurat normals (device).
//
// Stream (restated in oracle/rng.py):
//   x_0 = splitmix64(seed), x_{n+1} = A x_n + C (mod 2^64), word n = x_n.
//   Frame t of a K-particle track: normal (k, c) at position t(2K+1)+2k+c,
//   resampling uniform at t(2K+1)+2K.
// Any position is reachable in O(1) mul-adds from precomputed affine powers
// (byte-digit jump table in constant memory for the tile base, a per-thread
// table for the in-tile offset), so draws are a pure function of position:
// independent of TPB, tile order and GPU count.
#pragma once
#include <stdint.h>

#include "pf_math.cuh"
#include "ziggurat_tables.h"

namespace pfr {

constexpr uint64_t kA = 6364136223846793005ULL;
constexpr uint64_t kC = 1442695040888963407ULL;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMask52 = (1ULL << 52) - 1;
constexpr double kZigR = 0x1.d3bb48209ad33p+1;
constexpr double kZigInvR = 0x1.183aa6c20e8c1p-2;
constexpr double kTwoM53 = 1.0 / 9007199254740992.0;

struct Affine {
  uint64_t a, c;
};

__host__ __device__ __forceinline__ uint64_t apply(const Affine& f, uint64_t x) { return f.a * x + f.c; }
// g after f
__host__ __device__ __forceinline__ Affine compose(const Affine& g, const Affine& f) {
  return Affine{g.a * f.a, g.a * f.c + g.c};
}

__host__ __device__ __forceinline__ uint64_t splitmix64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t seed_state(uint64_t seed) { return splitmix64_mix(seed + kGolden); }

// host: f^n
inline Affine affine_pow(uint64_t n) {
  Affine r{1, 0}, b{kA, kC};
  while (n) {
    if (n & 1) r = compose(b, r);
    b = compose(b, b);
    n >>= 1;
  }
  return r;
}

// jump table: kJump[d][v] = f^(v * 256^d), d < 6 (positions < 2^48)
constexpr int kJumpDigits = 6;
__constant__ Affine kJump[kJumpDigits][256];

__device__ __forceinline__ uint64_t word_at(uint64_t x0, uint64_t pos) {
  // kJump[d][0] is the identity, so all six table loads are unconditional and
  // independent (one memory latency), followed by six dependent mul-adds.
  Affine f[kJumpDigits];
#pragma unroll
  for (int d = 0; d < kJumpDigits; ++d) f[d] = kJump[d][(pos >> (8 * d)) & 0xff];
  uint64_t x = x0;
#pragma unroll
  for (int d = 0; d < kJumpDigits; ++d) x = apply(f[d], x);
  return x;
}

__device__ __forceinline__ double uniform_of(uint64_t w) { return (double)(w >> 11) * kTwoM53; }

// Ziggurat slow path (oracle/rng.py _zig_slow_lcg): retry words from a
// splitmix64 sequence seeded with the primary word.
static __device__ __noinline__ double zig_slow(uint64_t r) {
  uint64_t s = r;
  for (;;) {
    unsigned idx = (unsigned)(r >> 56);
    unsigned sign = (unsigned)((r >> 55) & 1);
    uint64_t rabs = (r >> 3) & kMask52;
    double x = pfm::dmul((double)rabs, __longlong_as_double((long long)PF_ZIG_WI_BITS[idx]));
    if (sign) x = -x;
    if (rabs < PF_ZIG_KI[idx]) return x;
    if (idx == 0) {
      for (;;) {
        s += kGolden;
        double u1 = uniform_of(splitmix64_mix(s));
        s += kGolden;
        double u2 = uniform_of(splitmix64_mix(s));
        double xx = pfm::dmul(-kZigInvR, pfm::log1p64(-u1));
        double yy = -pfm::log1p64(-u2);
        if (pfm::dadd(yy, yy) > pfm::dmul(xx, xx)) return sign ? -pfm::dadd(kZigR, xx) : pfm::dadd(kZigR, xx);
      }
    } else {
      s += kGolden;
      double u = uniform_of(splitmix64_mix(s));
      double fi0 = __longlong_as_double((long long)PF_ZIG_FI_BITS[idx - 1]);
      double fi1 = __longlong_as_double((long long)PF_ZIG_FI_BITS[idx]);
      double lhs = pfm::dadd(pfm::dmul(pfm::dsub(fi0, fi1), u), fi1);
      if (lhs < pfm::exp64(pfm::dmul(pfm::dmul(-0.5, x), x))) return x;
    }
    s += kGolden;
    r = splitmix64_mix(s);
  }
}

// Fast path with shared-memory tables: ki_hi[idx] = KI[idx] >> 20, wi[idx].
__device__ __forceinline__ double normal_of(uint64_t w, const uint32_t* ki_hi, const double* wi) {
  unsigned idx = (unsigned)(w >> 56);
  uint64_t rabs = (w >> 3) & kMask52;
  unsigned rhi = (unsigned)(rabs >> 20);
  unsigned khi = ki_hi[idx];
  if (rhi < khi) {
    double x = pfm::dmul((double)rabs, wi[idx]);
    return ((w >> 55) & 1) ? -x : x;
  }
  return zig_slow(w);
}

// ---------------------------------------------------------------------------
// NumPy-compatible reference stream (Generator(Philox(seed)), filter.py:71-82):
// Philox4x64-10 with NumPy's counter semantics and glibc's log1p restated from
// its x86-64 FMA variant (oracle/rng.py log1p_glibc).  The stream itself is
// generated in parallel by pf_philox.cuh.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void philox_block(const unsigned long long ctr_in[4], const unsigned long long key_in[2],
                                             unsigned long long out[4]) {
  unsigned long long c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  unsigned long long k0 = key_in[0], k1 = key_in[1];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const unsigned long long lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const unsigned long long lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    const unsigned long long n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// glibc 2.39 log1p (x86-64 FMA variant), domain -1 < x <= 0.41422
static __device__ double log1p_glibc(double x) {
  const double L1 = 0x1.5555555555593p-1, L2 = 0x1.999999997fa04p-2, L3 = 0x1.2492494229359p-2;
  const double L4 = 0x1.c71c51d8e78afp-3, L5 = 0x1.7466496cb03dep-3, L6 = 0x1.39a09d078c69fp-3;
  const double L7 = 0x1.2f112df3e5244p-3, LN2_LO = 0x1.a39ef35793c76p-33, LN2_HI = 0x1.62e42fee00000p-1;
  const double C23 = 0x1.5555555555555p-1;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  if (ax <= 0x3e1fffff) {
    if (ax <= 0x3c8fffff) return x;
    return __fma_rn(-__dmul_rn(x, x), 0.5, x);
  }
  double c = 0.0, f;
  int k, hu;
  if ((unsigned)(hx + 0x402d413c) > 0x402d413cu) {
    k = 0;
    f = x;
    hu = 1;
  } else {
    double u = __dadd_rn(1.0, x);
    hu = __double2hiint(u);
    k = (hu >> 20) - 1023;
    c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
    c = __ddiv_rn(c, u);
    hu &= 0xfffff;
    const int lo = __double2loint(u);
    if (hu > 0x6a09d) {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, lo);
      hu = (0x100000 - hu) >> 2;
    } else {
      u = __hiloint2double(hu | 0x3ff00000, lo);
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
  const double kf = (double)k;
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : __fma_rn(kf, LN2_HI, __fma_rn(kf, LN2_LO, c));
    const double R = __dmul_rn(__fma_rn(-f, C23, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(kf, LN2_HI, -__dsub_rn(__dsub_rn(R, __fma_rn(kf, LN2_LO, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
  const double z = __dmul_rn(s, s);
  const double t11 = __fma_rn(z, L3, L2), t10 = __fma_rn(z, L5, L4), t9 = __fma_rn(z, L7, L6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  const double R = __fma_rn(z6, t9, __fma_rn(z4, t10, __fma_rn(z, L1, __dmul_rn(z2, t11))));
  const double t = __dmul_rn(__dadd_rn(R, hfsq), s);
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  const double klo = __fma_rn(kf, LN2_LO, c);
  return __fma_rn(kf, LN2_HI, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(klo, t)), f));
}

}  // namespace pfr
