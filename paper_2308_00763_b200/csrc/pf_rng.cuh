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
__device__ __noinline__ double zig_slow(uint64_t r) {
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

}  // namespace pfr
