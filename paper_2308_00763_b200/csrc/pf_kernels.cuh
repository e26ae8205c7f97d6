// pf_kernels.cuh -- sm_100a kernels of the per-frame particle-filter step.
//
//   pf_map_wide / pf_map_half : per-frame likelihood map L(ix, iy) over the
//       extended grid [-r, W-1+r] x [-r, H-1+r]; frame rows staged in shared
//       memory by one cp.async.bulk (TMA bulk copy), template offsets in
//       shared memory.  Bit-identical to the reference likelihood
//       (filter.py:204-217 wide, 384-423 binary16) because L depends only on
//       the clamped rounded position and the per-pixel sum order is NumPy's.
//   pf_fused_frame<MODE, VPT> : one CTA per 1024-particle tile: systematic
//       resampling against the previous frame's hierarchical CDF, 128/64/32-bit
//       ancestor gathers, LCG normals, propagation (filter.py:195-202 /
//       346-382), map lookup, tile max, exact fixed-point weight scan, rescaled
//       local CDF, position moments.  One launch per frame.
//   pf_tile_table<MODE> : one CTA per track: global max, exact int64 prefix of
//       tile masses, normalised tile offsets, per-tile first output index,
//       estimate (filter.py:241-246) and degeneracy check (filter.py:228-230).
// oracle/fused.py restates all three; tests check the CUDA path bit-exactly.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "pf_math.cuh"
#include "pf_rng.cuh"

#include <type_traits>

#define PF_TILE 1024
#define PF_MAX_SHARDS 8
#ifndef PF_FULL_SPEC
#define PF_FULL_SPEC 1  // full-tile threads take a bounds-free phase-1 path
#endif
#define PF_XQ_BITS 10

#include <climits>

namespace pfk {

enum { M_FP64 = 0, M_FP32 = 1, M_FP16 = 2 };

template <int MODE>
struct Tr;
template <>
struct Tr<M_FP64> {
  using real = double;
  using vec = double2;
  using wq_t = long long;
  static constexpr int FB = 52;
};
template <>
struct Tr<M_FP32> {
  using real = float;
  using vec = float2;
  using wq_t = long long;
  static constexpr int FB = 40;
};
template <>
struct Tr<M_FP16> {
  using real = __half;
  using vec = __half2;
  using wq_t = int;
  static constexpr int FB = 20;
};

__device__ __forceinline__ double to_d(double v) { return v; }
__device__ __forceinline__ double to_d(float v) { return (double)v; }
__device__ __forceinline__ double to_d(__half v) { return (double)__half2float(v); }

// "naive" binary16 ops of the scalar-lane kernels: half storage, f32 compute,
// every result rounded back to binary16 -- RN16(RN32(a op b)) == RN16(a op b)
// for + and * (24 >= 2*11 + 2 bits: double rounding is innocuous), so values
// equal the native half2 path.  (Scalar add.rn.f16 was tried first: ptxas
// re-pairs adjacent lanes into one HADD2 -- measured in the SASS.)
__device__ __forceinline__ __half hadd_s(__half a, __half b) {
  return __float2half_rn(__fadd_rn(__half2float(a), __half2float(b)));
}
__device__ __forceinline__ __half hmul_s(__half a, __half b) {
  return __float2half_rn(__fmul_rn(__half2float(a), __half2float(b)));
}
__device__ __forceinline__ __half hsub_s(__half a, __half b) {
  return __float2half_rn(__fsub_rn(__half2float(a), __half2float(b)));
}
// The naive kernel's per-particle re-derivation of shared constants (the
// reference's naive FP16 path, filter.py:482-490,535-541, and the paper's
// un-optimised resampling kernel): casts and reciprocals are
// issued for every particle instead of once per tile.  `asm volatile` keeps
// the compiler from hoisting them; the values are those of the hoisted forms.
__device__ __forceinline__ float cvt_f32_f64_naive(double d) {
  float f;
  asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(d));
  return f;
}
__device__ __forceinline__ float rcp_f32_s64_naive(long long S) {
  float s, r;
  asm volatile("cvt.rn.f32.s64 %0, %1;" : "=f"(s) : "l"(S));
  asm volatile("div.rn.f32 %0, 0f3F800000, %1;" : "=f"(r) : "f"(s));
  return r;
}
// ------------------------------------------------------------------------
// TMA bulk copy helpers (cp.async.bulk + mbarrier)
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// Programmatic dependent launch: let the next kernel in the stream start
// early, and wait for the previous kernel's results only where they are
// consumed (no-ops when launched without the PDL attribute).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void bulk_load_rows(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  uint32_t b = smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(b)
      : "memory");
}

// ------------------------------------------------------------------------
// likelihood maps
// ------------------------------------------------------------------------
struct MapArgs {
  const uint8_t* frames;  // [n_videos][F][H][W]
  int n_frames;           // frames per video in this buffer
  int H, W, r, Hm, Wm;
  int n_off;
  const int2* offsets;    // device, template order
  const short* plan;      // pairwise plan ops (wide); leaf index >= 0, -1 = combine
  const short2* leaves;   // (start, len)
  int n_plan;
  double bg, fg, denom;   // wide params (cast to real in-kernel)
  unsigned short bg16, fg16, s16;  // binary16 constants
  void* maps;             // [n_videos][F][Hm][Wm]
  int band;               // map rows per CTA
  const int2* runs;       // pf_map_wide_runs: per horizontal run, row-prefix displacements (end, start)
  int n_runs;
};

// NumPy pairwise_sum leaf (n <= 128): 8 accumulators, then tail.
template <typename real>
__device__ __forceinline__ real pw_leaf(const real* t, int n) {
  if (n < 8) {
    real res = (real)0;
    for (int i = 0; i < n; ++i) res = res + t[i];
    return res;
  }
  real r0 = t[0], r1 = t[1], r2 = t[2], r3 = t[3], r4 = t[4], r5 = t[5], r6 = t[6], r7 = t[7];
  int i = 8;
  int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    r0 = r0 + t[i + 0];
    r1 = r1 + t[i + 1];
    r2 = r2 + t[i + 2];
    r3 = r3 + t[i + 3];
    r4 = r4 + t[i + 4];
    r5 = r5 + t[i + 5];
    r6 = r6 + t[i + 6];
    r7 = r7 + t[i + 7];
  }
  real res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res = res + t[i];
  return res;
}

template <typename real>
__device__ __forceinline__ real term_wide(int v, real bg, real fg) {
  real x = (real)v;
  real a = x - bg;
  real b = x - fg;
  return a * a - b * b;  // -fmad=false: separately rounded
}

template <typename real>
__global__ void pf_map_wide(MapArgs a) {
  pdl_launch_dependents();  // a one-frame step's fused kernel may start its draws (it waits for the map)
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  real* term = reinterpret_cast<real*>(smem + 16);
  int2* offs = reinterpret_cast<int2*>(smem + 16 + 256 * sizeof(real));
  short* plan = reinterpret_cast<short*>(offs + a.n_off);
  short2* leaves = reinterpret_cast<short2*>(plan + ((a.n_plan + 1) & ~1));
  // byte offsets from the shared base (a uintptr_t round trip would hide the
  // address space: generic loads instead of LDS)
  uint8_t* rows = smem + ((reinterpret_cast<unsigned char*>(leaves + a.n_plan) - smem + 15) & ~15);

  const int vf = blockIdx.y;  // video * n_frames + frame
  const int my0 = blockIdx.x * a.band;
  const int my1 = min(a.Hm, my0 + a.band);
  const int R0 = max(0, my0 - 2 * a.r);
  const int R1 = min(a.H - 1, my1 - 1);
  const uint8_t* frame = a.frames + (size_t)vf * a.H * a.W;

  real bg = (real)a.bg, fg = (real)a.fg;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) term[i] = term_wide<real>(i, bg, fg);
  for (int i = threadIdx.x; i < a.n_off; i += blockDim.x) offs[i] = a.offsets[i];
  for (int i = threadIdx.x; i < a.n_plan; i += blockDim.x) {
    plan[i] = a.plan[i];
    leaves[i] = a.leaves[i];
  }
  const int nrows = R1 >= R0 ? R1 - R0 + 1 : 0;
  const uint32_t bytes = (uint32_t)nrows * (uint32_t)a.W;
  const uint8_t* src = frame + (size_t)R0 * a.W;
  if (nrows > 0 && ((uintptr_t)src % 16 == 0) && (bytes % 16 == 0)) {
    bulk_load_rows(rows, src, bytes, bar);  // includes a __syncthreads
  } else {
    for (uint32_t i = threadIdx.x; i < bytes; i += blockDim.x) rows[i] = src[i];
  }
  __syncthreads();

  real* out = reinterpret_cast<real*>(a.maps) + (size_t)vf * a.Hm * a.Wm;
  const real denom = (real)a.denom;
  real t[128];
  for (int e = threadIdx.x; e < (my1 - my0) * a.Wm; e += blockDim.x) {
    const int my = my0 + e / a.Wm, mx = e % a.Wm;
    const int iy = my - a.r, ix = mx - a.r;
    // evaluate the pairwise plan
    real stack[12];
    int sp = 0;
    for (int pi = 0; pi < a.n_plan; ++pi) {
      short op = plan[pi];
      if (op >= 0) {
        short2 lf = leaves[op];
        for (int j = 0; j < lf.y; ++j) {
          int2 o = offs[lf.x + j];
          int yy = min(max(iy + o.y, 0), a.H - 1);
          int xx = min(max(ix + o.x, 0), a.W - 1);
          t[j] = term[rows[(yy - R0) * a.W + xx]];
        }
        stack[sp++] = pw_leaf<real>(t, lf.y);
      } else {
        real b2 = stack[--sp];
        real b1 = stack[--sp];
        stack[sp++] = b1 + b2;
      }
    }
    out[(size_t)my * a.Wm + mx] = stack[0] / denom;
  }
}

// FP32 / FP64 map through a padded term image (templates of <= 128 offsets:
// one NumPy pairwise leaf).  The CTA expands its band of clamped source rows
// once into term values (rows my0-2r .. my1-1, columns -2r .. W+2r-1 with
// replicated edges), so every tap is one shared load at a per-offset
// constant displacement and one add -- no clamps, no byte-then-term double
// lookup, no local-memory term array (pf_map_wide).  Two map entries per
// thread share each displacement load.  Same pairwise order, same sums.
struct MapWideGeom {
  int band, Wp, rows;
  size_t smem;
};
__host__ __device__ inline MapWideGeom map_wide_geom(int W, int r, int n_off, int rs, int band) {
  MapWideGeom g;
  g.band = band;
  g.Wp = W + 4 * r;
  g.rows = band + 2 * r;
  g.smem = 256 * (size_t)rs + (((size_t)n_off * 4 + 15) & ~(size_t)15) + (size_t)g.rows * g.Wp * rs;
  return g;
}
constexpr int kMapWideThreads = 256;

template <typename real>
__device__ __forceinline__ void leaf_pair(const real* b0, const real* b1, const int* toff, int n, real& s0,
                                          real& s1) {
  if (n < 8) {
    s0 = (real)0;
    s1 = (real)0;
    for (int j = 0; j < n; ++j) {
      const int o = toff[j];
      s0 = s0 + b0[o];
      s1 = s1 + b1[o];
    }
    return;
  }
  real r0[8], r1[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int o = toff[q];
    r0[q] = b0[o];
    r1[q] = b1[o];
  }
  int j = 8;
  const int lim = n - (n % 8);
  for (; j < lim; j += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int o = toff[j + q];
      r0[q] = r0[q] + b0[o];
      r1[q] = r1[q] + b1[o];
    }
  }
  s0 = ((r0[0] + r0[1]) + (r0[2] + r0[3])) + ((r0[4] + r0[5]) + (r0[6] + r0[7]));
  s1 = ((r1[0] + r1[1]) + (r1[2] + r1[3])) + ((r1[4] + r1[5]) + (r1[6] + r1[7]));
  for (; j < n; ++j) {
    const int o = toff[j];
    s0 = s0 + b0[o];
    s1 = s1 + b1[o];
  }
}

template <typename real>
__global__ void __launch_bounds__(1024) pf_map_wide_img(MapArgs a) {
  pdl_launch_dependents();  // a one-frame step's fused kernel may start its draws (it waits for the map)
  extern __shared__ __align__(16) unsigned char smem[];
  const MapWideGeom g = map_wide_geom(a.W, a.r, a.n_off, (int)sizeof(real), a.band);
  real* term = reinterpret_cast<real*>(smem);
  int* toff = reinterpret_cast<int*>(term + 256);
  real* img = reinterpret_cast<real*>(reinterpret_cast<unsigned char*>(toff) + (((size_t)a.n_off * 4 + 15) & ~(size_t)15));
  const int vf = blockIdx.y;
  const int my0 = blockIdx.x * g.band;
  const int my1 = min(a.Hm, my0 + g.band);
  const int r = a.r;
  const uint8_t* frame = a.frames + (size_t)vf * a.H * a.W;
  const real bg = (real)a.bg, fg = (real)a.fg;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) term[i] = term_wide<real>(i, bg, fg);
  for (int i = threadIdx.x; i < a.n_off; i += blockDim.x) {
    const int2 o = a.offsets[i];
    toff[i] = (o.y + r) * g.Wp + o.x + r;
  }
  __syncthreads();
  const int nrow = (my1 - my0) + 2 * r;
  for (int e = threadIdx.x; e < nrow * g.Wp; e += blockDim.x) {
    const int ry = e / g.Wp, cx = e - ry * g.Wp;
    const int yy = min(max(my0 - 2 * r + ry, 0), a.H - 1);
    const int xx = min(max(cx - 2 * r, 0), a.W - 1);
    img[e] = term[__ldg(frame + (size_t)yy * a.W + xx)];
  }
  __syncthreads();
  real* out = reinterpret_cast<real*>(a.maps) + (size_t)vf * a.Hm * a.Wm;
  const real denom = (real)a.denom;
  const int n_e = (my1 - my0) * a.Wm;
  for (int e0 = threadIdx.x; e0 < n_e; e0 += 2 * blockDim.x) {
    const int e1 = min(e0 + (int)blockDim.x, n_e - 1);  // duplicate the last entry when odd
    const int y0 = e0 / a.Wm, x0 = e0 - y0 * a.Wm;
    const int y1 = e1 / a.Wm, x1 = e1 - y1 * a.Wm;
    real s0, s1;
    leaf_pair<real>(img + y0 * g.Wp + x0, img + y1 * g.Wp + x1, toff, a.n_off, s0, s1);
    out[(size_t)(my0 + y0) * a.Wm + x0] = s0 / denom;
    if (e0 + (int)blockDim.x < n_e) out[(size_t)(my0 + y1) * a.Wm + x1] = s1 / denom;
  }
}

// FP32 / FP64 map from integer row prefix sums.  With integral background /
// foreground means every term (v-bg)^2 - (v-fg)^2 is an integer and, when
// N * max|term| < 2^24, every partial sum of the reference's pairwise order
// is exact in FP32 and FP64 -- the sum is the same integer in any order
// (SURVEY 8a a7).  The CTA builds int32 term rows for its band, prefix-sums
// each row (one warp per row), and evaluates the template as horizontal runs
// (dy, dx0..dx1): two shared loads per run instead of one per offset (the
// r = 5 disk: 11 runs for 81 offsets).  The host picks this kernel only when
// the exactness conditions hold (pf_api.cu), else pf_map_wide_img.
struct MapRunsGeom {
  int band, Wz, rows;
  size_t smem;
};
__host__ __device__ inline MapRunsGeom map_runs_geom(int W, int r, int n_runs, int band) {
  MapRunsGeom g;
  g.band = band;
  g.Wz = W + 4 * r + 1;
  g.rows = band + 2 * r;
  g.smem = 256 * 4 + (size_t)n_runs * 8 + (size_t)g.rows * g.Wz * 4;
  return g;
}

template <typename real>
__global__ void __launch_bounds__(1024) pf_map_wide_runs(MapArgs a) {
  pdl_launch_dependents();  // a one-frame step's fused kernel may start its draws (it waits for the map)
  extern __shared__ __align__(16) unsigned char smem[];
  const MapRunsGeom g = map_runs_geom(a.W, a.r, a.n_runs, a.band);
  int* term = reinterpret_cast<int*>(smem);
  int2* runs = reinterpret_cast<int2*>(term + 256);
  int* pz = reinterpret_cast<int*>(runs + a.n_runs);
  const int vf = blockIdx.y;
  const int my0 = blockIdx.x * g.band;
  const int my1 = min(a.Hm, my0 + g.band);
  const int r = a.r;
  const uint8_t* frame = a.frames + (size_t)vf * a.H * a.W;
  const int ibg = (int)a.bg, ifg = (int)a.fg;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) term[i] = (i - ibg) * (i - ibg) - (i - ifg) * (i - ifg);
  for (int i = threadIdx.x; i < a.n_runs; i += blockDim.x) runs[i] = a.runs[i];
  __syncthreads();
  const int nrow = (my1 - my0) + 2 * r, Wp = g.Wz - 1;
  for (int e = threadIdx.x; e < nrow * Wp; e += blockDim.x) {
    const int ry = e / Wp, cx = e - ry * Wp;
    const int yy = min(max(my0 - 2 * r + ry, 0), a.H - 1);
    const int xx = min(max(cx - 2 * r, 0), a.W - 1);
    pz[ry * g.Wz + cx + 1] = term[__ldg(frame + (size_t)yy * a.W + xx)];
  }
  __syncthreads();
  {  // inclusive prefix sum of every row, one warp per row
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int ry = wid; ry < nrow; ry += nw) {
      int* row = pz + ry * g.Wz;
      int carry = 0;
      for (int c0 = 1; c0 < g.Wz; c0 += 32) {
        const int c = c0 + lane;
        int v = c < g.Wz ? row[c] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += t;
        }
        v += carry;
        if (c < g.Wz) row[c] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
      }
      if (lane == 0) row[0] = 0;
    }
  }
  __syncthreads();
  real* out = reinterpret_cast<real*>(a.maps) + (size_t)vf * a.Hm * a.Wm;
  const real denom = (real)a.denom;
  const int n_e = (my1 - my0) * a.Wm;
  for (int e0 = threadIdx.x; e0 < n_e; e0 += 2 * blockDim.x) {
    const int e1 = min(e0 + (int)blockDim.x, n_e - 1);
    const int y0 = e0 / a.Wm, x0 = e0 - y0 * a.Wm;
    const int y1 = e1 / a.Wm, x1 = e1 - y1 * a.Wm;
    const int* b0 = pz + y0 * g.Wz + x0;
    const int* b1 = pz + y1 * g.Wz + x1;
    int s0 = 0, s1 = 0;
    for (int j = 0; j < a.n_runs; ++j) {
      const int2 d = runs[j];
      s0 += b0[d.x] - b0[d.y];
      s1 += b1[d.x] - b1[d.y];
    }
    out[(size_t)(my0 + y0) * a.Wm + x0] = (real)s0 / denom;
    if (e0 + (int)blockDim.x < n_e) out[(size_t)(my0 + y1) * a.Wm + x1] = (real)s1 / denom;
  }
}

// binary16: term16 table per intensity (model.half_term_stabilized, 7 RN16
// ops), sequential RN16 fold in template order from +0; two adjacent map
// entries per thread in one half2.
#ifndef PF_FUSED_ONLY  // launched from pf_api.cu only
__global__ void pf_map_half(MapArgs a) {
  pdl_launch_dependents();  // a one-frame step's fused kernel may start its draws (it waits for the map)
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  __half* term = reinterpret_cast<__half*>(smem + 16);
  int2* offs = reinterpret_cast<int2*>(smem + 16 + 256 * sizeof(__half));
  uint8_t* rows = smem + ((reinterpret_cast<unsigned char*>(offs + a.n_off) - smem + 15) & ~15);

  const int vf = blockIdx.y;
  const int my0 = blockIdx.x * a.band;
  const int my1 = min(a.Hm, my0 + a.band);
  const int R0 = max(0, my0 - 2 * a.r);
  const int R1 = min(a.H - 1, my1 - 1);
  const uint8_t* frame = a.frames + (size_t)vf * a.H * a.W;

  const __half bg = __ushort_as_half(a.bg16), fg = __ushort_as_half(a.fg16), s = __ushort_as_half(a.s16);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    __half v = __int2half_rn(i);
    __half x = __hmul_rn(__hsub_rn(v, bg), s);
    __half x2 = __hmul_rn(x, x);
    __half y = __hmul_rn(__hsub_rn(v, fg), s);
    __half y2 = __hmul_rn(y, y);
    term[i] = __hsub_rn(x2, y2);
  }
  for (int i = threadIdx.x; i < a.n_off; i += blockDim.x) offs[i] = a.offsets[i];
  const int nrows = R1 >= R0 ? R1 - R0 + 1 : 0;
  const uint32_t bytes = (uint32_t)nrows * (uint32_t)a.W;
  const uint8_t* src = frame + (size_t)R0 * a.W;
  if (nrows > 0 && ((uintptr_t)src % 16 == 0) && (bytes % 16 == 0)) {
    bulk_load_rows(rows, src, bytes, bar);
  } else {
    for (uint32_t i = threadIdx.x; i < bytes; i += blockDim.x) rows[i] = src[i];
  }
  __syncthreads();

  __half* out = reinterpret_cast<__half*>(a.maps) + (size_t)vf * a.Hm * a.Wm;
  const int pairs_per_row = (a.Wm + 1) / 2;
  for (int e = threadIdx.x; e < (my1 - my0) * pairs_per_row; e += blockDim.x) {
    const int my = my0 + e / pairs_per_row;
    const int mx0 = 2 * (e % pairs_per_row);
    const int mx1 = min(mx0 + 1, a.Wm - 1);
    const int iy = my - a.r;
    const int ix0 = mx0 - a.r, ix1 = mx1 - a.r;
    __half2 acc = __float2half2_rn(0.0f);
    for (int j = 0; j < a.n_off; ++j) {
      int2 o = offs[j];
      int yy = min(max(iy + o.y, 0), a.H - 1);
      const uint8_t* row = rows + (yy - R0) * a.W;
      int x0 = min(max(ix0 + o.x, 0), a.W - 1);
      int x1 = min(max(ix1 + o.x, 0), a.W - 1);
      acc = __hadd2_rn(acc, __halves2half2(term[row[x0]], term[row[x1]]));
    }
    out[(size_t)my * a.Wm + mx0] = __low2half(acc);
    if (mx1 != mx0) out[(size_t)my * a.Wm + mx1] = __high2half(acc);
  }
}
#endif

// binary16 map, term-image formulation (used when its shared memory fits):
// the CTA's band of map rows reads a padded image T[py][px] = term16(frame
// pixel, edge-clamped) held twice -- A and B = A shifted by one half -- so
// every tap of every entry pair is ONE aligned 32-bit shared load (A for even,
// B for odd tap offsets, a warp-uniform choice) feeding one HADD2: per entry
// pair and tap, LDS + IADD + HADD2 instead of two clamped pixel and term
// lookups.  Same per-entry fold (template order from +0, each add RN16), so
// the map is bit-identical to pf_map_half.
constexpr int kMapHalfThreads = 512;
constexpr int kMapHalfPairs = 8;  // entry pairs per thread (<= 4096 per CTA)
struct MapHalfGeom {
  int band, P, rows_img;  // map rows per CTA, image pitch (halves, even), image rows
  size_t smem;            // dynamic shared memory bytes
};
// band_cap > 0 limits the map rows per CTA (few frames: more, shorter CTAs)
__host__ __device__ inline MapHalfGeom map_half_geom(int W, int H, int r, int n_off, int band_cap = 0) {
  MapHalfGeom g;
  const int Wm = W + 2 * r, Hm = H + 2 * r, npr = (Wm + 1) / 2;
  g.band = max(1, min(Hm, kMapHalfThreads * kMapHalfPairs / npr));
  if (band_cap > 0) g.band = min(g.band, band_cap);
  g.P = (Wm + 2 * r + 2) & ~1;
  g.rows_img = g.band + 2 * r;
  const size_t frame_rows = (size_t)(g.band + 2 * r) * W + 32;
  g.smem = 16 + 256 * 2 + (size_t)n_off * 4 + 16 + ((frame_rows + 15) & ~(size_t)15) + (size_t)2 * g.rows_img * g.P * 2;
  return g;
}

template <bool PK>  // PK: one HADD2 per entry pair and tap; else two scalar HADDs (same values)
__global__ void __launch_bounds__(kMapHalfThreads) pf_map_half_img(MapArgs a) {
  pdl_launch_dependents();  // a one-frame step's fused kernel may start its draws (it waits for the map)
  extern __shared__ __align__(16) unsigned char smem[];
  const MapHalfGeom g = map_half_geom(a.W, a.H, a.r, a.n_off, a.band);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  __half* term = reinterpret_cast<__half*>(smem + 16);
  int* tapw = reinterpret_cast<int*>(smem + 16 + 512);
  uint8_t* rows = smem + ((reinterpret_cast<unsigned char*>(tapw + a.n_off) - smem + 15) & ~15);
  const size_t frame_rows = (size_t)(g.band + 2 * a.r) * a.W + 32;
  __half* imgA = reinterpret_cast<__half*>(rows + ((frame_rows + 15) & ~(size_t)15));
  __half* imgB = imgA + (size_t)g.rows_img * g.P;
  const unsigned* wA = reinterpret_cast<const unsigned*>(imgA);

  const int vf = blockIdx.y;
  const int my0 = blockIdx.x * g.band;
  const int my1 = min(a.Hm, my0 + g.band);
  const int R0 = max(0, my0 - 2 * a.r);
  const int R1 = min(a.H - 1, my1 - 1);
  const uint8_t* frame = a.frames + (size_t)vf * a.H * a.W;

  const __half bg = __ushort_as_half(a.bg16), fg = __ushort_as_half(a.fg16), s = __ushort_as_half(a.s16);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {  // model.half_term_stabilized, 7 RN16 ops
    __half v = __int2half_rn(i);
    __half x = __hmul_rn(__hsub_rn(v, bg), s);
    __half x2 = __hmul_rn(x, x);
    __half y = __hmul_rn(__hsub_rn(v, fg), s);
    __half y2 = __hmul_rn(y, y);
    term[i] = __hsub_rn(x2, y2);
  }
  // tap offsets in 32-bit words from imgA: (dy + r) * P + (dx + r) halves,
  // odd offsets read B (its word w holds A halves 2w + 1, 2w + 2)
  const int bwords = g.rows_img * g.P / 2;
  for (int j = threadIdx.x; j < a.n_off; j += blockDim.x) {
    const int2 o = a.offsets[j];
    const int t = (o.y + a.r) * g.P + (o.x + a.r);
    tapw[j] = (t >> 1) + ((t & 1) ? bwords : 0);
  }
  const int nrows = R1 >= R0 ? R1 - R0 + 1 : 0;
  const uint32_t bytes = (uint32_t)nrows * (uint32_t)a.W;
  const uint8_t* src = frame + (size_t)R0 * a.W;
  if (nrows > 0 && ((uintptr_t)src % 16 == 0) && (bytes % 16 == 0)) {
    bulk_load_rows(rows, src, bytes, bar);
  } else {
    for (uint32_t i = threadIdx.x; i < bytes; i += blockDim.x) rows[i] = src[i];
  }
  __syncthreads();
  // padded term images: row py <-> frame row clamp(my0 + py - 2r), column px <-> clamp(px - 2r)
  for (int i = threadIdx.x; i < g.rows_img * g.P; i += blockDim.x) {
    const int py = i / g.P, px = i - py * g.P;
    const int y = min(max(my0 + py - 2 * a.r, 0), a.H - 1);
    const uint8_t* row = rows + (max(y, R0) - R0) * a.W;
    const int x0 = min(max(px - 2 * a.r, 0), a.W - 1), x1 = min(max(px + 1 - 2 * a.r, 0), a.W - 1);
    imgA[i] = term[row[x0]];
    imgB[i] = term[row[x1]];
  }
  __syncthreads();

  const int npr = (a.Wm + 1) / 2, npairs = (my1 - my0) * npr;
  // pair slots in use by this CTA (a narrow band -- one-frame steps -- fills
  // only the first; the others are skipped, not computed on clamped indices)
  const int kmax = min(kMapHalfPairs, (npairs + kMapHalfThreads - 1) / kMapHalfThreads);
  int base[kMapHalfPairs];
  __half2 acc[kMapHalfPairs];
#pragma unroll
  for (int k = 0; k < kMapHalfPairs; ++k) {
    const int p = min(threadIdx.x + k * kMapHalfThreads, max(npairs - 1, 0));
    const int row = p / npr, x2 = p - row * npr;
    base[k] = row * (g.P / 2) + x2;
    acc[k] = __float2half2_rn(0.0f);
  }
  auto taps = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    for (int j = 0; j < a.n_off; ++j) {
      const int tw = tapw[j];
#pragma unroll
      for (int k = 0; k < kMapHalfPairs; ++k) {
        if (!FULL && k >= kmax) break;
        const unsigned v = wA[base[k] + tw];
        const __half2 tv = *reinterpret_cast<const __half2*>(&v);
        if constexpr (PK)
          acc[k] = __hadd2_rn(acc[k], tv);
        else
          acc[k] = __halves2half2(hadd_s(__low2half(acc[k]), __low2half(tv)), hadd_s(__high2half(acc[k]), __high2half(tv)));
      }
    }
  };
  if (kmax == kMapHalfPairs)  // every pair slot in use (multi-frame maps): no per-slot test
    taps(std::true_type{});
  else
    taps(std::false_type{});
  __half* out = reinterpret_cast<__half*>(a.maps) + (size_t)vf * a.Hm * a.Wm;
#pragma unroll
  for (int k = 0; k < kMapHalfPairs; ++k) {
    const int p = threadIdx.x + k * kMapHalfThreads;
    if (p < npairs) {
      const int row = p / npr, mx = 2 * (p - row * npr);
      const size_t o = (size_t)(my0 + row) * a.Wm + mx;
      out[o] = __low2half(acc[k]);
      if (mx + 1 < a.Wm) out[o + 1] = __high2half(acc[k]);
    }
  }
}

// ------------------------------------------------------------------------
// systematic points (per-mode formula; identical in the table kernel)
// ------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ double point_of(long long k, double u, long long K, double invK) {
  if (MODE == M_FP64) return __ddiv_rn(__dadd_rn(__ll2double_rn(k), u), __ll2double_rn(K));
  if (MODE == M_FP32) {
    float p = __fdiv_rn(__fadd_rn(__ll2float_rn(k), __double2float_rn(u)), __ll2float_rn(K));
    return (double)p;
  }
  return __dmul_rn(__dadd_rn(__ll2double_rn(k), u), invK);
}

// ------------------------------------------------------------------------
// fused frame kernel
// ------------------------------------------------------------------------
// Source tiles of a frame's resampling may live on other shards of a
// sharded filter: every source-tile access goes through the
// per-shard base pointers below (peer-mapped over NVLink, or the handle's own
// buffers when unsharded, n_shards == 1).
struct SrcShards {
  int n_shards;     // 1 = unsharded
  int shard_tiles;  // tiles per shard (all but the last shard are full)
  const void* X[PF_MAX_SHARDS];  // previous-frame positions
  const void* C[PF_MAX_SHARDS];  // previous-frame local CDFs
  const long long* ts[PF_MAX_SHARDS];
  const double* tO[PF_MAX_SHARDS];
  const double* tM[PF_MAX_SHARDS];
};

struct FusedArgs {
  long long K;        // particles per track (global, over all shards)
  int n_tiles;        // tiles per track (global)
  long long K_local;  // particles per track held by this handle
  int n_local;        // tiles per track held by this handle
  int tile0;          // global index of this handle's first tile
  SrcShards src;
  int H, W, r, Wm;
  int t;      // frame index in the stream (RNG position)
  int ident;  // identity ancestors: frame 0, or a state injected by pf_set_state (no previous table)
  void* X_new;
  void* C_new;
  const double* u_prev;
  const void* map;             // map of video 0 for this frame
  long long map_video_stride;  // elements
  int n_videos;
  const unsigned long long* x0;
  const ulonglong2* tj;  // f^(2 v VPT) per virtual thread v
  double* rec_m;
  long long* rec_S;
  long long* rec_X;  // fp16: int64 moments; wide: double bits
  long long* rec_Y;
  const unsigned short* exp16;
  const int* exp16q;  // FP16 fixed-point weights: rint(exp16[d] * 2^20) per binary16 pattern d
  double drift_x, drift_y, std_x, std_y;
  long long* dbg_anc;  // optional
  void* dbg_L;         // optional
  const void* zig;     // packed ziggurat fast-path tables: ki>>20 (u32 x 256) then wi (f64 x 256)
  unsigned long long fa, fc;  // f^(t(2K+1)): frame base state = fa * x0[track] + fc
  const ulonglong2* tt;       // per tile: f^(2 * tile * PF_TILE)
  const void* win;            // [track][tile] int2: first / last source tile (tile table of the previous frame)
  unsigned long long* tmax;   // per track (stride 4): [0] order key of the running max of the tile maxima,
                              //   [1] table-ready counter (+1 per table chunk and frame)
  unsigned long long ready_target;  // frame t > 0 proceeds once tmax[1] >= this (n_chunks * t)
  int wait_prev;                    // launched behind the map kernel (PDL): grid-dependency wait before the map reads
  unsigned long long* trace;  // optional: [tile][8] %globaltimer stamps (track 0)
  const double2* noise;       // NZ variants: this frame's draws (n, d) per particle (the reference's
                              //   own stream, generated by pf_philox.cuh), one track
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PF_TRACE(A, SLOT)                                                   \
  do {                                                                      \
    if ((A).trace != nullptr && threadIdx.x == 0 && blockIdx.y == 0)        \
      (A).trace[(size_t)blockIdx.x * 8 + (SLOT)] = gtimer();                \
  } while (0)
#define PF_TRACE_DBG(A, SLOT)   \
  do {                          \
    if constexpr (DBG) PF_TRACE(A, SLOT); \
  } while (0)

// order-preserving map double -> uint64 (for atomicMax); 0 is below every key
__device__ __forceinline__ unsigned long long okey(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)b);
}

template <typename T>
__device__ __forceinline__ T shfl_up(T v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* warp_buf, T* total) {
  // inclusive warp scan
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = shfl_up(x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_buf[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? warp_buf[lane] : (T)0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T y = shfl_up(w, d);
      if (lane >= d) w += y;
    }
    if (lane < nw) warp_buf[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  T base = wid ? warp_buf[wid - 1] : (T)0;
  *total = warp_buf[nw - 1];
  __syncthreads();
  return base + x - v;
}

template <int MODE>
__device__ __forceinline__ typename Tr<MODE>::vec propagate_one(typename Tr<MODE>::vec xa, double n0, double n1,
                                                                 const FusedArgs& a);

template <>
__device__ __forceinline__ double2 propagate_one<M_FP64>(double2 xa, double n0, double n1, const FusedArgs& a) {
  double2 o;
  o.x = __dadd_rn(__dadd_rn(xa.x, a.drift_x), __dmul_rn(a.std_x, n0));
  o.y = __dadd_rn(__dadd_rn(xa.y, a.drift_y), __dmul_rn(a.std_y, n1));
  return o;
}
template <>
__device__ __forceinline__ float2 propagate_one<M_FP32>(float2 xa, double n0, double n1, const FusedArgs& a) {
  float2 o;
  o.x = __fadd_rn(__fadd_rn(xa.x, __double2float_rn(a.drift_x)),
                  __fmul_rn(__double2float_rn(a.std_x), __double2float_rn(n0)));
  o.y = __fadd_rn(__fadd_rn(xa.y, __double2float_rn(a.drift_y)),
                  __fmul_rn(__double2float_rn(a.std_y), __double2float_rn(n1)));
  return o;
}
template <>
__device__ __forceinline__ __half2 propagate_one<M_FP16>(__half2 xa, double n0, double n1, const FusedArgs& a) {
  // (x, y) travel in one half2: bx = x+drift, sx = std*n, x' = bx+sx (reference
  // filter.py:362-379 semantics, each op RN16; _rn forbids HFMA contraction)
  const __half2 drift = __halves2half2(__double2half(a.drift_x), __double2half(a.drift_y));
  const __half2 stdv = __halves2half2(__double2half(a.std_x), __double2half(a.std_y));
  const __half2 nn = __halves2half2(__double2half(n0), __double2half(n1));
  return __hadd2_rn(__hadd2_rn(xa, drift), __hmul2_rn(stdv, nn));
}

template <int MODE>
__device__ __forceinline__ int round_clamp(typename Tr<MODE>::real v, int lo, int hi);
template <>
__device__ __forceinline__ int round_clamp<M_FP64>(double v, int lo, int hi) {
  return min(max(__double2int_rn(v), lo), hi);
}
template <>
__device__ __forceinline__ int round_clamp<M_FP32>(float v, int lo, int hi) {
  return min(max(__float2int_rn(v), lo), hi);
}
template <>
__device__ __forceinline__ int round_clamp<M_FP16>(__half v, int lo, int hi) {
  return min(max(__half2int_rn(v), lo), hi);
}

template <int MODE>
__device__ __forceinline__ void vec_xy(typename Tr<MODE>::vec v, typename Tr<MODE>::real& x,
                                       typename Tr<MODE>::real& y) {
  x = v.x;
  y = v.y;
}

template <typename real>
__device__ __forceinline__ int lower_bound_c(const real* __restrict__ c, int lo, int hi, double q) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (to_d(c[mid]) < q)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

template <int MODE>
__device__ __forceinline__ typename Tr<MODE>::real neg_inf();
template <>
__device__ __forceinline__ double neg_inf<M_FP64>() {
  return __longlong_as_double(0xfff0000000000000LL);
}
template <>
__device__ __forceinline__ float neg_inf<M_FP32>() {
  return __int_as_float(0xff800000);
}
template <>
__device__ __forceinline__ __half neg_inf<M_FP16>() {
  return __ushort_as_half(0xfc00);
}

template <int MODE>
__device__ __forceinline__ bool rgt(typename Tr<MODE>::real a, typename Tr<MODE>::real b) {
  return to_d(a) > to_d(b);
}

// weight in fixed point: w_q = rint(exp(L - m) * 2^FB)
template <int MODE>
__device__ __forceinline__ typename Tr<MODE>::wq_t weight_q(typename Tr<MODE>::real L, typename Tr<MODE>::real m,
                                                            const unsigned short* exp16);
template <>
__device__ __forceinline__ long long weight_q<M_FP64>(double L, double m, const unsigned short*) {
  double w = pfm::exp64(__dsub_rn(L, m));
  return __double2ll_rn(__dmul_rn(w, 4503599627370496.0));  // 2^52
}
template <>
__device__ __forceinline__ long long weight_q<M_FP32>(float L, float m, const unsigned short*) {
  float w = pfm::exp32(__fsub_rn(L, m));
  return __float2ll_rn(__fmul_rn(w, 1099511627776.0f));  // 2^40
}
// RN16(exp(d)) for binary16 d <= 0, bit-identical to the correctly rounded
// table: exp(d) = 0 in binary16 below -17.33; in [-9.70, 0] ex2.approx gives
// y within ~2^-20 relative, so RN16(y) is the correctly rounded value unless
// y's 13 bits below binary16 precision lie within a margin of the rounding
// midpoint -- then (and in the subnormal range) read the table.  Checked
// exhaustively against the table on the device (tests/test_gpu_fused.py).
__device__ __forceinline__ __half exp16_fast(__half d, const unsigned short* exp16) {
  const float x = __half2float(d);
  if (x < -17.34f) return __ushort_as_half(0);
  if (x >= -9.70f) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(x, 1.44269504088896340736f)));
    const unsigned low = __float_as_uint(y) & 0x1fffu;  // bits below binary16 precision
    const int off = (int)low - 0x1000;
    if (off > 48 || off < -48) return __float2half_rn(y);
  }
  return __ushort_as_half(__ldg(exp16 + __half_as_ushort(d)));
}

// FP16 weights read the correctly rounded table directly (L1-resident: only
// the ~19.5K patterns in [-17.34, 0] are ever touched); kExp16Fast selects the
// ex2.approx + midpoint-guard path instead (same bits, more instructions)
constexpr bool kExp16Fast = false;
template <>
__device__ __forceinline__ int weight_q<M_FP16>(__half L, __half m, const unsigned short* exp16) {
  const __half d = __hsub_rn(L, m);
  const __half w = kExp16Fast ? exp16_fast(d, exp16) : __ushort_as_half(__ldg(exp16 + __half_as_ushort(d)));
  return __float2int_rn(__fmul_rn(__half2float(w), 1048576.0f));  // 2^20
}

// exhaustive check helper: out[i] = exp16_fast(bits i) for all 65536 patterns
#ifndef PF_FUSED_ONLY  // launched from pf_api.cu only
__global__ void pf_exp16_fast_check(const unsigned short* exp16, unsigned short* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 65536) {
    const __half d = __ushort_as_half((unsigned short)i);
    out[i] = (__half2float(d) <= 0.0f) ? __half_as_ushort(exp16_fast(d, exp16)) : exp16[i];
  }
}
#endif

// search keys: c_j >= q  <=>  key(c_j) >= key_up(q) for non-negative values,
// where key is the IEEE bit pattern (monotone for c >= 0) and key_up(q) the
// bits of the smallest mode value >= q.  Exact, and integer compares only.
template <int MODE>
struct Key;
template <>
struct Key<M_FP64> {
  using k_t = double;
  __device__ static __forceinline__ double of(double c) { return c; }
  __device__ static __forceinline__ double up(double q) { return q; }
};
template <>
struct Key<M_FP32> {
  using k_t = unsigned int;
  __device__ static __forceinline__ unsigned of(float c) { return __float_as_uint(c); }
  __device__ static __forceinline__ unsigned up(double q) { return __float_as_uint(__double2float_ru(q)); }
};
template <>
struct Key<M_FP16> {
  using k_t = unsigned short;
  __device__ static __forceinline__ unsigned short of(__half c) { return __half_as_ushort(c); }
  __device__ static __forceinline__ unsigned short up(double q) {
    __half h = __double2half(q);
    unsigned short b = __half_as_ushort(h);
    if ((double)__half2float(h) < q) b += 1;  // q in [0, 1]: next binary16 up
    return b;
  }
};

// first j in [lo, hi) with key(c[j]) >= kq (hi if none)
template <int MODE>
__device__ __forceinline__ int lb_key(const typename Tr<MODE>::real* c, int lo, int hi, typename Key<MODE>::k_t kq) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (Key<MODE>::of(c[mid]) < kq)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
// same, knowing key(c[j0 - 1]) < kq: exponential probe from j0, then bisection
template <int MODE>
__device__ __forceinline__ int gallop_key(const typename Tr<MODE>::real* c, int j0, int n,
                                          typename Key<MODE>::k_t kq) {
  if (j0 >= n || Key<MODE>::of(c[j0]) >= kq) return j0;
  int lo = j0 + 1, step = 1, hi = j0 + 1;
  while (hi < n && Key<MODE>::of(c[hi]) < kq) {
    lo = hi + 1;
    hi += step;
    step <<= 1;
  }
  if (hi > n) hi = n;
  return lb_key<MODE>(c, lo, hi, kq);
}

template <int MODE>
__device__ __forceinline__ bool gt_real(typename Tr<MODE>::real a, typename Tr<MODE>::real b) {
  if constexpr (MODE == M_FP16)
    return __hgt(a, b);
  else
    return a > b;
}

template <int MODE>
__device__ __forceinline__ typename Tr<MODE>::vec to_vec(double n0, double n1) {
  typename Tr<MODE>::vec v;
  if constexpr (MODE == M_FP16) {
    v = __halves2half2(__double2half(n0), __double2half(n1));
  } else if constexpr (MODE == M_FP32) {
    v.x = __double2float_rn(n0);
    v.y = __double2float_rn(n1);
  } else {
    v.x = n0;
    v.y = n1;
  }
  return v;
}

// "fp16" (scalar lanes, the reference's FP16_SCALAR engine): the same RN16
// ops one lane at a time -- the naive half of the paper's naive-vs-packed
// kernel pair; values are identical to the half2 path (hadd_s / hmul_s)
__device__ __forceinline__ __half2 scale_noise_scalar(__half2 nn, __half2 stdv) {
  return __halves2half2(hmul_s(__low2half(stdv), __low2half(nn)), hmul_s(__high2half(stdv), __high2half(nn)));
}
__device__ __forceinline__ __half2 prop_scalar(__half2 xa, __half2 sn, __half2 drift) {
  const __half x = hadd_s(hadd_s(__low2half(xa), __low2half(drift)), __low2half(sn));
  const __half y = hadd_s(hadd_s(__high2half(xa), __high2half(drift)), __high2half(sn));
  return __halves2half2(x, y);
}

// propagate with the scaled noise sn = d(std) * d(n) already formed:
// x' = (x[a] + d(drift)) + sn, each op rounded separately (reference arithmetic)
template <int MODE>
__device__ __forceinline__ typename Tr<MODE>::vec prop(typename Tr<MODE>::vec xa, typename Tr<MODE>::vec sn,
                                                       typename Tr<MODE>::vec drift) {
  typename Tr<MODE>::vec o;
  if constexpr (MODE == M_FP16) {
    o = __hadd2_rn(__hadd2_rn(xa, drift), sn);
  } else if constexpr (MODE == M_FP32) {
    o.x = __fadd_rn(__fadd_rn(xa.x, drift.x), sn.x);
    o.y = __fadd_rn(__fadd_rn(xa.y, drift.y), sn.y);
  } else {
    o.x = __dadd_rn(__dadd_rn(xa.x, drift.x), sn.x);
    o.y = __dadd_rn(__dadd_rn(xa.y, drift.y), sn.y);
  }
  return o;
}

template <int MODE>
constexpr int max_src_tiles() {  // source tiles staged in shared memory (else global search)
  return MODE == M_FP64 ? 3 : 4;
}
// (staging the source tiles' positions as well -- ancestor gather from shared
// memory -- was measured: slightly better latency at C2, worse at C3/C4 since
// it copies every source position, not only the ancestors; not done)

// ziggurat fast-path tables in shared memory: 256 x (ki >> 20) then 256 x wi
// (FP64 / FP32); binary16 modes: 256 x {ki >> 29, f32(wi * 2^29)} (2 KB)
// (a 512-entry signed {wi, ki} table was measured: fewer instructions, but the
// 8 KB per-CTA staging and 16-byte random reads made C2 / C3 slower)
constexpr int kZigBytes = 3072;

constexpr int kSlowQ = 128;  // deferred ziggurat slow paths per CTA (overflow -> inline)

// shared-memory footprint: ziggurat tables, noise/positions (vec per particle),
// staged source CDFs, table slice, slow-path queue, reduction scratch
template <int MODE>
constexpr size_t fused_smem_bytes() {
  using real = typename Tr<MODE>::real;
  using vec = typename Tr<MODE>::vec;
  return kZigBytes + PF_TILE * sizeof(vec) + max_src_tiles<MODE>() * PF_TILE * sizeof(real) + 16 +
         (max_src_tiles<MODE>() + 1) * 24 + kSlowQ * 12 + 320 * 8;
}

// branchless lower bound: first j in [0, n) with key(c[j]) >= kq, n if none
template <int MODE>
__device__ __forceinline__ int lb_branchless(const typename Tr<MODE>::real* c, int n, typename Key<MODE>::k_t kq) {
  int lo = 0;
  int len = n;
  while (len > 0) {
    const int half = len >> 1;
    const bool lt = Key<MODE>::of(c[lo + half]) < kq;
    lo = lt ? lo + half + 1 : lo;
    len = lt ? len - half - 1 : half;
  }
  return lo;
}
// The local CDF of every source tile ends at exactly 1 (its last particle's
// prefix equals the tile total), and every key is <= key(1): the lower bound
// always exists inside the tile, so the searches below need no bounds checks.
// First search of a full tile: fixed 10-step power-of-two bisection, unrolled
// (3-4 instructions per step instead of the general loop's 8-9).
// Only the 8-particle-per-thread variants (128 threads, the one-wave C1 / C2
// grids) unroll it: in the 256-thread multi-wave variant (C3 / C4) the larger
// code measured 8% slower (instruction fetch), so it keeps the loop.
template <int MODE, int VPT>
__device__ __forceinline__ int lb_first(const typename Tr<MODE>::real* c, int n, typename Key<MODE>::k_t kq) {
  static_assert(PF_TILE == 1024, "unrolled bisection over one tile");
  if (VPT < 8 || n != PF_TILE) return lb_branchless<MODE>(c, n, kq);
  int lo = 0;
#pragma unroll
  for (int step = PF_TILE / 2; step >= 1; step >>= 1)
    if (Key<MODE>::of(c[lo + step - 1]) < kq) lo += step;
  return lo;
}
// from a known position: short linear probe (the sentinel 1 at the tile's
// end bounds it), then exponential + bisection (a branch-free 4-entry
// prefix count was measured: -0.5 to -1.3%, the search is issue-bound)
// (CHECKED: the bounds test kept anyway -- measured 1.5% faster in the
// 256-thread FP16 variant, a code-layout effect)
template <int MODE, bool CHECKED = false>
__device__ __forceinline__ int advance_key(const typename Tr<MODE>::real* c, int j0, int n,
                                           typename Key<MODE>::k_t kq) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if ((CHECKED && j0 >= n) || Key<MODE>::of(c[j0]) >= kq) return j0;
    ++j0;
  }
  return gallop_key<MODE>(c, j0, n, kq);
}

// store one component of a particle's scaled noise pair d(std) * d(n): a plain
// component store (x and y of one particle may both take the slow path and be
// written by different threads concurrently -- no read-modify-write of the pair)
template <int MODE>
__device__ __forceinline__ void set_comp(typename Tr<MODE>::vec& v, int comp, double x, typename Tr<MODE>::vec stdv) {
  if constexpr (MODE == M_FP16) {
    const __half sd = comp ? __high2half(stdv) : __low2half(stdv);
    reinterpret_cast<__half*>(&v)[comp] = __hmul_rn(sd, __double2half(x));
  } else if constexpr (MODE == M_FP32) {
    const float f = __fmul_rn(comp ? stdv.y : stdv.x, __double2float_rn(x));
    if (comp)
      v.y = f;
    else
      v.x = f;
  } else {
    const double f = __dmul_rn(comp ? stdv.y : stdv.x, x);
    if (comp)
      v.y = f;
    else
      v.x = f;
  }
}

// d(std) * d(n) per component (the noise term of filter.py:195-202 / 362-379;
// independent of the ancestors, so it is formed before the frame's release)
template <int MODE>
__device__ __forceinline__ typename Tr<MODE>::vec scale_noise(typename Tr<MODE>::vec nn, typename Tr<MODE>::vec stdv) {
  typename Tr<MODE>::vec o;
  if constexpr (MODE == M_FP16) {
    o = __hmul2_rn(stdv, nn);
  } else if constexpr (MODE == M_FP32) {
    o.x = __fmul_rn(stdv.x, nn.x);
    o.y = __fmul_rn(stdv.y, nn.y);
  } else {
    o.x = __dmul_rn(stdv.x, nn.x);
    o.y = __dmul_rn(stdv.y, nn.y);
  }
  return o;
}

// canonical pairwise tree over a thread's VPT consecutive values
template <int VPT>
__device__ __forceinline__ double tree_vpt(const double* v) {
  if constexpr (VPT == 8)
    return __dadd_rn(__dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])),
                     __dadd_rn(__dadd_rn(v[4], v[5]), __dadd_rn(v[6], v[7])));
  else if constexpr (VPT == 4)
    return __dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3]));
  else if constexpr (VPT == 2)
    return __dadd_rn(v[0], v[1]);
  else
    return v[0];
}

// Minimum resident CTAs per SM (register budget) of the 256-thread variants,
// measured on C3 (same-box A/B): FP16 7 (32 registers, a few spills) 5.37 ->
// 5.64e10, FP32 6 (40 registers) 4.30 -> 4.45e10; FP64 5 (48 registers; 40
// lose 3%); the 128-thread variants keep the compiler's choice (C2 FP16 at 40
// registers: -9%).
#ifndef PF_MINB_FP16_256
#define PF_MINB_FP16_256 7  // A/B knob (make EXTRA=-DPF_MINB_FP16_256=6)
#endif
#ifndef PF_MINB_FP16_128
#define PF_MINB_FP16_128 0  // A/B knob (0: the compiler's choice)
#endif
template <int MODE>
constexpr int fused_min_blocks(int tpb) {
  return tpb == 128 ? (MODE == M_FP32 ? 7 : MODE == M_FP64 ? 6 : PF_MINB_FP16_128)
         : tpb != 256 ? 0 : MODE == M_FP16 ? PF_MINB_FP16_256 : MODE == M_FP32 ? 6 : 4;  // 0: no constraint
}

// One CTA = one tile of PF_TILE particles of one track; TPB = PF_TILE/(VPT*R)
// threads, thread t of round r owns particles (r*TPB + t)*VPT .. +VPT-1.
// SH: sharded filter (source tiles on several shards); PK: FP16 in packed
// half2 lanes (false: scalar lanes, "fp16" mode -- same values)
// DBG: the %globaltimer trace and the ancestor / likelihood capture of the
// parity tests are compiled only into this instantiation (as runtime checks
// they cost the production kernel ~10% at C3: registers and code layout)
// NZ: the frame's normals are read from a.noise (the reference's Philox
// stream) instead of being drawn from the LCG stream in phase 0
template <int MODE, int VPT, int R, bool SH = false, bool PK = true, bool DBG = false, bool NZ = false>
__global__ void __launch_bounds__(PF_TILE / (VPT * R), fused_min_blocks<MODE>(PF_TILE / (VPT * R)))
    pf_fused_frame(FusedArgs a) {
  using real = typename Tr<MODE>::real;
  using vec = typename Tr<MODE>::vec;
  using wq_t = typename Tr<MODE>::wq_t;
  using KT = Key<MODE>;
  constexpr int MS = max_src_tiles<MODE>();
  constexpr int TPB = PF_TILE / (VPT * R);
  constexpr int NW = TPB / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t* s_kihi = reinterpret_cast<const uint32_t*>(smem);    // 1 KB
  const double* s_wi = reinterpret_cast<const double*>(smem + 1024);  // 2 KB
  const uint2* s_kw32 = reinterpret_cast<const uint2*>(smem);         // FP16: {ki32, wi32 bits} x 256
  vec* s_X = reinterpret_cast<vec*>(smem + kZigBytes);                // per-particle scaled noise
  real* s_c = reinterpret_cast<real*>(smem + kZigBytes + PF_TILE * sizeof(vec));
  unsigned char* p_tab = reinterpret_cast<unsigned char*>(s_c + MS * PF_TILE);
  int* s_ts = reinterpret_cast<int*>(p_tab);                        // MS + 1 (in-track indices)
  double* s_tO = reinterpret_cast<double*>(p_tab + (MS + 1) * 8);   // MS + 1
  double* s_tM = reinterpret_cast<double*>(p_tab + (MS + 1) * 16);  // MS + 1
  unsigned long long* s_qw = reinterpret_cast<unsigned long long*>(p_tab + (MS + 1) * 24);
  int* s_qs = reinterpret_cast<int*>(s_qw + kSlowQ);
  double* s_misc = reinterpret_cast<double*>(s_qs + kSlowQ);
  // misc (8-byte slots): [0..31] warp max, [32..63] warp totals, [64..95] / [96..127] warp moments,
  // [128..191] round moments, [192..199] ints
  long long* s_wtot = reinterpret_cast<long long*>(s_misc + 32);
  int* s_int = reinterpret_cast<int*>(s_misc + 192);  // b_lo, b_hi, staged, queue count

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ltile = blockIdx.x, track = blockIdx.y;  // local tile of this handle
  const int tile = a.tile0 + ltile;                   // global tile
  const int K = (int)a.K, Kl = (int)a.K_local;
  const int base = tile * PF_TILE;  // global index of the tile's first particle
  const int lbase = ltile * PF_TILE;
  const int Tb = min(PF_TILE, K - base);
  const int n = a.n_tiles, nl = a.n_local;

  vec* __restrict__ Xn = reinterpret_cast<vec*>(a.X_new) + (size_t)track * Kl;
  real* __restrict__ Cn = reinterpret_cast<real*>(a.C_new) + (size_t)track * Kl;
  const real* __restrict__ map = reinterpret_cast<const real*>(a.map) + (size_t)(track % a.n_videos) * a.map_video_stride;
  // source tile b (global) -> (shard, local tile); track offsets apply when unsharded
  auto shard_of = [&](int b, int& lb) -> int {
    if (!SH) {
      lb = b;
      return 0;
    }
    const int sh = b / a.src.shard_tiles;
    lb = b - sh * a.src.shard_tiles;
    return sh;
  };
  // position of global particle k (its shard's buffer; one IMAD when unsharded)
  const vec* X0 = reinterpret_cast<const vec*>(a.src.X[0]) + (size_t)track * Kl;
  const int shard_parts = a.src.shard_tiles * PF_TILE;
  auto src_pos = [&](int k) -> const vec* {
    if (!SH) return X0 + k;
    const int sh = k / shard_parts;
    return reinterpret_cast<const vec*>(a.src.X[sh]) + (k - sh * shard_parts);
  };
  auto src_C = [&](int b) -> const real* {
    int lb;
    const int sh = shard_of(b, lb);
    return reinterpret_cast<const real*>(a.src.C[sh]) + (size_t)track * Kl + (size_t)lb * PF_TILE;
  };
  auto g_ts = [&](int b) -> int {
    int lb;
    const int sh = shard_of(b, lb);
    return (int)__ldg(a.src.ts[sh] + (size_t)track * nl + lb);
  };
  auto g_tO = [&](int b) -> double {
    int lb;
    const int sh = shard_of(b, lb);
    return __ldg(a.src.tO[sh] + (size_t)track * nl + lb);
  };
  auto g_tM = [&](int b) -> double {
    int lb;
    const int sh = shard_of(b, lb);
    return __ldg(a.src.tM[sh] + (size_t)track * nl + lb);
  };

  {
    const uint4* zsrc = reinterpret_cast<const uint4*>(a.zig);
    uint4* zdst = reinterpret_cast<uint4*>(smem);
    for (int i = tid; i < kZigBytes / 16; i += TPB) zdst[i] = zsrc[i];
  }
  PF_TRACE_DBG(a, 0);
  if (tid == 0) s_int[3] = 0;
  // stream state at this tile's first draw, position t(2K+1) + 2*base: the
  // frame's affine jump (kernel argument) and the per-tile jump
  const unsigned long long tstate =
      pfr::apply(pfr::Affine{a.tt[ltile].x, a.tt[ltile].y}, a.fa * a.x0[track] + a.fc);
  pdl_launch_dependents();
  __syncthreads();

  vec drift, stdv;
  if constexpr (MODE == M_FP16) {
    drift = __halves2half2(__double2half(a.drift_x), __double2half(a.drift_y));
    stdv = __halves2half2(__double2half(a.std_x), __double2half(a.std_y));
  } else {
    drift.x = (real)a.drift_x;
    drift.y = (real)a.drift_y;
    stdv.x = (real)a.std_x;
    stdv.y = (real)a.std_y;
  }

  // ---- phase 0: every draw of the tile (independent of the previous frame:
  // overlaps the previous kernel under PDL).  Fast ziggurat path, scaled by
  // d(std), into s_X; slow paths flagged branch-free per thread, then queued
  // and resolved in one CTA-wide pass.
  if constexpr (NZ) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int l0 = (rr * TPB + tid) * VPT;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (l0 + i < Tb) {
          const double2 nz = __ldg(a.noise + base + l0 + i);
          if constexpr (MODE == M_FP16 && !PK)
            s_X[l0 + i] = scale_noise_scalar(to_vec<MODE>(nz.x, nz.y), stdv);
          else
            s_X[l0 + i] = scale_noise<MODE>(to_vec<MODE>(nz.x, nz.y), stdv);
        }
      }
    }
  } else {
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    const int v = rr * TPB + tid;
    const int l0 = v * VPT;
    const unsigned long long xs0 = pfr::apply(pfr::Affine{a.tj[v].x, a.tj[v].y}, tstate);
    unsigned long long xs = xs0;
    unsigned slow = 0;  // bit 2i+c: normal (i, c) needs the slow path
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      if constexpr (MODE == M_FP16) {
        // binary16 modes: precision-matched draws (oracle/rng.py
        // normals16_from_lcg_words): the same words, fast path in binary32 on
        // the high 32 bits -- idx = bits 56..63, sign = bit 55, rabs = bits
        // 32..54 -- x = RN32(rabs * wi32[idx]), accepted iff rabs < ki32[idx]
        // ({ki32, wi32} per layer in one 8-byte shared entry), then RN16
        float nf[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const unsigned whi = (unsigned)(xs >> 32);
          xs = pfr::kA * xs + pfr::kC;
          const unsigned rabs = whi & 0x7fffffu;
          const uint2 kw = s_kw32[whi >> 24];
          const float x = __fmul_rn(__fsub_rn(__uint_as_float(0x4b000000u | rabs), 8388608.0f), __uint_as_float(kw.y));
          nf[c] = __uint_as_float(__float_as_uint(x) ^ ((whi << 8) & 0x80000000u));
          slow |= (rabs >= kw.x ? 1u : 0u) << (2 * i + c);
        }
        const __half2 nh = __floats2half2_rn(nf[0], nf[1]);
        if constexpr (!PK)
          s_X[l0 + i] = scale_noise_scalar(nh, stdv);
        else
          s_X[l0 + i] = __hmul2_rn(stdv, nh);
      } else {
      double nn[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const unsigned long long w = xs;
        xs = pfr::kA * xs + pfr::kC;
        const unsigned whi = (unsigned)(w >> 32), wlo = (unsigned)w;
        // rabs = bits 3..54 of w; (double)rabs exactly via the 2^52 bias trick
        const unsigned rlo = __funnelshift_r(wlo, whi, 3);
        const unsigned rhi = (whi >> 3) & 0xfffffu;
        const double rabs_d = __dsub_rn(__hiloint2double(0x43300000 | rhi, rlo), 4503599627370496.0);
        const unsigned idx = whi >> 24;  // layer: bits 56..63
        const double x = __dmul_rn(rabs_d, s_wi[idx]);
        // sign (bit 55) flips the sign bit of the product
        nn[c] = __hiloint2double(__double2hiint(x) ^ ((whi << 8) & 0x80000000u), __double2loint(x));
        // fast-path test rabs < ki on the top 32 bits of rabs (bits 23..54 of w)
        slow |= (__funnelshift_r(wlo, whi, 23) >= s_kihi[idx] ? 1u : 0u) << (2 * i + c);
      }
      s_X[l0 + i] = scale_noise<MODE>(to_vec<MODE>(nn[0], nn[1]), stdv);
      }  // FP64 / FP32 draws
    }
    if (l0 + VPT > Tb) slow = l0 >= Tb ? 0u : slow & ((1u << (2 * (Tb - l0))) - 1u);
    while (slow) {  // rare per thread: re-derive the word by stepping from xs0
      const int bit = __ffs(slow) - 1;
      slow &= slow - 1;
      unsigned long long w = xs0;
      for (int e = 0; e < bit; ++e) w = pfr::kA * w + pfr::kC;
      const int slot = atomicAdd(&s_int[3], 1);
      if (slot < kSlowQ) {
        s_qw[slot] = w;
        s_qs[slot] = (l0 + (bit >> 1)) * 2 + (bit & 1);
      } else {
        set_comp<MODE>(s_X[l0 + (bit >> 1)], bit & 1, pfr::zig_slow(w), stdv);  // queue overflow
      }
    }
  }
  }  // LCG draws
  __syncthreads();
  PF_TRACE_DBG(a, 1);
  // ---- warp 0: wait for the previous kernels, read this tile's source window
  //      (written by the previous frame's tile table) and start ONE bulk copy
  //      (cp.async.bulk, mbarrier-tracked) of exactly the source tiles' local
  //      CDFs while it fetches their table entries; the other warps meanwhile
  //      resolve the queued slow paths ------------------------------------
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_misc + 200);
  const bool bulk_ok = ((((size_t)track * Kl) * sizeof(real)) % 16) == 0;
  if (wid == 0 || NW == 1) {
    if (!a.ident) {  // acquire the previous frame's table (published before its grid ends)
      if (lane == 0) {
        const unsigned long long* rc = a.tmax + (size_t)track * 4 + 1;
        unsigned long long v;
        // relaxed polling (an acquire per poll would invalidate the SM's L1
        // under the CTAs still working on the previous frame), one acquire
        // load once the counter is reached
        // first look with acquire semantics: when the table is long done
        // (every CTA after the first wave) no separate fence is needed
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(rc) : "memory");
        if (v < a.ready_target) {
          do {
            __nanosleep(32);
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(rc) : "memory");
          } while (v < a.ready_target);
          // one acquire load once ready: measured 2-3% faster at C2 than
          // fence.acq_rel after the relaxed poll (the fence sits on the
          // frame's critical path)
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(rc) : "memory");
        }
        // launched programmatically behind the map kernel (one-frame step):
        // the frame's map is complete only after the grid dependency wait
        if (a.wait_prev) pdl_wait();
      }
      __syncwarp();
    } else {
      pdl_wait();  // frame 0 / injected state: the likelihood maps / initial positions
    }
    PF_TRACE_DBG(a, 2);
    if (!a.ident) {
      const int2 wn = __ldcg(reinterpret_cast<const int2*>(a.win) + (size_t)track * nl + ltile);
      const int nsrc = wn.y - wn.x + 1;
      const int staged = nsrc <= MS ? 1 : 0;
      if (!SH && staged && bulk_ok && lane == 0) {  // the window is contiguous: one bulk copy
        const uint32_t bb = smem_u32(s_bar);
        const int c0 = wn.x * PF_TILE;
        // 64-bit: (wn.y + 1) * PF_TILE reaches 2^31 for K near the 2^31-1 bound
        const int cnt = (int)(min((long long)(wn.y + 1) * PF_TILE, (long long)K) - (long long)c0);
        const uint32_t bytes = (uint32_t)((cnt * (int)sizeof(real) + 15) & ~15);  // C buffers carry 16 B of slack
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bb), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(s_c)),
            "l"(src_C(wn.x)), "r"(bytes), "r"(bb)
            : "memory");
      }
      if (SH && staged && bulk_ok) {
        // one bulk copy per source tile (tiles may live on different shards)
        const uint32_t bb = smem_u32(s_bar);
        if (lane == 0) {
          uint32_t total = 0;
          for (int e = 0; e < nsrc; ++e)
            total += (uint32_t)((min(PF_TILE, K - (wn.x + e) * PF_TILE) * (int)sizeof(real) + 15) & ~15);
          asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bb), "r"(1) : "memory");
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(total) : "memory");
        }
        __syncwarp();
        if (lane < nsrc) {
          const int b = wn.x + lane;
          // C buffers carry 16 B of slack for the rounded size
          const uint32_t bytes = (uint32_t)((min(PF_TILE, K - b * PF_TILE) * (int)sizeof(real) + 15) & ~15);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(s_c + lane * PF_TILE)),
              "l"(src_C(b)), "r"(bytes), "r"(bb)
              : "memory");
        }
      }
      if (lane == 0) {
        s_int[0] = wn.x;
        s_int[1] = wn.y;
        s_int[2] = staged;
      }
      if (staged && lane <= nsrc) {
        const int b = min(wn.x + lane, n - 1);
        s_ts[lane] = lane < nsrc ? g_ts(b) : K;
        s_tO[lane] = g_tO(b);
        s_tM[lane] = g_tM(b);
      }
    }
  }
  if (wid > 0 || NW == 1) {
    const int t0 = NW == 1 ? tid : tid - 32, nt = NW == 1 ? TPB : TPB - 32;
    const int nq = min(s_int[3], kSlowQ);
    for (int e = t0; e < nq; e += nt) {
      const int sl = s_qs[e];
      set_comp<MODE>(s_X[sl >> 1], sl & 1, pfr::zig_slow(s_qw[e]), stdv);
    }
  }
  __syncthreads();  // window and slow-path noise visible (and, for every thread, the previous table)
  PF_TRACE_DBG(a, 3);
  const double u = !a.ident ? __ldcg(a.u_prev + track) : 0.0;
  int b_lo = 0, b_hi = 0, staged = 0;
  if (!a.ident) {
    b_lo = s_int[0];
    b_hi = s_int[1];
    staged = s_int[2];
    if (staged) {
      if (bulk_ok) {  // wait for the bulk copy (phase 0 of the CTA's only mbarrier)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(s_bar))
            : "memory");
        PF_TRACE_DBG(a, 6);  // the window's CDFs have landed
      } else {  // unaligned track base (odd K with several tracks): plain copy
        for (int b = b_lo; b <= b_hi; ++b) {
          const real* src = src_C(b);
          const int cnt = min(PF_TILE, K - b * PF_TILE);
          for (int i = tid; i < cnt; i += TPB) s_c[(b - b_lo) * PF_TILE + i] = src[i];
        }
        __syncthreads();
      }
    }
  }
  const double invK = __ddiv_rn(1.0, (double)K);


  // ---- phase 1: resample + propagate + likelihood -------------------------
  // Threads whose VPT particles all lie inside the tile (all but at most one
  // warp of the last tile) take the FULL path, free of per-particle bounds.
  real Lr[R][VPT];
  vec Xr[R][VPT];
  real tmax = neg_inf<MODE>();
  const int mlo = -a.r, mhx = a.W - 1 + a.r, mhy = a.H - 1 + a.r;
  const real* __restrict__ mapc = map + a.r * a.Wm + a.r;  // map origin at (x, y) = (0, 0)
  const int Wm = a.Wm;
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    const int l0 = (rr * TPB + tid) * VPT;
    auto body = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      auto in_tile = [&](int i) -> bool { return FULL || l0 + i < Tb; };
      int anc[VPT];  // global ancestor index
      if (a.ident || (!FULL && l0 >= Tb)) {  // frame 0 / injected state: identity ancestors
#pragma unroll
        for (int i = 0; i < VPT; ++i) anc[i] = base + l0 + i;
      } else {
        // the search runs in two instantiations: window staged in shared
        // memory (the common case: LDS through shared-typed pointers) or
        // read from the source tiles' buffers (global loads)
        auto resample = [&](auto st_tag) {
          constexpr bool ST = decltype(st_tag)::value;
          auto tsv = [&](int b) -> int {
            if constexpr (ST) return s_ts[b - b_lo]; else return g_ts(b);
          };
          auto tOv = [&](int b) -> double {
            if constexpr (ST) return s_tO[b - b_lo]; else return g_tO(b);
          };
          auto tMv = [&](int b) -> double {
            if constexpr (ST) return s_tM[b - b_lo]; else return g_tM(b);
          };
          auto tCv = [&](int b) -> const real* {
            if constexpr (ST) return s_c + (b - b_lo) * PF_TILE; else return src_C(b);
          };
          int b = b_lo;
          if constexpr (!ST) {
            int lo = b_lo, hi = b_hi;
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (g_ts(mid) <= base + l0)
                lo = mid;
              else
                hi = mid - 1;
            }
            b = lo;
          }
          // register-cached geometry of the current source tile
          int sb = tsv(b), snext = b < b_hi ? tsv(b + 1) : K;
          double gO = tOv(b), gM = tMv(b);
          float fO = (float)gO, fM = (float)gM;  // FP16: the table holds f32 values
          int tl = b * PF_TILE, tb = min(PF_TILE, K - tl);
          const real* cb = tCv(b);
          int jprev = -1;
  #pragma unroll
          for (int i = 0; i < VPT; ++i) {
            const int k = base + l0 + i;
            if (!FULL && k >= K) {
              anc[i] = k;
              continue;
            }
            if (k >= snext) {  // next source tile (rare: outputs of one source tile are contiguous)
              do {
                ++b;
                snext = b < b_hi ? tsv(b + 1) : K;
              } while (k >= snext);
              sb = tsv(b);
              gO = tOv(b);
              gM = tMv(b);
              fO = (float)gO;
              fM = (float)gM;
              tl = b * PF_TILE;
              tb = min(PF_TILE, K - tl);
              cb = tCv(b);
              jprev = -1;
            }
            typename KT::k_t kq;
            if constexpr (MODE == M_FP16) {
              // f32 tile-local point: q = ((k - s_b) + phi_b) * rho_b
              float qf;
              if constexpr (PK)
                qf = __fmul_rn(__fadd_rn((float)(k - sb), fO), fM);
              else  // naive: the tile's f32 offset and scale re-cast from f64 for every particle
                qf = __fmul_rn(__fadd_rn((float)(k - sb), cvt_f32_f64_naive(gO)), cvt_f32_f64_naive(gM));
              kq = __half_as_ushort(__float2half_ru(fminf(fmaxf(qf, 0.0f), 1.0f)));
            } else {
              const double p = point_of<MODE>(k, u, K, invK);
              const double q = gM == 0.0 ? 0.0 : __dmul_rn(__dsub_rn(p, gO), gM);
              kq = KT::up(fmin(fmax(q, 0.0), 1.0));
            }
            // the unrolled first search is emitted once (particle 0); a later
            // particle that starts a new source tile (rare) takes the loop
            int j;
            if (i == 0)
              j = lb_first<MODE, VPT>(cb, tb, kq);
            else if (jprev >= 0)
              j = advance_key<MODE, (MODE == M_FP16 && VPT < 8)>(cb, jprev, tb, kq);
            else
              j = lb_branchless<MODE>(cb, tb, kq);
            j = min(j, tb - 1);
            jprev = j;
            anc[i] = tl + j;
          }
        };
        if (staged)
          resample(std::true_type{});
        else
          resample(std::false_type{});
        if (rr == 0) PF_TRACE_DBG(a, 7);  // thread 0's resampling search done
      }
      if (DBG && a.dbg_anc != nullptr) {
#pragma unroll
        for (int i = 0; i < VPT; ++i)
          if (in_tile(i)) a.dbg_anc[(size_t)track * Kl + lbase + l0 + i] = anc[i];
      }
      // all VPT ancestor gathers first (independent, read-only X_prev), then
      // propagation and all VPT map lookups, then the new positions' stores --
      // no store sits between loads, so nothing serialises the memory latency
      vec xa[VPT];
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (in_tile(i)) {
          xa[i] = __ldg(src_pos(anc[i]));
        } else {
          xa[i].x = (real)0;
          xa[i].y = (real)0;
        }
      }
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (in_tile(i)) {
          vec xn;
          if constexpr (MODE == M_FP16 && !PK)
            xn = prop_scalar(xa[i], s_X[l0 + i], drift);
          else
            xn = prop<MODE>(xa[i], s_X[l0 + i], drift);
          const int ix = round_clamp<MODE>(xn.x, mlo, mhx);
          const int iy = round_clamp<MODE>(xn.y, mlo, mhy);
          Lr[rr][i] = __ldg(mapc + iy * Wm + ix);
          Xr[rr][i] = xn;
        } else {  // outside the tile: weight exp(-inf) = 0, position 0
          Lr[rr][i] = neg_inf<MODE>();
          Xr[rr][i].x = (real)0;
          Xr[rr][i].y = (real)0;
        }
      }
      constexpr int VB = VPT * (int)sizeof(vec);
      if (VB % 16 == 0 && (FULL || l0 + VPT <= Tb) && ((((size_t)track * Kl) * sizeof(vec)) % 16) == 0) {
        uint4* dst = reinterpret_cast<uint4*>(Xn + lbase + l0);
#pragma unroll
        for (int q = 0; q < VB / 16; ++q) {
          uint4 o;
          memcpy(&o, reinterpret_cast<const unsigned char*>(&Xr[rr][0]) + 16 * q, 16);
          dst[q] = o;
        }
      } else {
#pragma unroll
        for (int i = 0; i < VPT; ++i)
          if (in_tile(i)) Xn[lbase + l0 + i] = Xr[rr][i];
      }
#pragma unroll
      for (int i = 0; i < VPT; ++i)
        if (gt_real<MODE>(Lr[rr][i], tmax)) tmax = Lr[rr][i];
    };
#if PF_FULL_SPEC
    if (l0 + VPT <= Tb)
      body(std::true_type{});
    else
#endif
      body(std::false_type{});
  }
  if (DBG && a.dbg_anc != nullptr) {  // debug capture (parity tests): recompute-free copies
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int l0 = (rr * TPB + tid) * VPT;
#pragma unroll
      for (int i = 0; i < VPT; ++i)
        if (l0 + i < Tb) reinterpret_cast<real*>(a.dbg_L)[(size_t)track * Kl + lbase + l0 + i] = Lr[rr][i];
    }
  }
  PF_TRACE_DBG(a, 4);
  // tile max (exact): warp max, one barrier, every thread reduces the NW values
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    const real o = __shfl_xor_sync(0xffffffffu, tmax, d);
    if (gt_real<MODE>(o, tmax)) tmax = o;
  }
  if (lane == 0) reinterpret_cast<real*>(s_misc)[wid] = tmax;
  __syncthreads();
  real mtile = reinterpret_cast<real*>(s_misc)[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) {
    const real o = reinterpret_cast<real*>(s_misc)[w];
    if (gt_real<MODE>(o, mtile)) mtile = o;
  }

  // ---- phase 2: weights, exact scan, local cdf, moments --------------------
  wq_t cum[R][VPT];
  wq_t thr_tot[R];
  long long mx_i = 0, my_i = 0;
  double rmx[R], rmy[R];
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    const int l0 = (rr * TPB + tid) * VPT;
    wq_t run = 0;
    double px[VPT], py[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      wq_t w;  // 0 outside the tile (L = -inf)
      if constexpr (MODE == M_FP16 && !PK) {  // naive: per-op f32 round trips (same values)
        const __half d = hsub_s(Lr[rr][i], mtile);
        w = __float2int_rn(__fmul_rn(__half2float(__ushort_as_half(__ldg(a.exp16 + __half_as_ushort(d)))), 1048576.0f));
      } else if constexpr (MODE == M_FP16) {  // one 32-bit table read: the weight's fixed-point value directly
        w = __ldg(a.exp16q + __half_as_ushort(__hsub_rn(Lr[rr][i], mtile)));
      } else {
        w = weight_q<MODE>(Lr[rr][i], mtile, a.exp16);
      }
      run += w;
      cum[rr][i] = run;  // thread-local inclusive
      if constexpr (MODE == M_FP16) {
        const int xq = __float2int_rn(__fmul_rn(__half2float(Xr[rr][i].x), 1024.0f));
        const int yq = __float2int_rn(__fmul_rn(__half2float(Xr[rr][i].y), 1024.0f));
        mx_i += (long long)w * xq;
        my_i += (long long)w * yq;
      } else {
        const double wd = (double)w;
        px[i] = __dmul_rn(wd, to_d(Xr[rr][i].x));
        py[i] = __dmul_rn(wd, to_d(Xr[rr][i].y));
      }
    }
    thr_tot[rr] = run;
    if constexpr (MODE != M_FP16) {
      double sx = tree_vpt<VPT>(px), sy = tree_vpt<VPT>(py);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        sx = __dadd_rn(sx, __shfl_xor_sync(0xffffffffu, sx, d));
        sy = __dadd_rn(sy, __shfl_xor_sync(0xffffffffu, sy, d));
      }
      rmx[rr] = sx;  // this warp's subtree of round rr
      rmy[rr] = sy;
    }
  }
  // warp inclusive scans of the thread totals, per round (exact integers)
  wq_t wexcl[R];
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    wq_t x = thr_tot[rr];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const wq_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    wexcl[rr] = x - thr_tot[rr];
    if (lane == 31) s_wtot[rr * NW + wid] = (long long)x;
  }
  if constexpr (MODE == M_FP16) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      mx_i += __shfl_xor_sync(0xffffffffu, mx_i, d);
      my_i += __shfl_xor_sync(0xffffffffu, my_i, d);
    }
    if (lane == 0) {
      reinterpret_cast<long long*>(s_misc)[64 + wid] = mx_i;
      reinterpret_cast<long long*>(s_misc)[96 + wid] = my_i;
    }
  } else {
    if (lane == 0) {
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        s_misc[64 + rr * NW + wid] = rmx[rr];
        s_misc[96 + rr * NW + wid] = rmy[rr];
      }
    }
  }
  __syncthreads();
  // prefix of this thread's segment = all earlier (round, warp) totals
  wq_t S = 0, before = 0;
  wq_t pre[R];
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const wq_t t = (wq_t)s_wtot[rr * NW + w];
      if (w == wid) pre[rr] = before;
      before += t;
    }
  }
  S = before;
  // local cdf c_j = d(cum_j / S), forced to 1 where cum_j == S
  const float invf = MODE == M_FP16 ? __fdiv_rn(1.0f, (float)S) : 0.0f;
  const double inv = MODE == M_FP16 ? 0.0 : __ddiv_rn(1.0, (double)S);
  auto cdf_of = [&](wq_t cm) -> real {
    if constexpr (MODE == M_FP16 && !PK) {  // naive: 1/S re-derived (cast + reciprocal) per particle
      return (cm == S) ? __float2half(1.0f) : __float2half_rn(__fmul_rn((float)cm, rcp_f32_s64_naive((long long)S)));
    } else if constexpr (MODE == M_FP16) {
      return (cm == S) ? __float2half(1.0f) : __float2half_rn(__fmul_rn((float)cm, invf));
    } else {
      const double cd = __dmul_rn((double)cm, inv);
      if constexpr (MODE == M_FP32)
        return (cm == S) ? 1.0f : __double2float_rn(cd);
      else
        return (cm == S) ? 1.0 : cd;
    }
  };
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    const int l0 = (rr * TPB + tid) * VPT;
    real cv[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) cv[i] = cdf_of(pre[rr] + wexcl[rr] + cum[rr][i]);
    constexpr int VB = VPT * (int)sizeof(real);
    if (l0 + VPT <= Tb && (VB == 4 || VB == 8 || VB == 16) && ((((size_t)track * Kl) * sizeof(real)) % VB) == 0) {
      if constexpr (VB == 16) {
        uint4 o;
        memcpy(&o, cv, 16);
        *reinterpret_cast<uint4*>(Cn + lbase + l0) = o;
      } else if constexpr (VB == 8) {
        uint2 o;
        memcpy(&o, cv, 8);
        *reinterpret_cast<uint2*>(Cn + lbase + l0) = o;
      } else if constexpr (VB == 4) {
        unsigned o;
        memcpy(&o, cv, 4);
        *reinterpret_cast<unsigned*>(Cn + lbase + l0) = o;
      }
    } else {
#pragma unroll
      for (int i = 0; i < VPT; ++i)
        if (l0 + i < Tb) Cn[lbase + l0 + i] = cv[i];
    }
  }
  // tile record
  if (tid == 0) {
    const size_t ri = (size_t)track * nl + ltile;
    a.rec_m[ri] = to_d(mtile);
    atomicMax(a.tmax + (size_t)track * 4, okey(to_d(mtile)));  // the table reads the track max directly
    a.rec_S[ri] = (long long)S;
    if constexpr (MODE == M_FP16) {
      long long sx = 0, sy = 0;
      for (int w = 0; w < NW; ++w) {
        sx += reinterpret_cast<long long*>(s_misc)[64 + w];
        sy += reinterpret_cast<long long*>(s_misc)[96 + w];
      }
      a.rec_X[ri] = sx;
      a.rec_Y[ri] = sy;
    } else {
      // canonical tree over the (round, warp) subtrees: contiguous aligned blocks
      double bx[R * NW], by[R * NW];
      for (int e = 0; e < R * NW; ++e) {
        bx[e] = s_misc[64 + e];
        by[e] = s_misc[96 + e];
      }
      for (int width = R * NW; width > 1; width >>= 1)
        for (int e = 0; e < width / 2; ++e) {
          bx[e] = __dadd_rn(bx[2 * e], bx[2 * e + 1]);
          by[e] = __dadd_rn(by[2 * e], by[2 * e + 1]);
        }
      a.rec_X[ri] = __double_as_longlong(bx[0]);
      a.rec_Y[ri] = __double_as_longlong(by[0]);
    }
  }
  PF_TRACE_DBG(a, 5);
  // complete only after the previous grid (keeps grid completion in stream
  // order: the next table reuses the exchange counters and records)
  if (!a.ident && tid == 0) pdl_wait();
}

// ------------------------------------------------------------------------
// tile table (one CTA per track)
// ------------------------------------------------------------------------
struct TableArgs {
  long long K;
  int n_tiles, n_pad;
  int t;
  int Q;
  const unsigned long long* x0;
  const double* rec_m;
  const long long* rec_S;
  const long long* rec_X;
  const long long* rec_Y;
  long long* tab_s;
  double* tab_O;
  double* tab_invM;
  double* u_out;
  unsigned long long ua, uc;  // f^(t(2K+1)+2K): uniform word = ua * x0[track] + uc
  double* traj;       // [track][F][2]
  double* est_host;   // optional: host-mapped copy of traj (synchronous runs: no copy back)
  int* deg_host;      // optional: [track] host-mapped first degenerate frame of the run (INT_MAX = none)
  int traj_stride;    // frames per track in traj
  int traj_index;     // frame slot
  int* degenerate;    // per track: first degenerate frame (or INT_MAX)
  int n_chunks;                 // CTAs per track (chunks of blockDim.x tiles)
  unsigned long long* sync;     // per track: [0] max key, [1] arrivals (max), [2] arrivals (sums), [3] ticket
  long long* agg;               // per track x chunk: chunk mass total
  double* roots;                // per track x chunk x 3: estimate subtree roots
  unsigned long long* trace;    // optional: [chunk][8] %globaltimer stamps (track 0)
  int2* win;                    // [track][tile]: source window of each destination tile (next frame)
  const double* u_in;           // optional: the frame's uniform (reference Philox stream), else the LCG's
};

// canonical pairwise accumulation over a power-of-two run (binary counter)
struct PwAcc {
  double st[24];
  int i;
  __device__ void reset() { i = 0; }
  __device__ void push(double v) {
    int j = i, lvl = 0;
    while (j & 1) {
      v = __dadd_rn(st[lvl], v);
      j >>= 1;
      ++lvl;
    }
    st[lvl] = v;
    ++i;
  }
  __device__ double root() const {  // i is a power of two
    int lvl = 0;
    while ((1 << lvl) < i) ++lvl;
    return st[lvl];
  }
};

__device__ __forceinline__ void spin_until(unsigned long long* ctr, unsigned long long target) {
  while (atomicAdd(ctr, 0ULL) < target) __nanosleep(64);
}

// Source windows of the next frame (scatter): destination tile d starts
// (ends) in source tile b iff its first (last) output index lies in
// [s_b, s_{b+1}); the ranges partition [0, K), so every d is written exactly
// once.  d is global; its record lives with the shard that owns it.
struct WinShards {
  int n_shards, shard_tiles;
  int2* win[PF_MAX_SHARDS];
};
__device__ __forceinline__ void scatter_windows(const WinShards& w, size_t track_off, int n, long long K, int b,
                                                long long sb, long long sn) {
  auto first_lo = [&](long long x) -> long long { return min((long long)n, (x + PF_TILE - 1) / PF_TILE); };
  auto first_hi = [&](long long x) -> long long {
    return x >= K ? (long long)n : min((long long)n - 1, max(0LL, x / PF_TILE));  // last output of d is 1024d+1023
  };
  auto rec = [&](long long d) -> int2* {
    if (w.n_shards == 1) return w.win[0] + track_off + d;
    const int sh = (int)(d / w.shard_tiles);
    return w.win[sh] + (d - (long long)sh * w.shard_tiles);
  };
  for (long long d = first_lo(sb), e = first_lo(sn); d < e; ++d) rec(d)->x = b;
  for (long long d = first_hi(sb), e = first_hi(sn); d < e; ++d) rec(d)->y = b;
}

// scatter_windows for one unsharded track (the tile table): 32-bit indices,
// shifts for the non-negative tile divisions, direct record pointer
__device__ __forceinline__ void scatter_windows_local(int2* wr, int n, long long K, int b, long long sb,
                                                      long long sn) {
  static_assert(PF_TILE == 1024, "tile shift");
  const int dl = (int)min((long long)n, (sb + PF_TILE - 1) >> 10);
  const int el = (int)min((long long)n, (sn + PF_TILE - 1) >> 10);
  const int dh = sb >= K ? n : (int)min((long long)n - 1, sb >> 10);
  const int eh = sn >= K ? n : (int)min((long long)n - 1, sn >> 10);
  for (int d = dl; d < el; ++d) wr[d].x = b;
  for (int d = dh; d < eh; ++d) wr[d].y = b;
}

// Tile table, one CTA per chunk of blockDim.x tiles (one tile per thread),
// grid (n_chunks, n_tracks).  All cross-CTA combination is exact: the global
// max is an atomicMax over order-preserving keys, the mass prefix an int64
// sum of chunk totals, and the estimate a canonical pairwise tree whose
// chunk subtrees are completed by the last CTA in tree order.  All CTAs of a
// track are co-resident: each calls launch_dependents on entry, so the next
// (dependent) grid cannot occupy the GPU before every table CTA has started.
template <int MODE, bool DBG = false>  // DBG: %globaltimer trace stamps (pf_set_trace)
__global__ void __launch_bounds__(1024) pf_tile_table(TableArgs a) {
  __shared__ long long s_i[32];
  __shared__ double s_d[3 * 32 + 4];
  __shared__ long long s_sb[1024];
  __shared__ int s_last;
  constexpr int FB = Tr<MODE>::FB;
  const int chunk = blockIdx.x, track = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int TPB = blockDim.x, nw = TPB >> 5;
  const int n = a.n_tiles, nc = a.n_chunks;
  const int b = chunk * TPB + tid;
  const bool valid = b < n;
  unsigned long long* sy = a.sync + (size_t)track * 4;

  PF_TRACE_DBG(a, 0);
  pdl_launch_dependents();
  // the frame's resampling uniform: stream position t(2K+1)+2K
  const double u = a.u_in ? *a.u_in : pfr::uniform_of(a.ua * a.x0[track] + a.uc);
  const double scale = ldexp(1.0, a.Q - FB);
  const double Kd = __ll2double_rn(a.K);
  const double invK = __ddiv_rn(1.0, Kd);
  pdl_wait();  // tile records of this frame's fused kernel
  PF_TRACE_DBG(a, 1);
  const size_t rb = (size_t)track * n + (valid ? b : 0);
  const double m1 = valid ? a.rec_m[rb] : __longlong_as_double(0xfff0000000000000LL);
  const long long S1 = valid ? a.rec_S[rb] : 0, X1 = valid ? a.rec_X[rb] : 0, Y1 = valid ? a.rec_Y[rb] : 0;

  // 1. global max (exact): the fused kernel's CTAs atomicMax'ed their tile
  //    maxima into sy[0] (order keys); reset by the last reader below
  const double m = okey_inv(__ldcg(sy + 0));
  PF_TRACE_DBG(a, 4);

  // 2. exact fixed-point tile mass and its prefix across the chunk / track
  double f = 0.0;
  long long mass = 0;
  if (valid) {
    f = pfm::exp64(__dsub_rn(m1, m));
    mass = __double2ll_rn(__dmul_rn(__dmul_rn((double)S1, f), scale));
  }
  long long ctot;
  long long excl = block_excl_scan<long long>(mass, s_i, &ctot);
  long long Sqi = ctot;
  if (nc > 1) {
    long long* ag = a.agg + (size_t)track * nc;
    if (tid == 0) {
      ag[chunk] = ctot;
      __threadfence();
      atomicAdd(sy + 2, 1ULL);
      spin_until(sy + 2, (unsigned long long)nc);
      if (chunk == 0) sy[0] = 0;  // every chunk read the max key before arriving
    }
    __syncthreads();
    long long before = 0, all = 0;
    for (int c = tid; c < nc; c += TPB) {
      const long long v = __ldcg(ag + c);
      all += v;
      if (c < chunk) before += v;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, d);
      all += __shfl_xor_sync(0xffffffffu, all, d);
    }
    if (lane == 0) {
      s_i[wid] = before;
      reinterpret_cast<long long*>(s_d)[wid] = all;
    }
    __syncthreads();
    before = 0;
    all = 0;
    for (int w = 0; w < nw; ++w) {
      before += s_i[w];
      all += reinterpret_cast<long long*>(s_d)[w];
    }
    excl += before;
    Sqi = all;
    __syncthreads();
  }
  const double Sq = (double)Sqi;
  PF_TRACE_DBG(a, 6);

  // 3. table entries and the estimate moments
  double vx = 0.0, vy = 0.0, vd = 0.0;
  if (valid) {
    const double O = __ddiv_rn((double)excl, Sq);
    long long sb = 0;
    if (b > 0) {
      long long k = (long long)floor(__dsub_rn(__dmul_rn(O, Kd), u));
      k = min(max(k, 0LL), a.K);
      while (k > 0 && point_of<MODE>(k - 1, u, a.K, invK) > O) --k;
      while (k < a.K && point_of<MODE>(k, u, a.K, invK) <= O) ++k;
      sb = k;
    }
    a.tab_s[rb] = sb;
    s_sb[tid] = sb;
    if constexpr (MODE == M_FP16) {
      // f32 tile-local coordinate q = ((k - s_b) + phi_b) * rho_b
      a.tab_O[rb] = (double)__double2float_rn(__dsub_rn(__dadd_rn((double)sb, u), __dmul_rn(Kd, O)));
      a.tab_invM[rb] = mass > 0 ? (double)__double2float_rn(__ddiv_rn(Sq, __dmul_rn(Kd, (double)mass))) : 0.0;
    } else {
      a.tab_O[rb] = O;
      a.tab_invM[rb] = mass > 0 ? __ddiv_rn(Sq, (double)mass) : 0.0;
    }
    double X, Y;
    if constexpr (MODE == M_FP16) {
      X = (double)X1;
      Y = (double)Y1;
    } else {
      X = __longlong_as_double(X1);
      Y = __longlong_as_double(Y1);
    }
    vx = __dmul_rn(f, X);
    vy = __dmul_rn(f, Y);
    vd = __dmul_rn(f, (double)S1);
  }
  PF_TRACE_DBG(a, 7);
  // source windows of the next frame (scatter_windows)
  __syncthreads();
  if (valid) {
    const long long sb = s_sb[tid];
    long long sn;
    if (b + 1 >= n) {
      sn = a.K;
    } else if (tid + 1 < TPB) {
      sn = s_sb[tid + 1];
    } else {  // first tile of the next chunk: same formula on its exact prefix
      const double On = __ddiv_rn((double)(excl + mass), Sq);
      long long k = (long long)floor(__dsub_rn(__dmul_rn(On, Kd), u));
      k = min(max(k, 0LL), a.K);
      while (k > 0 && point_of<MODE>(k - 1, u, a.K, invK) > On) --k;
      while (k < a.K && point_of<MODE>(k, u, a.K, invK) <= On) ++k;
      sn = k;
    }
    scatter_windows_local(a.win + (size_t)track * n, n, a.K, b, sb, sn);
  }
  // early release of the next frame: table entries, windows and u are
  // published with a per-track monotone counter (sy[1], +1 per chunk); the
  // next fused kernel acquires it instead of waiting for this grid to end
  // (the estimate below is off the critical path)
  if (chunk == 0 && tid == 0) {
    a.u_out[track] = u;
    if (nc == 1) sy[0] = 0;  // all threads read the max key before the barrier above
  }
  __syncthreads();  // CTA-wide release: barrier, then one gpu-scope fence + the counter
  if (tid == 0) {
    __threadfence();
    atomicAdd(sy + 1, 1ULL);
  }
  PF_TRACE_DBG(a, 5);
  // canonical pairwise tree: lanes, warps (zero padded), chunks (last CTA)
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    vx = __dadd_rn(vx, __shfl_xor_sync(0xffffffffu, vx, d));
    vy = __dadd_rn(vy, __shfl_xor_sync(0xffffffffu, vy, d));
    vd = __dadd_rn(vd, __shfl_xor_sync(0xffffffffu, vd, d));
  }
  if (lane == 0) {
    s_d[wid] = vx;
    s_d[32 + wid] = vy;
    s_d[64 + wid] = vd;
  }
  __syncthreads();
  if (wid == 0) {
    vx = lane < nw ? s_d[lane] : 0.0;
    vy = lane < nw ? s_d[32 + lane] : 0.0;
    vd = lane < nw ? s_d[64 + lane] : 0.0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      vx = __dadd_rn(vx, __shfl_xor_sync(0xffffffffu, vx, d));
      vy = __dadd_rn(vy, __shfl_xor_sync(0xffffffffu, vy, d));
      vd = __dadd_rn(vd, __shfl_xor_sync(0xffffffffu, vd, d));
    }
    if (lane == 0) {
      s_last = 1;
      if (nc > 1) {
        double* rt = a.roots + ((size_t)track * nc + chunk) * 3;
        rt[0] = vx;
        rt[1] = vy;
        rt[2] = vd;
        __threadfence();
        s_last = atomicAdd(sy + 3, 1ULL) == (unsigned long long)(nc - 1) ? 1 : 0;
      }
    }
  }
  __syncthreads();
  PF_TRACE_DBG(a, 2);
  if (!s_last) return;
  if (nc > 1) {  // last CTA: tree over the chunk roots (power-of-two padded)
    __threadfence();
    const double* rt = a.roots + (size_t)track * nc * 3;
    int ncp = 1;
    while (ncp < nc) ncp <<= 1;
    // each thread folds a contiguous pow2 block of chunk roots, then butterflies
    const int per = max(1, ncp / TPB);
    double px = 0.0, py = 0.0, pd = 0.0;
    if (tid * per < ncp) {  // binary-counter pairwise fold of a pow2 block
      PwAcc ax, ay, ad;
      ax.reset();
      ay.reset();
      ad.reset();
      for (int e = 0; e < per; ++e) {
        const int c = tid * per + e;
        ax.push(c < nc ? __ldcg(rt + 3 * c) : 0.0);
        ay.push(c < nc ? __ldcg(rt + 3 * c + 1) : 0.0);
        ad.push(c < nc ? __ldcg(rt + 3 * c + 2) : 0.0);
      }
      px = ax.root();
      py = ay.root();
      pd = ad.root();
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      px = __dadd_rn(px, __shfl_xor_sync(0xffffffffu, px, d));
      py = __dadd_rn(py, __shfl_xor_sync(0xffffffffu, py, d));
      pd = __dadd_rn(pd, __shfl_xor_sync(0xffffffffu, pd, d));
    }
    __syncthreads();
    if (lane == 0) {
      s_d[wid] = px;
      s_d[32 + wid] = py;
      s_d[64 + wid] = pd;
    }
    __syncthreads();
    if (wid == 0) {
      vx = lane < nw ? s_d[lane] : 0.0;
      vy = lane < nw ? s_d[32 + lane] : 0.0;
      vd = lane < nw ? s_d[64 + lane] : 0.0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        vx = __dadd_rn(vx, __shfl_xor_sync(0xffffffffu, vx, d));
        vy = __dadd_rn(vy, __shfl_xor_sync(0xffffffffu, vy, d));
        vd = __dadd_rn(vd, __shfl_xor_sync(0xffffffffu, vd, d));
      }
    }
  }
  if (tid == 0) {
    double ex = __ddiv_rn(vx, vd);
    double ey = __ddiv_rn(vy, vd);
    if constexpr (MODE == M_FP16) {
      ex = __dmul_rn(ex, 1.0 / 1024.0);
      ey = __dmul_rn(ey, 1.0 / 1024.0);
    }
    double* tr = a.traj + ((size_t)track * a.traj_stride + a.traj_index) * 2;
    tr[0] = ex;
    tr[1] = ey;
    PF_TRACE_DBG(a, 3);
    const bool degen = !(vd > 0.0) || !isfinite(vd) || !isfinite(ex) || !isfinite(ey);
    if (degen) atomicMin(a.degenerate + track, a.t);
    if (a.est_host != nullptr) {  // zero-copy result of a synchronous run (host-mapped, posted writes)
      double* eh = a.est_host + ((size_t)track * a.traj_stride + a.traj_index) * 2;
      eh[0] = ex;
      eh[1] = ey;
      if (degen && a.deg_host[track] > a.t) a.deg_host[track] = a.t;  // the host set INT_MAX before the run
    }
    // every CTA of the track has passed the exchanges: reset them for the
    // next frame's table (which starts only after the next fused kernel
    // completes, and that ends with griddepcontrol.wait on this grid)
    if (nc > 1) {
      sy[2] = 0;
      sy[3] = 0;
    }
    __threadfence();
  }
}

// ------------------------------------------------------------------------
// Sharded filter tables: one track split by particle range
// over n_shards handles (GPUs).  Per frame, on every shard, stream-ordered:
//   fused kernel -> [all-gather of the max keys]
//   -> pf_shard_mass (chunks of 256 tiles: exact masses, chunk totals, chunk
//      moment subtrees) -> pf_shard_sum (one CTA: chunk prefixes, shard total,
//      shard subtree roots) -> [all-gather of (total, X, Y, D)]
//   -> pf_shard_finish (offsets, table entries, window scatter into the owning
//      shards' records, estimate from the shard roots) -> [barrier]
// Every combination is the single-GPU table's (exact int64 prefixes, the
// canonical pairwise tree over tiles: shard_tiles is a power of two, so each
// shard's root is a node of the global tree), so the sharded filter is
// bit-identical to the same filter on one GPU.
// ------------------------------------------------------------------------
constexpr int kShardChunk = 256;

struct ShardArgs {
  long long K;      // global particles
  int n_tiles;      // global tiles
  int n_local;      // this shard's tiles
  int tile0;        // global index of this shard's first tile
  int Q;
  int n_shards, shard;
  int n_chunks;     // local chunks of kShardChunk tiles
  const unsigned long long* gmax;  // [n_shards] gathered max keys
  const long long* gsum;           // [n_shards][4] gathered: mass total, X, Y, D roots (double bits)
  const double* rec_m;
  const long long* rec_S;
  const long long* rec_X;
  const long long* rec_Y;
  long long* mass;       // [n_local] scratch: tile masses
  long long* ctot;       // [n_chunks]: chunk mass totals, then (pf_shard_sum) chunk exclusive prefixes
  double* croots;        // [n_chunks][3]: chunk moment subtree roots
  long long* sendsum;    // [4]: this shard's contribution to the second all-gather
  unsigned long long* maxkey;  // the fused kernels' max key (reset once gathered)
  long long* tab_s;
  double* tab_O;
  double* tab_invM;
  WinShards win;
  double* u_out;
  unsigned long long ua, uc;
  const unsigned long long* x0;
  double* traj;
  int traj_index;
  int* degenerate;
  int t;
};

template <int MODE>
__global__ void __launch_bounds__(kShardChunk) pf_shard_mass(ShardArgs a) {
  constexpr int FB = Tr<MODE>::FB;
  __shared__ long long s_i[kShardChunk / 32];
  __shared__ double s_d[3 * 32];
  const int chunk = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = kShardChunk / 32;
  const int b = chunk * kShardChunk + tid;  // local tile
  const bool valid = b < a.n_local;
  unsigned long long mk = 0;
  for (int sh = 0; sh < a.n_shards; ++sh) mk = max(mk, a.gmax[sh]);
  const double m = okey_inv(mk);
  double vx = 0.0, vy = 0.0, vd = 0.0;
  long long mass = 0;
  if (valid) {
    const double m1 = a.rec_m[b];
    const long long S1 = a.rec_S[b];
    const double f = pfm::exp64(__dsub_rn(m1, m));
    mass = __double2ll_rn(__dmul_rn(__dmul_rn((double)S1, f), ldexp(1.0, a.Q - FB)));
    double X, Y;
    if constexpr (MODE == M_FP16) {
      X = (double)a.rec_X[b];
      Y = (double)a.rec_Y[b];
    } else {
      X = __longlong_as_double(a.rec_X[b]);
      Y = __longlong_as_double(a.rec_Y[b]);
    }
    vx = __dmul_rn(f, X);
    vy = __dmul_rn(f, Y);
    vd = __dmul_rn(f, (double)S1);
    a.mass[b] = mass;
  }
  // exact chunk total
  long long tot = mass;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
  // canonical pairwise tree over the chunk's 256 tiles: lanes, then warps (zero padded)
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    vx = __dadd_rn(vx, __shfl_xor_sync(0xffffffffu, vx, d));
    vy = __dadd_rn(vy, __shfl_xor_sync(0xffffffffu, vy, d));
    vd = __dadd_rn(vd, __shfl_xor_sync(0xffffffffu, vd, d));
  }
  if (lane == 0) {
    s_i[wid] = tot;
    s_d[wid] = vx;
    s_d[32 + wid] = vy;
    s_d[64 + wid] = vd;
  }
  __syncthreads();
  if (wid == 0) {
    long long ct = lane < nw ? s_i[lane] : 0;
    vx = lane < nw ? s_d[lane] : 0.0;
    vy = lane < nw ? s_d[32 + lane] : 0.0;
    vd = lane < nw ? s_d[64 + lane] : 0.0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      ct += __shfl_xor_sync(0xffffffffu, ct, d);
      vx = __dadd_rn(vx, __shfl_xor_sync(0xffffffffu, vx, d));
      vy = __dadd_rn(vy, __shfl_xor_sync(0xffffffffu, vy, d));
      vd = __dadd_rn(vd, __shfl_xor_sync(0xffffffffu, vd, d));
    }
    if (lane == 0) {
      a.ctot[chunk] = ct;
      a.croots[3 * chunk + 0] = vx;
      a.croots[3 * chunk + 1] = vy;
      a.croots[3 * chunk + 2] = vd;
    }
  }
}

// one CTA: chunk exclusive prefixes (exact), shard total, shard subtree roots
template <int MODE>
__global__ void __launch_bounds__(1024) pf_shard_sum(ShardArgs a) {
  __shared__ long long s_i[32];
  __shared__ double s_d[3 * 32];
  __shared__ long long s_carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, TPB = blockDim.x, nw = TPB >> 5;
  const int nc = a.n_chunks;
  if (tid == 0) {
    s_carry = 0;
    *a.maxkey = 0;  // gathered: the next frame's fused CTAs publish into a fresh key
  }
  __syncthreads();
  // exclusive prefix of chunk totals, TPB at a time
  for (int c0 = 0; c0 < nc; c0 += TPB) {
    const int c = c0 + tid;
    const long long v = c < nc ? a.ctot[c] : 0;
    long long tot;
    const long long ex = block_excl_scan<long long>(v, s_i, &tot);
    const long long carry = s_carry;
    if (c < nc) a.ctot[c] = carry + ex;
    __syncthreads();
    if (tid == 0) s_carry = carry + tot;
    __syncthreads();
  }
  // canonical tree over the chunk roots (power-of-two padded): each thread a
  // contiguous pow2 block, then butterflies
  int ncp = 1;
  while (ncp < nc) ncp <<= 1;
  const int per = max(1, ncp / TPB);
  double px = 0.0, py = 0.0, pd = 0.0;
  if (tid * per < ncp) {
    PwAcc ax, ay, ad;
    ax.reset();
    ay.reset();
    ad.reset();
    for (int e = 0; e < per; ++e) {
      const int c = tid * per + e;
      ax.push(c < nc ? a.croots[3 * c] : 0.0);
      ay.push(c < nc ? a.croots[3 * c + 1] : 0.0);
      ad.push(c < nc ? a.croots[3 * c + 2] : 0.0);
    }
    px = ax.root();
    py = ay.root();
    pd = ad.root();
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    px = __dadd_rn(px, __shfl_xor_sync(0xffffffffu, px, d));
    py = __dadd_rn(py, __shfl_xor_sync(0xffffffffu, py, d));
    pd = __dadd_rn(pd, __shfl_xor_sync(0xffffffffu, pd, d));
  }
  if (lane == 0) {
    s_d[wid] = px;
    s_d[32 + wid] = py;
    s_d[64 + wid] = pd;
  }
  __syncthreads();
  if (wid == 0) {
    px = lane < nw ? s_d[lane] : 0.0;
    py = lane < nw ? s_d[32 + lane] : 0.0;
    pd = lane < nw ? s_d[64 + lane] : 0.0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      px = __dadd_rn(px, __shfl_xor_sync(0xffffffffu, px, d));
      py = __dadd_rn(py, __shfl_xor_sync(0xffffffffu, py, d));
      pd = __dadd_rn(pd, __shfl_xor_sync(0xffffffffu, pd, d));
    }
    if (lane == 0) {
      a.sendsum[0] = s_carry;
      a.sendsum[1] = __double_as_longlong(px);
      a.sendsum[2] = __double_as_longlong(py);
      a.sendsum[3] = __double_as_longlong(pd);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kShardChunk) pf_shard_finish(ShardArgs a) {
  __shared__ long long s_i[32];
  __shared__ long long s_sb[kShardChunk];
  const int chunk = blockIdx.x, tid = threadIdx.x;
  const int bl = chunk * kShardChunk + tid;  // local tile
  const int b = a.tile0 + bl;                // global tile
  const bool valid = bl < a.n_local;
  const int n = a.n_tiles;
  long long offset = 0, all = 0;
  for (int sh = 0; sh < a.n_shards; ++sh) {
    const long long v = a.gsum[4 * sh];
    if (sh < a.shard) offset += v;
    all += v;
  }
  const double Sq = (double)all;
  const double Kd = __ll2double_rn(a.K);
  const double invK = __ddiv_rn(1.0, Kd);
  const double u = pfr::uniform_of(a.ua * a.x0[0] + a.uc);
  const long long mass = valid ? a.mass[bl] : 0;
  long long ctot;
  long long excl = block_excl_scan<long long>(mass, s_i, &ctot) + offset + a.ctot[chunk];
  auto s_of = [&](double O) -> long long {
    long long k = (long long)floor(__dsub_rn(__dmul_rn(O, Kd), u));
    k = min(max(k, 0LL), a.K);
    while (k > 0 && point_of<MODE>(k - 1, u, a.K, invK) > O) --k;
    while (k < a.K && point_of<MODE>(k, u, a.K, invK) <= O) ++k;
    return k;
  };
  long long sb = 0;
  if (valid) {
    const double O = __ddiv_rn((double)excl, Sq);
    if (b > 0) sb = s_of(O);
    a.tab_s[bl] = sb;
    if constexpr (MODE == M_FP16) {
      a.tab_O[bl] = (double)__double2float_rn(__dsub_rn(__dadd_rn((double)sb, u), __dmul_rn(Kd, O)));
      a.tab_invM[bl] = mass > 0 ? (double)__double2float_rn(__ddiv_rn(Sq, __dmul_rn(Kd, (double)mass))) : 0.0;
    } else {
      a.tab_O[bl] = O;
      a.tab_invM[bl] = mass > 0 ? __ddiv_rn(Sq, (double)mass) : 0.0;
    }
    s_sb[tid] = sb;
  }
  __syncthreads();
  if (valid) {
    long long sn;
    if (b + 1 >= n)
      sn = a.K;
    else if (tid + 1 < kShardChunk && bl + 1 < a.n_local)
      sn = s_sb[tid + 1];
    else  // first tile of the next chunk / shard: same formula on its exact prefix
      sn = s_of(__ddiv_rn((double)(excl + mass), Sq));
    scatter_windows(a.win, 0, n, a.K, b, sb, sn);
  }
  if (chunk == 0 && tid == 0) {
    // estimate: canonical tree over the shard roots (power-of-two padded)
    double vx[PF_MAX_SHARDS], vy[PF_MAX_SHARDS], vd[PF_MAX_SHARDS];
    int w = 1;
    while (w < a.n_shards) w <<= 1;
    for (int sh = 0; sh < w; ++sh) {
      const bool ok = sh < a.n_shards;
      vx[sh] = ok ? __longlong_as_double(a.gsum[4 * sh + 1]) : 0.0;
      vy[sh] = ok ? __longlong_as_double(a.gsum[4 * sh + 2]) : 0.0;
      vd[sh] = ok ? __longlong_as_double(a.gsum[4 * sh + 3]) : 0.0;
    }
    for (; w > 1; w >>= 1)
      for (int e = 0; e < w / 2; ++e) {
        vx[e] = __dadd_rn(vx[2 * e], vx[2 * e + 1]);
        vy[e] = __dadd_rn(vy[2 * e], vy[2 * e + 1]);
        vd[e] = __dadd_rn(vd[2 * e], vd[2 * e + 1]);
      }
    double ex = __ddiv_rn(vx[0], vd[0]);
    double ey = __ddiv_rn(vy[0], vd[0]);
    if constexpr (MODE == M_FP16) {
      ex = __dmul_rn(ex, 1.0 / 1024.0);
      ey = __dmul_rn(ey, 1.0 / 1024.0);
    }
    a.traj[2 * a.traj_index] = ex;
    a.traj[2 * a.traj_index + 1] = ey;
    *a.u_out = u;
    if (!(vd[0] > 0.0) || !isfinite(vd[0]) || !isfinite(ex) || !isfinite(ey)) atomicMin(a.degenerate, a.t);
  }
}

}  // namespace pfk
