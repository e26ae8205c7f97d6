// pf_staged.cuh -- reference-semantics stage kernels (make_engine / stage_hook path).
//
// One kernel (or short sequence) per reference stage method, operating on a
// structure-of-arrays particle set (xs, ys, loglik, weights, cdf in the mode
// dtype, ancestors int64), exactly as halfpf's ParticleSet
// (/root/reference/pkg/src/halfpf/filter.py:85-134).  Sums and scans follow
// NumPy's evaluation order (pairwise_sum leaves of <=128 + recursive tree,
// sequential cumsum), and the binary16 engine's sequential lane folds
// (filter.py:461-467, 499-506) run as single-thread kernels, so every stage is
// bit-exact against the reference given the same inputs -- except the wide
// `exp`, where NumPy's SIMD exp is replaced by the portable exp (ulp-level,
// documented in DESIGN.md).
#pragma once
#include "pf_kernels.cuh"

namespace pfs {
using pfk::M_FP16;
using pfk::M_FP32;
using pfk::M_FP64;
using pfk::to_d;
using pfk::Tr;

template <int MODE>
__global__ void st_init(long long K, void* xs, void* ys, void* ll, void* w, void* cdf, long long* anc, double x0,
                        double y0) {
  using real = typename Tr<MODE>::real;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  real* X = (real*)xs;
  real* Y = (real*)ys;
  real* L = (real*)ll;
  real* Wt = (real*)w;
  real* C = (real*)cdf;
  if constexpr (MODE == M_FP16) {
    X[k] = __double2half(x0);
    Y[k] = __double2half(y0);
    L[k] = __ushort_as_half(0);
    C[k] = __ushort_as_half(0);
    // invK = recip16(RN16(K)) (filter.py:331-332): RN16 of the f64 reciprocal
    double kk = (double)__half2float(__double2half((double)K));
    Wt[k] = __double2half(kk == 0.0 ? __longlong_as_double(0x7ff0000000000000LL) : 1.0 / kk);
  } else {
    X[k] = (real)x0;
    Y[k] = (real)y0;
    L[k] = (real)0;
    C[k] = (real)0;
    Wt[k] = (real)1 / (real)K;
  }
  anc[k] = k;
}

template <int MODE>
__global__ void st_propagate(long long K, const void* xs_old, const void* ys_old, void* xs, void* ys,
                             const long long* anc, const double* noise, double dx, double sx, double dy, double sy) {
  using real = typename Tr<MODE>::real;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const real* Xo = (const real*)xs_old;
  const real* Yo = (const real*)ys_old;
  long long a = anc[k];
  if constexpr (MODE == M_FP16) {
    __half2 xa = __halves2half2(Xo[a], Yo[a]);
    __half2 drift = __halves2half2(__double2half(dx), __double2half(dy));
    __half2 stdv = __halves2half2(__double2half(sx), __double2half(sy));
    __half2 nn = __halves2half2(__double2half(noise[2 * k]), __double2half(noise[2 * k + 1]));
    __half2 o = __hadd2_rn(__hadd2_rn(xa, drift), __hmul2_rn(stdv, nn));
    ((__half*)xs)[k] = __low2half(o);
    ((__half*)ys)[k] = __high2half(o);
  } else {
    real d_x = (real)dx, s_x = (real)sx, d_y = (real)dy, s_y = (real)sy;
    ((real*)xs)[k] = (Xo[a] + d_x) + s_x * (real)noise[2 * k];
    ((real*)ys)[k] = (Yo[a] + d_y) + s_y * (real)noise[2 * k + 1];
  }
}

template <int MODE>
__global__ void st_lookup(long long K, const void* xs, const void* ys, void* ll, const void* map, int W, int H, int r,
                          int Wm) {
  using real = typename Tr<MODE>::real;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  int ix = pfk::round_clamp<MODE>(((const real*)xs)[k], -r, W - 1 + r);
  int iy = pfk::round_clamp<MODE>(((const real*)ys)[k], -r, H - 1 + r);
  ((real*)ll)[k] = ((const real*)map)[(size_t)(iy + r) * Wm + (ix + r)];
}

// max over K values (exact); result as double
template <int MODE>
__global__ void st_max(long long K, const void* v, double* out) {
  using real = typename Tr<MODE>::real;
  __shared__ double sm[32];
  double m = __longlong_as_double(0xfff0000000000000LL);
  for (long long k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, to_d(((const real*)v)[k]));
  for (int d = 16; d >= 1; d >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, d));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sm[w]);
    m = fmax(m, sm[0]);
    *out = m;
  }
}

// wide weights: w = w * exp(L - d(m))
template <int MODE>
__global__ void st_weight_wide(long long K, void* w, const void* ll, double m) {
  using real = typename Tr<MODE>::real;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  real* Wt = (real*)w;
  const real L = ((const real*)ll)[k];
  if constexpr (MODE == M_FP64)
    Wt[k] = Wt[k] * pfm::exp64(L - m);
  else
    Wt[k] = Wt[k] * pfm::exp32(L - (float)m);
}

// binary16 weights: d = RN16(L - m); w = RN16(w * exp16(d))
__global__ void st_weight_half(long long K, __half* w, const __half* ll, unsigned short m16, const unsigned short* exp16) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  __half d = __hsub_rn(ll[k], __ushort_as_half(m16));
  __half f = __ushort_as_half(exp16[__half_as_ushort(d)]);
  w[k] = __hmul_rn(w[k], f);
}

// NumPy pairwise leaves: out[i] = pw_leaf(v[leaf_i]) (optionally v = a*b in f64)
template <typename acc_t, typename in_t>
__global__ void st_pw_leaves(const in_t* v, const short2* dummy, const long long* lstart, const int* llen, int nleaves,
                             acc_t* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nleaves) return;
  acc_t t[128];
  const long long s = lstart[i];
  const int n = llen[i];
  for (int j = 0; j < n; ++j) t[j] = (acc_t)to_d(v[s + j]);
  out[i] = pfk::pw_leaf<acc_t>(t, n);
}
// products f64(w)*f64(x) leaves (estimate, filter.py:241-246)
template <typename real>
__global__ void st_pw_leaves_prod(const real* w, const real* x, const long long* lstart, const int* llen, int nleaves,
                                  double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nleaves) return;
  double t[128];
  const long long s = lstart[i];
  const int n = llen[i];
  for (int j = 0; j < n; ++j) t[j] = to_d(w[s + j]) * to_d(x[s + j]);
  out[i] = pfk::pw_leaf<double>(t, n);
}
// combine leaves by the recursive plan (ops: >=0 push leaf, -1 add top two)
template <typename acc_t>
__global__ void st_pw_combine(const acc_t* leaves, const int* ops, int nops, double* out) {
  acc_t st[40];
  int sp = 0;
  for (int i = 0; i < nops; ++i) {
    int op = ops[i];
    if (op >= 0)
      st[sp++] = leaves[op];
    else {
      acc_t b = st[--sp];
      acc_t a = st[--sp];
      st[sp++] = a + b;
    }
  }
  *out = (double)st[0];
}

// binary16 two-lane weight fold (filter.py:461-467)
__global__ void st_half_sum(long long K, const __half* w, double* out) {
  __half a0 = __ushort_as_half(0), a1 = __ushort_as_half(0);
  for (long long k0 = 0; k0 + 1 < K; k0 += 2) {
    a0 = __hadd_rn(a0, w[k0]);
    a1 = __hadd_rn(a1, w[k0 + 1]);
  }
  if (K % 2) a0 = __hadd_rn(a0, w[K - 1]);
  *out = (double)__half2float(a0) + (double)__half2float(a1);
}

// wide normalise: w *= inv; cdf = sequential cumsum (np.cumsum)
template <int MODE>
__global__ void st_scale(long long K, void* w, double inv) {
  using real = typename Tr<MODE>::real;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  ((real*)w)[k] = ((real*)w)[k] * (real)inv;
}
template <int MODE>
__global__ void st_cumsum(long long K, const void* w, void* cdf) {
  using real = typename Tr<MODE>::real;
  real acc = (real)0;
  const real* W = (const real*)w;
  real* C = (real*)cdf;
  for (long long k = 0; k < K; ++k) {
    acc = acc + W[k];
    C[k] = acc;
  }
}
// binary16 normalise: wn = RN16(w * inv16); pair-carry scan (filter.py:492-508)
__global__ void st_half_scale(long long K, __half* w, unsigned short inv16) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  w[k] = __hmul_rn(w[k], __ushort_as_half(inv16));
}
__global__ void st_half_scan(long long K, const __half* wn, __half* cdf) {
  const __half z = __ushort_as_half(0);
  __half carry = z;
  for (long long k0 = 0; k0 + 1 < K; k0 += 2) {
    __half t0 = __hadd_rn(wn[k0], z);
    __half t1 = __hadd_rn(wn[k0 + 1], wn[k0]);
    cdf[k0] = __hadd_rn(t0, carry);
    cdf[k0 + 1] = __hadd_rn(t1, carry);
    carry = cdf[k0 + 1];
  }
  if (K % 2) cdf[K - 1] = __hadd_rn(carry, wn[K - 1]);
}
// binary16 estimate: sequential f64 accumulation (filter.py:510-519)
__global__ void st_half_estimate(long long K, const __half* w, const __half* xs, const __half* ys, double* out) {
  double ex = 0.0, ey = 0.0;
  for (long long k = 0; k < K; ++k) {
    double wk = (double)__half2float(w[k]);
    ex = ex + wk * (double)__half2float(xs[k]);
    ey = ey + wk * (double)__half2float(ys[k]);
  }
  out[0] = ex;
  out[1] = ey;
}

// resample: wide p = (d(k)+d(u))/d(K); binary16 p = RN16(RN16(k16+u16)*invK)
template <int MODE>
__global__ void st_resample(long long K, const void* cdf, long long* anc, void* w, double u, unsigned short u16,
                            unsigned short invK16) {
  using real = typename Tr<MODE>::real;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const real* C = (const real*)cdf;
  double p;
  if constexpr (MODE == M_FP16) {
    __half s = __hadd_rn(__ll2half_rn(k), __ushort_as_half(u16));
    p = to_d(__hmul_rn(s, __ushort_as_half(invK16)));
  } else {
    p = to_d(((real)k + (real)u) / (real)K);
  }
  long long lo = 0, hi = K;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (to_d(C[mid]) < p)
      lo = mid + 1;
    else
      hi = mid;
  }
  anc[k] = lo < K - 1 ? lo : K - 1;
  if constexpr (MODE == M_FP16)
    ((real*)w)[k] = __ushort_as_half(invK16);
  else
    ((real*)w)[k] = (real)1 / (real)K;
}

// systematic_ancestors(cdf, u) -- float64 (filter.py:583-588)
__global__ void st_systematic(long long K, const double* cdf, double u, long long* anc) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double p = ((double)k + u) / (double)K;
  long long lo = 0, hi = K;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (cdf[mid] < p)
      lo = mid + 1;
    else
      hi = mid;
  }
  anc[k] = lo < K - 1 ? lo : K - 1;
}

// LCG stream normals at positions [pos, pos+n)
__global__ void st_rng_normals(unsigned long long x0, unsigned long long pos, long long n, double* out) {
  __shared__ uint32_t kihi[256];
  __shared__ double wi[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    kihi[i] = (uint32_t)(PF_ZIG_KI[i] >> 20);
    wi[i] = __longlong_as_double((long long)PF_ZIG_WI_BITS[i]);
  }
  __syncthreads();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = pfr::normal_of(pfr::word_at(x0, pos + (unsigned long long)i), kihi, wi);
}
__global__ void st_rng_uniforms(unsigned long long x0, unsigned long long pos, long long n, double* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = pfr::uniform_of(pfr::word_at(x0, pos + (unsigned long long)i));
}

template <int MODE>
__global__ void fill_start(long long n, void* X, double x0, double y0) {
  using vec = typename Tr<MODE>::vec;
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  vec v;
  if constexpr (MODE == M_FP16) {
    v = __halves2half2(__double2half(x0), __double2half(y0));
  } else {
    v.x = (typename Tr<MODE>::real)x0;
    v.y = (typename Tr<MODE>::real)y0;
  }
  ((vec*)X)[k] = v;
}

}  // namespace pfs
