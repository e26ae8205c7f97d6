// pf_philox.cuh -- the reference's own draw stream, Generator(Philox(seed))
// (/root/reference/pkg/src/halfpf/filter.py:71-82), generated in parallel.
//
// NumPy's standard_normal is a ziggurat over 64-bit Philox4x64-10 words with a
// VARIABLE number of words per normal: one word on the fast path (~98.8%),
// more when the wedge or tail test runs (and again after a rejection).  Words
// are counter-addressable (word w of the stream = Philox(ctr0 + 1 + w/4)[w%4]
// after the initial buffer), so the stream of one frame -- standard_normal(2K)
// then random() -- is generated in four launches over a window of M words
// starting at the device-resident position P:
//
//   classify  every word position p: the normal that would START at p, its
//             value v[p] and its length L[p] (words consumed); per block of
//             kBlk positions, the exit of the start chain entered at offset 0
//   resolve   per block: entry d = exit of the previous block's chain taken
//             from offset 0 (speculation), count of starts and exit from d;
//             flag when the exit differs from the offset-0 exit (the walks
//             did not merge inside the block)
//   scan      one CTA: repairs the (rare) flagged blocks sequentially from
//             their true entries, exclusive scan of the counts, locates the
//             2K-th start (= position of the frame's uniform), advances P
//   emit      per block: ranks its starts and writes v into normal slots
//
// Start positions are exactly NumPy's sequential consumption, so the values
// equal Generator(Philox(seed)).standard_normal / random bit for bit, except
// the wedge test's exp (portable exp64 vs glibc exp, <= 1 ulp apart; a flip
// needs a uniform within ~2^-52 of the wedge boundary -- DESIGN.md).
#pragma once
#include <stdint.h>

#include "pf_rng.cuh"

namespace pfp {

constexpr int kBlk = 1024;     // word positions per block
constexpr int kThreads = 256;  // 4 positions per thread

struct PhxStream {
  unsigned long long key[2], ctr[4], buf[4];
  int pos;  // NumPy buffer_pos of the initial state (4: empty buffer)
};

__device__ __forceinline__ void ctr_add(const unsigned long long c[4], unsigned long long n, unsigned long long o[4]) {
  o[0] = c[0] + n;
  unsigned long long carry = o[0] < n ? 1ULL : 0ULL;
  o[1] = c[1] + carry;
  carry = (carry && o[1] == 0) ? 1ULL : 0ULL;
  o[2] = c[2] + carry;
  carry = (carry && o[2] == 0) ? 1ULL : 0ULL;
  o[3] = c[3] + carry;
}

// word w (0-based) of the stream: the initial buffer, then one Philox block per 4 words
__device__ __forceinline__ unsigned long long word_at(const PhxStream& s, unsigned long long w) {
  const unsigned long long nb = (unsigned long long)(4 - s.pos);
  if (w < nb) return s.buf[s.pos + (int)w];
  const unsigned long long j = w - nb;
  unsigned long long c[4], out[4];
  ctr_add(s.ctr, 1 + (j >> 2), c);
  pfr::philox_block(c, s.key, out);
  return out[j & 3];
}

// NumPy random_standard_normal (distributions.c) whose first word r0 is at
// position w: returns the value and L = words consumed
__device__ __noinline__ double normal_walk(const PhxStream& s, unsigned long long w, unsigned long long r0, int& L) {
  unsigned long long p = w, r = r0;
  for (;;) {
    p += 1;
    const unsigned idx = (unsigned)(r & 0xff);
    r >>= 8;
    const unsigned sign = (unsigned)(r & 1);
    const unsigned long long rabs = (r >> 1) & pfr::kMask52;
    double x = pfm::dmul((double)rabs, __longlong_as_double((long long)PF_ZIG_WI_BITS[idx]));
    if (sign) x = -x;
    if (rabs < PF_ZIG_KI[idx]) {
      L = (int)(p - w);
      return x;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = pfm::dmul(-pfr::kZigInvR, pfr::log1p_glibc(-pfr::uniform_of(word_at(s, p))));
        const double yy = -pfr::log1p_glibc(-pfr::uniform_of(word_at(s, p + 1)));
        p += 2;
        if (pfm::dadd(yy, yy) > pfm::dmul(xx, xx)) {
          L = (int)(p - w);
          return ((rabs >> 8) & 1) ? -pfm::dadd(pfr::kZigR, xx) : pfm::dadd(pfr::kZigR, xx);
        }
      }
    } else {
      const double fi0 = __longlong_as_double((long long)PF_ZIG_FI_BITS[idx - 1]);
      const double fi1 = __longlong_as_double((long long)PF_ZIG_FI_BITS[idx]);
      const double u = pfr::uniform_of(word_at(s, p));
      p += 1;
      if (pfm::dadd(pfm::dmul(pfm::dsub(fi0, fi1), u), fi1) < pfm::exp64(pfm::dmul(pfm::dmul(-0.5, x), x))) {
        L = (int)(p - w);
        return x;
      }
    }
    r = word_at(s, p);
  }
}

struct GenArgs {
  PhxStream s;
  unsigned long long* P;  // device: next unconsumed word position (advanced by scan)
  long long n;            // normals this frame (2K)
  int nblk;               // blocks of kBlk positions in the window
  double* v;              // [nblk * kBlk] value of the normal starting at each position
  int* L;                 // [nblk * kBlk] its length in words
  int* exit0;             // [nblk] exit (relative) of the chain entered at offset 0
  int* entry;             // [nblk] entry offset used
  int* count;             // [nblk] starts in the block from that entry
  int* exitb;             // [nblk] exit from that entry
  int* bad;               // [nblk] exit != exit0 (next block's speculation invalid)
  long long* base;        // [nblk] index of the block's first normal
  double* out;            // [n] normals of the frame
  double* u_out;          // the frame's uniform (random())
  int* status;            // 0 ok; 1 window too small
  int take_uniform;       // 1: random() follows the normals (a frame); 0: normals only
};

// slow positions (L > 1) of a block in ascending order -> s_list, returns count
__device__ __forceinline__ int block_slow_list(const int* Lb, int* s_list, int* s_cnt) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int c = 0, Lq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    Lq[q] = Lb[4 * tid + q];
    c += Lq[q] > 1 ? 1 : 0;
  }
  int x = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) s_cnt[wid] = x;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      const int t = s_cnt[w];
      s_cnt[w] = acc;
      acc += t;
    }
    s_cnt[kThreads / 32] = acc;
  }
  __syncthreads();
  int o = s_cnt[wid] + x - c;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (Lq[q] > 1) s_list[o++] = 4 * tid + q;
  __syncthreads();
  return s_cnt[kThreads / 32];
}

// walk the start chain from entry d over the block's slow list: starts are
// the positions not inside a chain; returns (count of starts < kBlk, exit)
__device__ __forceinline__ void block_walk(const int* Lb, const int* s_list, int ns, int d, int& count, int& exit) {
  if (d >= kBlk) {
    count = 0;
    exit = d;
    return;
  }
  int cov = d, interior = 0;
  for (int i = 0; i < ns; ++i) {
    const int s = s_list[i];
    if (s < cov) continue;  // inside an earlier chain: not a start
    const int e = s + Lb[s];
    interior += min(e, kBlk) - s - 1;
    cov = e;
  }
  count = (kBlk - d) - interior;
  exit = max(cov, kBlk);
}

__global__ void __launch_bounds__(kThreads) phx_classify(GenArgs a) {
  __shared__ int s_list[kBlk];
  __shared__ int s_cnt[kThreads / 32 + 1];
  const int b = blockIdx.x, tid = threadIdx.x;
  const unsigned long long P = *a.P;
  const unsigned long long p0 = P + (unsigned long long)b * kBlk + 4ULL * tid;
  double* vb = a.v + (size_t)b * kBlk;
  int* Lb = a.L + (size_t)b * kBlk;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const unsigned long long p = p0 + q;
    const unsigned long long r0 = word_at(a.s, p);
    // fast path inline (NumPy layout: idx = low byte, sign = bit 8, rabs = bits 9..60)
    const unsigned idx = (unsigned)(r0 & 0xff);
    const unsigned long long rabs = (r0 >> 9) & pfr::kMask52;
    double x;
    int len = 1;
    if (rabs < PF_ZIG_KI[idx]) {
      x = pfm::dmul((double)rabs, __longlong_as_double((long long)PF_ZIG_WI_BITS[idx]));
      if ((r0 >> 8) & 1) x = -x;
    } else {
      x = normal_walk(a.s, p, r0, len);
    }
    vb[4 * tid + q] = x;
    Lb[4 * tid + q] = len;
  }
  __syncthreads();
  const int ns = block_slow_list(Lb, s_list, s_cnt);
  if (tid == 0) {
    int c, e;
    block_walk(Lb, s_list, ns, 0, c, e);
    a.exit0[b] = e;
  }
}

__global__ void __launch_bounds__(kThreads) phx_resolve(GenArgs a) {
  __shared__ int s_list[kBlk];
  __shared__ int s_cnt[kThreads / 32 + 1];
  const int b = blockIdx.x;
  const int* Lb = a.L + (size_t)b * kBlk;
  const int ns = block_slow_list(Lb, s_list, s_cnt);
  if (threadIdx.x == 0) {
    const int d = b == 0 ? 0 : a.exit0[b - 1] - kBlk;
    int c, e;
    block_walk(Lb, s_list, ns, d, c, e);
    a.entry[b] = d;
    a.count[b] = c;
    a.exitb[b] = e;
    a.bad[b] = e != a.exit0[b] ? 1 : 0;
  }
}

// smallest flagged block index >= from (nblk if none); whole CTA
__device__ int next_bad(const int* bad, int from, int nblk, int* s_red) {
  int m = nblk;
  for (int i = from + (int)threadIdx.x; i < nblk; i += blockDim.x)
    if (bad[i]) {
      m = i;
      break;
    }
  for (int d = 16; d >= 1; d >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, d));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    int r = nblk;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = min(r, s_red[w]);
    s_red[32] = r;
  }
  __syncthreads();
  const int r = s_red[32];
  __syncthreads();
  return r;
}

// one CTA of kThreads threads
__global__ void __launch_bounds__(kThreads) phx_scan(GenArgs a) {
  __shared__ int s_list[kBlk];
  __shared__ int s_cnt[kThreads / 32 + 1];
  __shared__ int s_red[33];
  __shared__ long long s_part[kThreads];
  __shared__ int s_hit[2];
  const int tid = threadIdx.x, nblk = a.nblk;
  // 1. repair: a flagged block's successor starts at the flagged block's true
  //    exit; recompute successors until a walk merges again
  for (int b = next_bad(a.bad, 0, nblk, s_red); b + 1 < nblk; b = next_bad(a.bad, b + 1, nblk, s_red)) {
    const int nb = b + 1;
    const int* Lb = a.L + (size_t)nb * kBlk;
    const int ns = block_slow_list(Lb, s_list, s_cnt);
    if (tid == 0) {
      const int d = a.exitb[b] - kBlk;
      int c, e;
      block_walk(Lb, s_list, ns, d, c, e);
      a.entry[nb] = d;
      a.count[nb] = c;
      a.exitb[nb] = e;
      a.bad[nb] = e != a.exit0[nb] ? 1 : 0;
    }
    __syncthreads();
  }
  // 2. exclusive scan of the counts (chunks of kThreads blocks)
  long long carry = 0;
  if (tid == 0) s_hit[0] = -1;
  __syncthreads();
  for (int c0 = 0; c0 < nblk; c0 += kThreads) {
    const int b = c0 + tid;
    const long long c = b < nblk ? a.count[b] : 0;
    s_part[tid] = c;
    __syncthreads();
    for (int d = 1; d < kThreads; d <<= 1) {
      const long long y = tid >= d ? s_part[tid - d] : 0;
      __syncthreads();
      s_part[tid] += y;
      __syncthreads();
    }
    const long long incl = carry + s_part[tid];
    if (b < nblk) {
      a.base[b] = incl - c;
      if (incl - c <= a.n && a.n < incl) s_hit[0] = b;  // the block holding start #n
    }
    carry += s_part[kThreads - 1];
    __syncthreads();
  }
  const int hb = s_hit[0];
  if (hb < 0) {  // the window ended before 2K normals and the uniform
    if (tid == 0) *a.status = 1;
    return;
  }
  // 3. position of start #n in block hb: the frame's uniform, then P advances
  const int* Lb = a.L + (size_t)hb * kBlk;
  const int ns = block_slow_list(Lb, s_list, s_cnt);
  if (tid == 0) {
    const long long want = a.n - a.base[hb];  // rank among the block's starts
    int pos = -1;
    long long rank = 0;
    for (int p = a.entry[hb]; p < kBlk; p += Lb[p]) {  // consecutive starts: p, p + L[p], ...
      if (rank == want) {
        pos = p;
        break;
      }
      ++rank;
    }
    const unsigned long long P = *a.P;
    const unsigned long long end = P + (unsigned long long)hb * kBlk + (unsigned long long)pos;
    if (a.take_uniform) {
      *a.u_out = pfr::uniform_of(word_at(a.s, end));
      *a.P = end + 1;
    } else {
      *a.P = end;
    }
  }
}

__global__ void __launch_bounds__(kThreads) phx_emit(GenArgs a) {
  __shared__ int s_list[kBlk];
  __shared__ int s_cnt[kThreads / 32 + 1];
  __shared__ unsigned char s_cov[kBlk];
  __shared__ int s_wsum[kThreads / 32];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long base = a.base[b];
  if (base >= a.n || *a.status) return;
  const int* Lb = a.L + (size_t)b * kBlk;
  const int d = a.entry[b];
  for (int i = tid; i < kBlk; i += kThreads) s_cov[i] = i < d ? 1 : 0;
  const int ns = block_slow_list(Lb, s_list, s_cnt);  // (barriers inside)
  if (tid == 0) {
    int cov = d;
    for (int i = 0; i < ns; ++i) {
      const int s = s_list[i];
      if (s < cov) continue;
      const int e = min(s + Lb[s], kBlk);
      for (int q = s + 1; q < e; ++q) s_cov[q] = 1;
      cov = s + Lb[s];
    }
  }
  __syncthreads();
  int st[4], c = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    st[q] = s_cov[4 * tid + q] ? 0 : 1;
    c += st[q];
  }
  int x = c;
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, dd);
    if (lane >= dd) x += y;
  }
  if (lane == 31) s_wsum[wid] = x;
  __syncthreads();
  int before = 0;
  for (int w = 0; w < wid; ++w) before += s_wsum[w];
  long long idx = base + before + x - c;
  const double* vb = a.v + (size_t)b * kBlk;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (st[q]) {
      if (idx < a.n) a.out[idx] = vb[4 * tid + q];
      ++idx;
    }
}

// random() draws at consecutive positions (RngStream.uniform outside a frame)
__global__ void phx_uniforms(PhxStream s, const unsigned long long* P, long long m, double* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < m) out[i] = pfr::uniform_of(word_at(s, *P + (unsigned long long)i));
}
__global__ void phx_advance(unsigned long long* P, long long m) { *P += (unsigned long long)m; }

// words in the window for n normals (+ the uniform): ~1.0215 words per normal
// (SURVEY 8a a1); 1/16 + 4096 words of margin
__host__ inline int window_blocks(long long n) {
  const long long M = n + n / 16 + 4096;
  return (int)((M + kBlk - 1) / kBlk);
}

}  // namespace pfp
