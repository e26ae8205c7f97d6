// pf_pipes.cu -- issue-rate microbenchmarks of the SM pipes the particle-filter
// kernels use, measured on the box (the roofline denominators of
// bench.py's roofline.pipes; the paper's pipe-utilisation evidence,
// /root/reference/PAPER.md:115,207-209, is relative to such peaks).
//
// Every kernel runs 8 independent dependency chains per thread of ONE
// instruction kind, 16x unrolled, at 32 resident warps per SM (2 CTAs x 512
// threads per SM, one wave).  Per CTA, clock64() brackets the loop; the rate is
// (warp-instructions of that kind per SM) / (max CTA cycles on that SM), so it
// is in warp-instructions per SM clock -- independent of the clock frequency.
// cuobjdump -sass of lib/libpf_pipes.so shows each loop body is the intended
// opcode (HFMA2, HADD2, FFMA, DFMA, IMAD, IADD3, LOP3.LUT, LDS, LDG, MUFU.EX2,
// F2F.F16.F64, I2F) plus the loop's own IADD / ISETP / BRA.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace {

constexpr int kThreads = 512;
constexpr int kCtasPerSm = 2;
constexpr int kUnroll = 16;
constexpr int kChains = 8;

enum Op { HFMA2 = 0, HADD2, FFMA, DFMA, IMAD, IADD3, LOP3, LDS, LDG, MUFU, F2F64, I2F, N_OPS };
const char* kNames[N_OPS] = {"hfma2", "hadd2", "ffma", "dfma", "imad", "iadd3", "lop3", "lds", "ldg", "mufu_ex2",
                             "f2f_f16_f64", "i2f"};

template <int OP>
__global__ void __launch_bounds__(kThreads) pipe_kernel(int iters, const unsigned* __restrict__ gbuf,
                                                         unsigned* sink, long long* cycles) {
  __shared__ unsigned sbuf[8192];  // 32 KB: two 16 KB halves, alternating per iteration
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sbuf[i] = i * 2654435761u;
  __syncthreads();
  const unsigned t = threadIdx.x + blockIdx.x * 7u;
  unsigned u[kChains];
  float f[kChains];
  double d[kChains];
  unsigned h[kChains];  // half2 bits
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    u[c] = t * (c + 3u);
    f[c] = (float)(t + c) * 1e-3f;
    d[c] = (double)(t + c) * 1e-3;
    const __half2 hv = __floats2half2_rn(1e-3f * c, 2e-3f * c);
    h[c] = *reinterpret_cast<const unsigned*>(&hv);
  }
  const unsigned k1 = 0x3c003c00u;  // half2(1, 1)
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sbuf) + 4u * (threadIdx.x & 31);
  const unsigned* gb = gbuf + (threadIdx.x & 31);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const unsigned sb_it = sbase + ((it & 1u) << 13);  // iteration-dependent base: no hoisting
    const unsigned* gb_it = gb + ((it & 1) << 12);
    const unsigned sb2 = t ^ (unsigned)it;
#pragma unroll
    for (int r = 0; r < kUnroll; ++r) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if constexpr (OP == HFMA2) {
          asm volatile("fma.rn.f16x2 %0, %0, %1, %1;" : "+r"(h[c]) : "r"(k1));
        } else if constexpr (OP == HADD2) {
          asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(h[c]) : "r"(k1));
        } else if constexpr (OP == FFMA) {
          asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[c]) : "f"(1.0001f));
        } else if constexpr (OP == DFMA) {
          asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[c]) : "d"(1.0001));
        } else if constexpr (OP == IMAD) {
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[c]) : "r"(0x9E3779B9u), "r"(t));
        } else if constexpr (OP == IADD3) {  // two adds -> one 3-input IADD3
          asm volatile("{\n\tadd.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;\n\t}" : "+r"(u[c]) : "r"(t), "r"(sb2));
        } else if constexpr (OP == LOP3) {
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c]) : "r"(t), "r"(0x55u));
        } else if constexpr (OP == LDS) {  // distinct conflict-free addresses (no load elimination)
          unsigned v;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sb_it + 128u * (r * kChains + c)));
          u[c] ^= v;
        } else if constexpr (OP == LDG) {  // L1-resident 16 KB buffer
          unsigned v;
          asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(gb_it + 32 * (r * kChains + c)));
          u[c] ^= v;
        } else if constexpr (OP == MUFU) {
          asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[c]));
        } else if constexpr (OP == F2F64) {  // input varies with the chain (not hoisted)
          unsigned short hv;
          asm volatile("{\n\t.reg .f64 dd;\n\tmov.b64 dd, {%1, %2};\n\tcvt.rn.f16.f64 %0, dd;\n\t}"
                       : "=h"(hv) : "r"(u[c]), "r"(0x3ff00000u));
          u[c] ^= hv;
        } else if constexpr (OP == I2F) {
          float fv;
          asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(fv) : "r"(u[c]));
          u[c] ^= __float_as_uint(fv);
        }
      }
    }
  }
  const long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= u[c] ^ __float_as_uint(f[c]) ^ h[c] ^ (unsigned)__double_as_longlong(d[c]);
  if (acc == 0x12345678u) sink[0] = acc;  // keeps every chain live
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

std::string g_err;

template <int OP>
int run_one(int sms, int iters, const unsigned* gbuf, unsigned* sink, long long* dcyc, double* out) {
  const int grid = sms * kCtasPerSm;
  pipe_kernel<OP><<<grid, kThreads>>>(iters / 4, gbuf, sink, dcyc);  // warm-up
  pipe_kernel<OP><<<grid, kThreads>>>(iters, gbuf, sink, dcyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return 3;
  }
  long long* cyc = new long long[grid];
  cudaMemcpy(cyc, dcyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
  delete[] cyc;
  // warp-instructions of this kind per SM: CTAs/SM x warps/CTA x iters x unroll x chains
  const double per_sm = (double)kCtasPerSm * (kThreads / 32) * iters * kUnroll * kChains;
  *out = per_sm / (double)mx;
  return 0;
}

}  // namespace

extern "C" {

int pf_pipe_count(void) { return N_OPS; }
const char* pf_pipe_name(int i) { return (i >= 0 && i < N_OPS) ? kNames[i] : ""; }
const char* pf_pipe_error(void) { return g_err.c_str(); }

/* out[i] = measured issue rate of instruction kind i (pf_pipe_name), warp-
 * instructions per SM per clock, at one full wave of 32 warps per SM. */
int pf_pipe_peaks(double* out, int32_t device) {
  if (!out) return 1;
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  unsigned *gbuf = nullptr, *sink = nullptr;
  long long* dcyc = nullptr;
  if (cudaMalloc(&gbuf, 16 * 1024 * sizeof(unsigned)) != cudaSuccess) return 3;
  cudaMemset(gbuf, 1, 16 * 1024 * sizeof(unsigned));
  cudaMalloc(&sink, 64);
  cudaMalloc(&dcyc, sms * kCtasPerSm * sizeof(long long));
  const int iters = 256;
  int rc = 0;
  rc |= run_one<HFMA2>(sms, iters, gbuf, sink, dcyc, out + HFMA2);
  rc |= run_one<HADD2>(sms, iters, gbuf, sink, dcyc, out + HADD2);
  rc |= run_one<FFMA>(sms, iters, gbuf, sink, dcyc, out + FFMA);
  rc |= run_one<DFMA>(sms, iters / 4, gbuf, sink, dcyc, out + DFMA);
  rc |= run_one<IMAD>(sms, iters, gbuf, sink, dcyc, out + IMAD);
  rc |= run_one<IADD3>(sms, iters, gbuf, sink, dcyc, out + IADD3);
  rc |= run_one<LOP3>(sms, iters, gbuf, sink, dcyc, out + LOP3);
  rc |= run_one<LDS>(sms, iters, gbuf, sink, dcyc, out + LDS);
  rc |= run_one<LDG>(sms, iters, gbuf, sink, dcyc, out + LDG);
  rc |= run_one<MUFU>(sms, iters, gbuf, sink, dcyc, out + MUFU);
  rc |= run_one<F2F64>(sms, iters / 4, gbuf, sink, dcyc, out + F2F64);
  rc |= run_one<I2F>(sms, iters, gbuf, sink, dcyc, out + I2F);
  cudaFree(gbuf);
  cudaFree(sink);
  cudaFree(dcyc);
  return rc;
}

}  // extern "C"
