// pf_video.cuh -- input side of the tracking step: synthetic
// video rendering on the device and PFVD container ingest into device memory.
//
// Reference: model.generate_video (/root/reference/pkg/src/halfpf/model.py:
// 123-157) and read_video / write_video (:270-297).
//
// The device renderer reproduces the reference model exactly -- background,
// the disk template stamped at the rint (half-even) centre with clipped
// offsets, additive Gaussian noise `base + std * z` (two roundings), rint,
// clip to [0, 255] -- and the ground-truth trajectory (specular bounces) is
// computed on the host by the reference recurrence.  Only the noise stream
// differs: z comes from the counter-based LCG ziggurat stream (video pixel
// (t, y, x) -> stream position (t H + y) W + x of the video seed), not NumPy's
// PCG64, so the frames are a pure function of (seed, t, y, x) that any number
// of threads can render independently (oracle/video.py restates it).
#pragma once
#include <stdint.h>

#include "pf_rng.cuh"

namespace pfv {

// video noise stream: independent of the filter's stream for the same seed
__host__ __device__ inline unsigned long long video_stream_state(unsigned long long seed) {
  return pfr::splitmix64_mix(pfr::seed_state(seed) ^ 0x56494445ULL);  // "VIDE"
}

// every pixel of every frame: background + noise (8 pixels per thread)
__global__ void render_background(uint8_t* frames, long long n_pixels, unsigned long long x0, double bg,
                                  double noise_std) {
  __shared__ uint32_t kihi[256];
  __shared__ double wi[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    kihi[i] = (uint32_t)(PF_ZIG_KI[i] >> 20);
    wi[i] = __longlong_as_double((long long)PF_ZIG_WI_BITS[i]);
  }
  __syncthreads();
  const long long p0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (p0 >= n_pixels) return;
  unsigned long long w = pfr::word_at(x0, (unsigned long long)p0);
  uint8_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double val = bg;
    if (noise_std > 0.0) val = __dadd_rn(val, __dmul_rn(noise_std, pfr::normal_of(w, kihi, wi)));
    w = pfr::kA * w + pfr::kC;
    v[i] = (uint8_t)fmin(fmax(rint(val), 0.0), 255.0);
  }
  if (p0 + 8 <= n_pixels && (p0 % 8) == 0) {
    uint2 o;
    memcpy(&o, v, 8);
    *reinterpret_cast<uint2*>(frames + p0) = o;
  } else {
    for (int i = 0; i < 8 && p0 + i < n_pixels; ++i) frames[p0 + i] = v[i];
  }
}

// the disk pixels of each frame (fg_index: [F][n_off] frame-local pixel
// indices after clipping; duplicates rewrite the same value)
__global__ void render_object(uint8_t* frames, const int* fg_index, int n_off, long long frame_pixels,
                              unsigned long long x0, double fg, double noise_std) {
  const int t = blockIdx.x;
  for (int j = threadIdx.x; j < n_off; j += blockDim.x) {
    const long long p = (long long)t * frame_pixels + fg_index[(size_t)t * n_off + j];
    double val = fg;
    if (noise_std > 0.0) {
      const unsigned long long w = pfr::word_at(x0, (unsigned long long)p);
      // fast path from the constant tables (one normal per thread)
      const unsigned idx = (unsigned)(w >> 56);
      const uint64_t rabs = (w >> 3) & pfr::kMask52;
      double z;
      if (rabs < PF_ZIG_KI[idx]) {
        z = __dmul_rn((double)rabs, __longlong_as_double((long long)PF_ZIG_WI_BITS[idx]));
        if ((w >> 55) & 1) z = -z;
      } else {
        z = pfr::zig_slow(w);
      }
      val = __dadd_rn(val, __dmul_rn(noise_std, z));
    }
    frames[p] = (uint8_t)fmin(fmax(rint(val), 0.0), 255.0);
  }
}

}  // namespace pfv
