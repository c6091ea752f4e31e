// mc_sampler.cuh — K3: the Monte-Carlo length sampler on the device,
// shared by the dispatch kernel (bsg_capi.cu) and the fleet kernel (closed_loop.cu).
#pragma once

#include <cstdint>

namespace bsg {

// ---- K3: Monte-Carlo length sampler -----------------------------
// estimate_length's Noisy formula (workload.cpp:126-136) applied to the
// candidate's predicted length, one SplitMix64 stream per sample
// (rand.h:11-56; stream seed mix_seed(seed, request_id * S + s)), exactly the
// host bsg_mc_lengths: u1 = 1 - (next >> 11) 2^-53, u2 = (next >> 11) 2^-53,
// |N| = |sqrt(-2 log u1) cos(2 pi u2)|, sign = next & 1, then
// L = max(1, round(est * (1 + sign |N| scale))), every product/sum rounded
// separately (no FMA). The integer stream and the rounding are exact; log/cos
// are CUDA's (<= 1 / 2 ulp) where the host uses glibc's, so a sample can only
// differ when est * (1 + e) lies within ~1e-12 of a half-integer.
__device__ __forceinline__ uint64_t sm64_next(uint64_t& st) {
  uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t sm64_mix_seed(uint64_t seed, uint64_t id) {
  uint64_t st = id * 0x9e3779b97f4a7c15ULL + 0x1b873593ULL;
  return seed ^ sm64_next(st);
}
__device__ __forceinline__ int32_t mc_sample(int32_t est, uint64_t request_id, int32_t S, int32_t s,
                                             uint64_t seed, double scale) {
  uint64_t st = sm64_mix_seed(seed, request_id * static_cast<uint64_t>(S) + static_cast<uint64_t>(s));
  const double u1 = __dadd_rn(1.0, -__dmul_rn(static_cast<double>(sm64_next(st) >> 11), 0x1.0p-53));
  const double u2 = __dmul_rn(static_cast<double>(sm64_next(st) >> 11), 0x1.0p-53);
  const double r = sqrt(__dmul_rn(-2.0, log(u1)));
  const double nrm = __dmul_rn(r, cos(__dmul_rn(6.283185307179586, u2)));  // (2.0 * pi) * u2
  const double half = fabs(nrm);
  const double sign = (sm64_next(st) & 1) ? 1.0 : -1.0;
  const double err = __dmul_rn(__dmul_rn(sign, half), scale);
  const double v = round(__dmul_rn(static_cast<double>(est), __dadd_rn(1.0, err)));
  return static_cast<int32_t>(fmax(1.0, v));
}

// Ascending bitonic sort of n (a power of two) int32 in shared memory by one warp.
__device__ __forceinline__ void warp_bitonic_sort(int32_t* a, int32_t n) {
  const int lane = threadIdx.x & 31;
  for (int32_t k = 2; k <= n; k <<= 1) {
    for (int32_t j = k >> 1; j > 0; j >>= 1) {
      __syncwarp();
      for (int32_t i = lane; i < n; i += 32) {
        const int32_t l = i ^ j;
        if (l > i) {
          const int32_t x = a[i], y = a[l];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
    }
  }
  __syncwarp();
}

// Ascending bitonic sort of 256 int32 held 8 per lane (position lane * 8 + e)
// in registers: distances < 8 are in-lane compare-exchanges, larger ones one
// shfl.xor per element (21 + 15 stages, no shared memory, no barriers).
__device__ __forceinline__ void warp_bitonic_sort256(int32_t (&x)[8]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 256; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < 8) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if ((e & j) == 0) {
            const int i = lane * 8 + e;
            const bool up = (i & k) == 0;
            const int32_t a = x[e], b = x[e | j];
            x[e] = up ? min(a, b) : max(a, b);
            x[e | j] = up ? max(a, b) : min(a, b);
          }
        }
      } else {
        const int lj = j >> 3;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = lane * 8 + e;
          const bool up = (i & k) == 0;
          const int32_t v = __shfl_xor_sync(0xffffffffu, x[e], lj);
          x[e] = (lower == up) ? min(x[e], v) : max(x[e], v);
        }
      }
    }
  }
}

__host__ __device__ constexpr int32_t pow2_ceil(int32_t x) {
  int32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Draws a request's S samples and leaves them sorted ascending in len[0, S)
// (shared memory of the calling warp; S <= 1024, len holds pow2_ceil(S) words).
// lengths_out (optional, global): the samples in sample order.
__device__ __forceinline__ void stage_mc_samples(int32_t* len, int32_t est, uint64_t request_id, int32_t S,
                                                 uint64_t seed, double scale, int32_t* lengths_out) {
  const int lane = threadIdx.x & 31;
  if (S <= 256) {  // samples lane * 8 + e in registers, sorted there
    int32_t x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int32_t j = lane * 8 + e;
      x[e] = j < S ? mc_sample(est, request_id, S, j, seed, scale) : INT32_MAX;
      if (lengths_out && j < S) lengths_out[j] = x[e];
    }
    warp_bitonic_sort256(x);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (lane * 8 + e < S) len[lane * 8 + e] = x[e];
    __syncwarp();
  } else {
    const int32_t Sp = pow2_ceil(S);
    for (int32_t j = lane; j < Sp; j += 32) {
      const int32_t v = j < S ? mc_sample(est, request_id, S, j, seed, scale) : INT32_MAX;
      len[j] = v;
      if (lengths_out && j < S) lengths_out[j] = v;
    }
    warp_bitonic_sort(len, Sp);
  }
}

}  // namespace bsg
