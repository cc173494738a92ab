// Per-epoch history update on the device: the plumbing between a rollout
// step's outputs and the next epoch's K1 ingest, so finished rollouts never round-trip through host
// memory on their way to the GPU that owns their prompt next.
//
//   hs_pack_rows      gather variable-length rows of a [n, stride] token matrix into one flat send
//                     buffer in routing order (one CTA per row, coalesced int4 copies when aligned)
//   hs_mutate_bursts  the (D) synthetic-drift step of the bench: G independent
//                     s-mutations of every routed rollout, with tracegen's burst semantics
//                     (tracegen.py:78-120: alternating geometric keep / mutate runs, mean mutate run
//                     `burst`, mean keep run burst * s / (1 - s), first run kept with probability s,
//                     mutated positions draw a uniform token) from a counter-based hash RNG instead of
//                     numpy's PCG64 stream -- same distribution, not the same bytes (the numpy
//                     restatement in synth.py stays the parity input).  Rewards Bernoulli(0.5) in
//                     reward fixed point.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hs_common.cuh"

namespace route {

__global__ void k_pack_rows(const int32_t* __restrict__ src, int64_t src_stride, const int32_t* __restrict__ row,
                            const int64_t* __restrict__ len, const int64_t* __restrict__ dst_off, int32_t n,
                            int32_t* __restrict__ dst) {
  for (int32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int32_t* s = src + (int64_t)row[i] * src_stride;
    int32_t* d = dst + dst_off[i];
    const int64_t L = len[i];
    const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
    if (vec) {
      const int64_t L4 = L >> 2;
      const int4* s4 = reinterpret_cast<const int4*>(s);
      int4* d4 = reinterpret_cast<int4*>(d);
      for (int64_t j = threadIdx.x; j < L4; j += blockDim.x) d4[j] = s4[j];
      for (int64_t j = (L4 << 2) + threadIdx.x; j < L; j += blockDim.x) d[j] = s[j];
    } else {
      for (int64_t j = threadIdx.x; j < L; j += blockDim.x) d[j] = s[j];
    }
  }
}

__device__ __forceinline__ uint64_t rng_at(uint64_t key, uint64_t ctr) {
  return hs::mix64(key + ctr * 0x9E3779B97F4A7C15ULL);
}
__device__ __forceinline__ double unit(uint64_t h) {   // (0, 1)
  return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
// geometric(p) on {1, 2, ...}: 1 + floor(log(u) / log(1 - p))
__device__ __forceinline__ int64_t geometric(uint64_t h, double p) {
  if (p >= 1.0) return 1;
  return 1 + (int64_t)floor(log(unit(h)) / log1p(-p));
}

// one thread per output response (source row i, member g)
__global__ void k_mutate_bursts(const int32_t* __restrict__ src, const int64_t* __restrict__ src_off, int32_t n,
                                int32_t G, double s, double burst, int32_t vocab, uint64_t seed,
                                int32_t* __restrict__ dst, int64_t* __restrict__ reward_fx) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (int64_t)n * G) return;
  const int32_t i = (int32_t)(k / G), g = (int32_t)(k % G);
  const int64_t o = src_off[i], L = src_off[i + 1] - o;
  const int32_t* p = src + o;
  int32_t* d = dst + (int64_t)G * o + (int64_t)g * L;
  const uint64_t key = hs::mix64(seed ^ hs::mix64(((uint64_t)(uint32_t)i << 32) | (uint32_t)g));
  uint64_t ctr = 0;
  reward_fx[k] = (rng_at(key, ctr++) >> 63) ? ((int64_t)1 << HS_REWARD_FRAC_BITS) : 0;
  if (s >= 1.0) {
    for (int64_t j = 0; j < L; ++j) d[j] = p[j];
    return;
  }
  const double mean_keep = s > 0.0 ? burst * s / (1.0 - s) : 0.0;
  const double p_keep = s > 0.0 ? fmin(1.0, 1.0 / mean_keep) : 1.0;
  const double p_mut = fmin(1.0, 1.0 / burst);
  bool keep = s > 0.0 && unit(rng_at(key, ctr++)) < s;
  int64_t j = 0;
  while (j < L) {
    int64_t run = keep ? geometric(rng_at(key, ctr++), p_keep) : geometric(rng_at(key, ctr++), p_mut);
    if (s <= 0.0) run = L;
    const int64_t e = min(L, j + run);
    if (keep) {
      for (; j < e; ++j) d[j] = p[j];
    } else {
      for (; j < e; ++j) d[j] = (int32_t)(rng_at(key, ctr++) % (uint64_t)vocab);
    }
    keep = !keep;
  }
}

}  // namespace route

extern "C" int hs_pack_rows(const int32_t* d_src, int64_t src_stride, const int32_t* d_row, const int64_t* d_len,
                            const int64_t* d_dst_off, int32_t n, int32_t* d_dst, hs_stream_t stream) {
  if (n < 0 || src_stride < 0) {
    hs_set_error("hs_pack_rows: n and src_stride must be >= 0");
    return HS_ERR_INVALID;
  }
  if (n == 0) return HS_OK;
  hs_count_launches(1);
  const int grid = n < 4 * hs::kNumSMs ? n : 4 * hs::kNumSMs;
  route::k_pack_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(d_src, src_stride, d_row, d_len, d_dst_off, n, d_dst);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_mutate_bursts(const int32_t* d_src, const int64_t* d_src_off, int32_t n, int32_t G, double s,
                                double burst, int32_t vocab, uint64_t seed, int32_t* d_dst, int64_t* d_reward_fx,
                                hs_stream_t stream) {
  if (n < 0 || G < 1 || !(s >= 0.0 && s <= 1.0) || !(burst >= 1.0) || vocab < 1) {
    hs_set_error("hs_mutate_bursts: n >= 0, G >= 1, s in [0, 1], burst >= 1, vocab >= 1 required");
    return HS_ERR_INVALID;
  }
  if (n == 0) return HS_OK;
  hs_count_launches(1);
  const int64_t threads = (int64_t)n * G;
  route::k_mutate_bursts<<<(unsigned)((threads + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      d_src, d_src_off, n, G, s, burst, vocab, seed, d_dst, d_reward_fx);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}
