// K3: verify-forward GEMMs on tcgen05 (sm_100a), persistent and warp-specialized.
//
//   Y[M, N] = X[M, K] . W[N, K]^T     (bf16 in, fp32 accumulate in TMEM)
//
// grid = #SMs; each CTA walks tiles t = blockIdx.x, blockIdx.x + gridDim.x, ...
// (m fastest, so concurrently running CTAs share the W tile in L2).
//   warp 0      TMA producer: 128B-swizzled K-major tiles of X and W into a
//               kStages-deep smem ring (full/empty mbarriers)
//   warp 1      TMEM owner + MMA issuer: one elected thread issues
//               tcgen05.mma (M=128, N=BN, K=16) per 16-wide K slice into one of
//               two TMEM accumulators, commits each smem stage back to the
//               producer and each finished accumulator to the epilogue
//   warps 2-9   epilogue: tcgen05.ld (TMEM lane = output row), fused op,
//               global store, then release the accumulator -- overlapping the
//               next tile's main loop.  Two warps per TMEM lane quadrant take
//               alternate 32-column chunks, so the epilogue of a CTA's last
//               tile (exposed when a CTA owns only 1-3 tiles, as the
//               verify-sized QKV / O / down GEMMs do) takes half as long
// Fused epilogues:
//   EPI_STORE    bf16 out (+ bias)                         QKV (bias), generic
//   EPI_SWIGLU   silu(gate) * up, W rows interleaved in BN/2 halves
//   EPI_RESIDUAL fp32 residual += acc (read-modify-write)
//   EPI_F32      fp32 out = acc                            O-proj, down-proj (add fused into RMSNorm)
//   EPI_ARGMAX   per-row (max, first argmax) partial per 128-column tile
//
// Batch invariance (bit-exact greedy under speculation): BN is a function of
// N only, the K loop of every tile runs in the same order, there is no split-K,
// and the live row count only decides how many tiles exist -- so a row's bits
// never depend on M or on the other rows.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>

#include "../../include/hsmodel.h"
#include "hm_ptx.cuh"

void hm_set_error(const char* msg);
void hm_count_launches(int64_t n);
int hm_cap(int n_sms, bool attn);

namespace hm {

constexpr int BM = 128;
constexpr int BK = 64;           // 64 bf16 = 128 B = one swizzle row
constexpr int kEpiWarps = 8;     // two warps per TMEM lane quadrant, splitting the tile's columns
constexpr int kThreads = 64 + 32 * kEpiWarps;   // TMA warp, MMA warp, epilogue warps

enum { EPI_STORE = 0, EPI_SWIGLU = 1, EPI_RESIDUAL = 2, EPI_ARGMAX = 3, EPI_F32 = 4, EPI_ROPE = 5 };

struct EpiParams {
  int M, N, K;
  const __nv_bfloat16* bias;   // [N] or null
  __nv_bfloat16* out;          // STORE: [M, ldo]; SWIGLU: [M, N/2]
  int ldo;
  float* resid;                // RESIDUAL: [M, ldr] fp32
  int ldr;
  float* amax_val;             // ARGMAX: [M, N/128]
  int* amax_idx;
  int n_amax_tiles;
  const int* m_dev;            // optional device-side M (CUDA-graph friendly)
  // ARGMAX sampling mode (inv_temp > 0): per-row RNG keys (sequence slot, position)
  const int* key0;
  const int* key1;
  unsigned long long seed;
  float inv_temp;
  // ROPE (fused QKV projection + RoPE + KV append): columns are H q heads, KVH k heads, KVH v heads of hd
  const int* pos;              // [M] position of each row
  const int* row_slot;         // [M] KV-cache slot of each row
  const float* cos_t;          // [max_pos, hd/2]
  const float* sin_t;
  __nv_bfloat16* q_out;        // [KVH][ldq rows][G][hd]
  __nv_bfloat16* kcache;       // [slot][KVH][max_len][hd]
  __nv_bfloat16* vcache;
  long long slot_stride;
  int H, KVH, hd, max_len, ldq;
};

// rotate-half RoPE pair, rounding pinned (hm_rope_kv_append computes the same bits)
__device__ __forceinline__ void rope_pair(float a, float b, float c, float s, float& ra, float& rb) {
  ra = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
  rb = __fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s));
}

// Counter-based hash RNG for Gumbel-max sampling: the noise of vocabulary entry v
// at (seed, sequence, position) is a pure function of those four integers, so a
// row samples the same token whatever else is in the batch.
__device__ __forceinline__ uint64_t mix_u64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27; x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}
__device__ __forceinline__ uint64_t gumbel_row_key(uint64_t seed, int k0, int k1) {
  return mix_u64(seed ^ mix_u64(((uint64_t)(uint32_t)k0 << 32) | (uint32_t)k1));
}
// u from the top 23 bits: (k + 0.5) * 2^-23, k < 2^23, is exact in fp32 and lies in [2^-24, 1 - 2^-24], so
// it never rounds to 0 or 1 (a 32-bit h converted to float rounds to 2^32 for the top 128 values, giving
// u = 1 and an infinite Gumbel value that wins the argmax).  The inner log is the accurate logf: near u = 1,
// -log(u) ~ 1 - u is tiny and __logf's absolute error could make it <= 0 (NaN / inf after the outer log).
__device__ __forceinline__ float gumbel(uint64_t rkey, int v) {
  const uint32_t h = (uint32_t)(mix_u64(rkey + (uint64_t)(uint32_t)v * 0x9E3779B97F4A7C15ULL) >> 41);
  const float u = ((float)h + 0.5f) * 1.1920928955078125e-07f;   // [2^-24, 1 - 2^-24]
  return -__logf(-logf(u));
}

template <int BN, int kStages>
struct Cfg {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;    // double-buffered accumulator
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// v[i] += bias[i], i < 32 (16-byte loads; the same fp32 adds as element-wise)
__device__ __forceinline__ void add_bias32(float* v, const __nv_bfloat16* bias) {
  const uint4* b4 = reinterpret_cast<const uint4*>(bias);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 w = b4[j];
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&u[e]);
      v[8 * j + 2 * e] += __low2float(h);
      v[8 * j + 2 * e + 1] += __high2float(h);
    }
  }
}
__device__ __forceinline__ void add_bias16(float* v, const __nv_bfloat16* bias) {
  const uint4* b4 = reinterpret_cast<const uint4*>(bias);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint4 w = b4[j];
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&u[e]);
      v[8 * j + 2 * e] += __low2float(h);
      v[8 * j + 2 * e + 1] += __high2float(h);
    }
  }
}
__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst_, const float* v) {
  uint4* dst = reinterpret_cast<uint4*>(dst_);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uint4 w;
    w.x = pack_bf16(v[8 * i + 0], v[8 * i + 1]);
    w.y = pack_bf16(v[8 * i + 2], v[8 * i + 3]);
    w.z = pack_bf16(v[8 * i + 4], v[8 * i + 5]);
    w.w = pack_bf16(v[8 * i + 6], v[8 * i + 7]);
    dst[i] = w;
  }
}
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst_, const float* v) {
  uint4* dst = reinterpret_cast<uint4*>(dst_);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 w;
    w.x = pack_bf16(v[8 * i + 0], v[8 * i + 1]);
    w.y = pack_bf16(v[8 * i + 2], v[8 * i + 3]);
    w.z = pack_bf16(v[8 * i + 4], v[8 * i + 5]);
    w.w = pack_bf16(v[8 * i + 6], v[8 * i + 7]);
    dst[i] = w;
  }
}

// Epilogue of one accumulator tile for one epilogue warp: its 32 rows (TMEM lanes from t_row), the
// alternate 32-column chunks of `part`.  Shared by the 1-CTA and the CTA-pair kernels.
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(const EpiParams& p, uint32_t t_row, int row, bool live, int n_blk,
                                              int cmax, int part) {
  if constexpr (EPI == EPI_STORE || EPI == EPI_RESIDUAL || EPI == EPI_F32) {
#pragma unroll 1
    for (int c = 32 * part; c < cmax; c += 64) {
      float v[32];
      tmem_ld32(t_row + c, v);
      const int col0 = n_blk * BN + c;
      if (p.bias) add_bias32(v, p.bias + col0);
      if (live) {
        if constexpr (EPI == EPI_STORE) {
          store_bf16x32(p.out + (size_t)row * p.ldo + col0, v);
        } else if constexpr (EPI == EPI_F32) {
          // fire-and-forget fp32 store (the residual add is fused into the next RMSNorm)
          float4* dst = reinterpret_cast<float4*>(p.resid + (size_t)row * p.ldr + col0);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
          float4* dst = reinterpret_cast<float4*>(p.resid + (size_t)row * p.ldr + col0);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 r = dst[i];
            r.x += v[4 * i + 0];
            r.y += v[4 * i + 1];
            r.z += v[4 * i + 2];
            r.w += v[4 * i + 3];
            dst[i] = r;
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_ROPE) {
    // q/k/v heads of this tile: bias, round to bf16 (the unfused path's qkv activations), rotate q and
    // k at the row's position, write q kv-group-major and k, v into the cache
    const int hd = p.hd, half = hd / 2, G = p.H / p.KVH;
    const int pos = live ? p.pos[row] : 0;
    const long long slot = live ? p.row_slot[row] : 0;
    // work units (head in tile, 32-column chunk of its first half), alternating between the two parts.  For
    // hd in {64, 128} a warp's chunk is the same for every head (units step by 2, chunks per head is 1 or 2),
    // so the row's cos / sin for that chunk are loaded once per tile, before the first TMEM load: their
    // latency overlaps it instead of following it for every head
    const int chunks = half / 32;
    const int units = (cmax / hd) * chunks;
    const int c = (part % chunks) * 32;
    float cc[32], ss[32];
    if (live) {
      const float4* cs = reinterpret_cast<const float4*>(p.cos_t + (size_t)pos * half + c);
      const float4* sn = reinterpret_cast<const float4*>(p.sin_t + (size_t)pos * half + c);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 c4 = cs[j], s4 = sn[j];
        cc[4 * j] = c4.x; cc[4 * j + 1] = c4.y; cc[4 * j + 2] = c4.z; cc[4 * j + 3] = c4.w;
        ss[4 * j] = s4.x; ss[4 * j + 1] = s4.y; ss[4 * j + 2] = s4.z; ss[4 * j + 3] = s4.w;
      }
    }
#pragma unroll 1
    for (int u = part; u < units; u += 2) {
      const int hc = (u / chunks) * hd;
      const int head = (n_blk * BN + hc) / hd;   // 0..H+2KVH-1
      __nv_bfloat16* dst;
      if (head < p.H)
        dst = p.q_out + (((size_t)(head / G) * p.ldq + row) * G + head % G) * hd;
      else if (head < p.H + p.KVH)
        dst = p.kcache + slot * p.slot_stride + ((size_t)(head - p.H) * p.max_len + pos) * hd;
      else
        dst = p.vcache + slot * p.slot_stride + ((size_t)(head - p.H - p.KVH) * p.max_len + pos) * hd;
      const bool rot = head < p.H + p.KVH;
      // two 16-column halves of the chunk (register budget: cos / sin stay live across the head loop)
#pragma unroll
      for (int h16 = 0; h16 < 32; h16 += 16) {
        float a[16], b[16];
        tmem_ld16(t_row + hc + c + h16, a);
        tmem_ld16(t_row + hc + half + c + h16, b);
        const int col = n_blk * BN + hc + c + h16;
        if (p.bias) {
          add_bias16(a, p.bias + col);
          add_bias16(b, p.bias + col + half);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          a[i] = __bfloat162float(__float2bfloat16_rn(a[i]));
          b[i] = __bfloat162float(__float2bfloat16_rn(b[i]));
        }
        if (rot && live) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float ra, rb;
            rope_pair(a[i], b[i], cc[h16 + i], ss[h16 + i], ra, rb);
            a[i] = ra;
            b[i] = rb;
          }
        }
        if (live) {
          store_bf16x16(dst + c + h16, a);
          store_bf16x16(dst + half + c + h16, b);
        }
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU) {
    constexpr int H = BN / 2;
#pragma unroll 1
    for (int c = 32 * part; c < H; c += 64) {
      float g[32], u[32];
      tmem_ld32(t_row + c, g);
      tmem_ld32(t_row + H + c, u);
#pragma unroll
      for (int i = 0; i < 32; ++i) g[i] = silu(g[i]) * u[i];
      if (live) store_bf16x32(p.out + (size_t)row * p.ldo + n_blk * H + c, g);
    }
  } else {  // EPI_ARGMAX: one partial per 128 columns
    // sampling (inv_temp > 0): Gumbel-max over logit/T + g(seed, key0[row], key1[row], col)
    const bool sample = p.inv_temp > 0.f && live;
    uint64_t rkey = 0;
    if (sample) rkey = gumbel_row_key(p.seed, p.key0[row], p.key1[row]);
#pragma unroll 1
    for (int h = 128 * part; h < cmax; h += 256) {
      float best = -INFINITY;
      int bidx = 0;
#pragma unroll 1
      for (int c = h; c < h + 128; c += 32) {
        float v[32];
        tmem_ld32(t_row + c, v);
        if (sample) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = v[i] * p.inv_temp + gumbel(rkey, n_blk * BN + c + i);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (v[i] > best) { best = v[i]; bidx = n_blk * BN + c + i; }   // strict: first max wins
        }
      }
      if (live) {
        const int tile128 = (n_blk * BN + h) / 128;
        p.amax_val[(size_t)row * p.n_amax_tiles + tile128] = best;
        p.amax_idx[(size_t)row * p.n_amax_tiles + tile128] = bidx;
      }
    }
  }
}

template <int BN, int kStages, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, EpiParams p) {
  using C = Cfg<BN, kStages>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = p.m_dev ? *p.m_dev : p.M;
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (p.N + BN - 1) / BN;
  const int total = m_tiles * n_tiles;
  if ((int)blockIdx.x >= total) return;   // uniform across the CTA
  const int num_k = p.K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps);   // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmW);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;   // global k-block counter (ring position)
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m_blk = t % m_tiles, n_blk = t / m_tiles;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* a = smem + s * C::kStageBytes;
          uint8_t* b = a + C::kABytes;
          mbar_arrive_expect_tx(&full[s], C::kStageBytes);
          tma_load_2d(&tmX, &full[s], a, kb * BK, m_blk * BM);
          tma_load_2d(&tmW, &full[s], b, kb * BK, n_blk * BN);   // (evict-first W measured slower)
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      uint32_t it = 0;
      int local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int buf = local & 1;
        const uint32_t use = (uint32_t)(local >> 1);
        mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * BN);
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint8_t* a = smem + s * C::kStageBytes;
          const uint8_t* b = a + C::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_f16(d, smem_desc_sw128(a + k * 32), smem_desc_sw128(b + k * 32), idesc, (kb | k) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // epilogue warps 2..9 -> TMEM lane quadrant (warp % 4); `part` picks alternate 32-column chunks
    const int q = warp & 3;
    const int part = (warp - 2) >> 2;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int m_blk = t % m_tiles, n_blk = t / m_tiles;
      const int buf = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      mbar_wait(&acc_full[buf], use & 1);
      tc_fence_after();
      const uint32_t t_row = tmem + (uint32_t)(buf * BN) + ((uint32_t)(q * 32) << 16);
      const int row = m_blk * BM + q * 32 + lane;
      const bool live = row < M;
      // a last N tile may be half empty (N % 128 == 0, BN = 256): W rows past N were zero-filled by TMA
      const int cmax = min(BN, p.N - n_blk * BN);
      epilogue_tile<BN, EPI>(p, t_row, row, live, n_blk, cmax, part);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 256 tile.  Each CTA
// stages its own 128 rows of X and 128 rows (of N) of W per K block -- 32 KB instead of the 48 KB a 1-CTA
// 128 x 256 tile needs -- and the leader's single MMA thread issues M = 256, N = 256, K = 16 MMAs that read
// both CTAs' shared memory; each CTA's TMEM holds its 128 rows x 256 columns.  The per-SM operand traffic
// from L2, which bounds the 1-CTA kernel (~100 GB/s per SM), drops by a third.
//   leader  (rank 0): TMA warp arms full[s] for both CTAs' bytes; MMA warp; epilogue warps
//   peer    (rank 1): TMA warp (signals the leader's full[s]); epilogue warps (arrive on the leader's
//                     acc_empty)
// Both CTAs' empty[s] and acc_full[b] receive the leader's multicast commits.  Same per-element MMA sequence
// as the 1-CTA kernel (K = 16 steps in order, no split-K): a row's bits do not depend on the variant
// (tests/test_model_gpu.py::test_gemm_pair_is_bit_neutral).
template <int kStages, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
k_gemm_pair(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, EpiParams p) {
  constexpr int BN = 256;
  constexpr int kHalfBytes = 128 * BK * 2;        // 16 KB: 128 rows x 64 bf16
  constexpr int kStageBytes = 2 * kHalfBytes;     // this CTA's X rows + W rows
  constexpr uint32_t kTmemCols = 2 * BN;          // double-buffered 128 x 256 accumulator per CTA
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2], used in the leader only
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int M = p.m_dev ? *p.m_dev : p.M;
  const int m_tiles = (M + 255) / 256;
  const int n_tiles = (p.N + BN - 1) / BN;
  const int total = m_tiles * n_tiles;
  if (pair >= total) return;   // uniform across the cluster
  const int num_k = p.K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);     // leader: its producer's arrive (+ both CTAs' bytes); peer: unused
      mbar_init(&empty[s], 1);    // the leader's multicast commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * kEpiWarps);   // every epilogue warp of both CTAs
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<kTmemCols>(tmem_slot);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmW);
  }
  tc_fence_before();
  cluster_sync();   // barriers initialised and TMEM allocated in both CTAs before any cross-CTA traffic
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = pair; t < total; t += n_pairs) {
        const int m_blk = t % m_tiles, n_blk = t / m_tiles;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* a = smem + s * kStageBytes;
          uint8_t* b = a + kHalfBytes;
          const uint32_t bar = mapa_shared(&full[s], 0);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kStageBytes);
          tma_load_2d_pair(&tmX, bar, a, kb * BK, m_blk * 256 + (int)rank * 128);
          tma_load_2d_pair(&tmW, bar, b, kb * BK, n_blk * BN + (int)rank * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(256, BN);
      uint32_t it = 0;
      int local = 0;
      for (int t = pair; t < total; t += n_pairs, ++local) {
        const int buf = local & 1;
        const uint32_t use = (uint32_t)(local >> 1);
        mbar_wait_cluster(&acc_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * BN);
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint8_t* a = smem + s * kStageBytes;
          const uint8_t* b = a + kHalfBytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_f16_pair(d, smem_desc_sw128(a + k * 32), smem_desc_sw128(b + k * 32), idesc, (kb | k) != 0);
          umma_commit_pair(&empty[s], 0x3);
        }
        umma_commit_pair(&acc_full[buf], 0x3);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int part = (warp - 2) >> 2;
    const uint32_t release = mapa_shared(&acc_empty[0], 0);
    int local = 0;
    for (int t = pair; t < total; t += n_pairs, ++local) {
      const int m_blk = t % m_tiles, n_blk = t / m_tiles;
      const int buf = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      mbar_wait(&acc_full[buf], use & 1);
      tc_fence_after();
      const uint32_t t_row = tmem + (uint32_t)(buf * BN) + ((uint32_t)(q * 32) << 16);
      const int row = m_blk * 256 + (int)rank * 128 + q * 32 + lane;
      const bool live = row < M;
      const int cmax = min(BN, p.N - n_blk * BN);
      epilogue_tile<BN, EPI>(p, t_row, row, live, n_blk, cmax, part);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(release + (uint32_t)(buf * sizeof(uint64_t)));
    }
  }
  tc_fence_before();
  cluster_sync();   // both CTAs' epilogues finished reading TMEM, the leader's MMAs retired
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<kTmemCols>(tmem);
  }
}

// final argmax over the per-tile partials (tiles in column order; ties -> smallest index)
__global__ void k_argmax_reduce(const float* __restrict__ val, const int* __restrict__ idx, int M, int n_tiles,
                                const int* m_dev, int* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int m = m_dev ? *m_dev : M;
  for (int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); row < m; row += gridDim.x * (blockDim.x / 32)) {
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = lane; t < n_tiles; t += 32) {
    float v = val[(size_t)row * n_tiles + t];
    int i = idx[(size_t)row * n_tiles + t];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (lane == 0) out[row] = bi;
  }
}

}  // namespace hm

// ------------------------------------------------------------------ host side
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// rows x cols bf16 row-major (cols contiguous), box = box_rows x 64 cols, 128B swizzle
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;

}  // namespace

bool hm_make_tma_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  return make_map(m, base, rows, cols, ld, box_rows);
}

namespace {

template <int BN, int kStages, int EPI>
int launch(const CUtensorMap& mx, const CUtensorMap& mw, const hm::EpiParams& p, cudaStream_t st) {
  using C = hm::Cfg<BN, kStages>;
  auto kern = hm::k_gemm<BN, kStages, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes) != cudaSuccess) {
      hm_set_error("cudaFuncSetAttribute(smem) failed");
      return HM_ERR_CUDA;
    }
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = ((p.M + hm::BM - 1) / hm::BM) * ((p.N + BN - 1) / BN);
  const int cap = hm_cap(g_num_sms, false);
  const int grid = tiles < cap ? tiles : cap;
  hm_count_launches(1);
  kern<<<grid, hm::kThreads, C::kSmemBytes, st>>>(mx, mw, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    hm_set_error(cudaGetErrorString(e));
    return HM_ERR_CUDA;
  }
  return HM_OK;
}

constexpr int kPairStages = 6;
constexpr int kPairSmem = kPairStages * 2 * (128 * hm::BK * 2) + 1024 + 256;

template <int EPI>
int launch_pair(const CUtensorMap& mx, const CUtensorMap& mw, const hm::EpiParams& p, cudaStream_t st) {
  auto kern = hm::k_gemm_pair<kPairStages, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem) != cudaSuccess) {
      hm_set_error("cudaFuncSetAttribute(smem) failed");
      return HM_ERR_CUDA;
    }
    attr_set = true;
  }
  const int tiles = ((p.M + 255) / 256) * ((p.N + 255) / 256);
  const int cap = hm_cap(g_num_sms, false) / 2;
  const int pairs = tiles < cap ? tiles : cap;
  hm_count_launches(1);
  kern<<<2 * pairs, hm::kThreads, kPairSmem, st>>>(mx, mw, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    hm_set_error(cudaGetErrorString(e));
    return HM_ERR_CUDA;
  }
  return HM_OK;
}

}  // namespace

// CTA-pair kernels on (1, default; HM_GEMM_PAIR=0 in the environment starts with them off) or off (0)
static int g_gemm_pair = (getenv("HM_GEMM_PAIR") && atoi(getenv("HM_GEMM_PAIR")) == 0) ? 0 : 1;

extern "C" int hm_set_gemm_pair(int32_t on) {
  if (on != 0 && on != 1) {
    hm_set_error("hm_set_gemm_pair: 0 or 1");
    return HM_ERR_INVALID;
  }
  g_gemm_pair = on;
  return HM_OK;
}

extern "C" int hm_gemm_bn(int32_t n) {
  // tile width is a function of N only (batch invariance): 256 for wide N (a last tile may be half
  // empty when N % 256 == 128, e.g. the 151,936-entry LM head), 128 otherwise.  N up to
  // HM_GEMM_BN128_MAX also uses 128 (A/B of the wave quantisation of narrow GEMMs)
  static const int bn128_max = getenv("HM_GEMM_BN128_MAX") ? atoi(getenv("HM_GEMM_BN128_MAX")) : 0;
  return (n >= 1536 && n > bn128_max) ? 256 : 128;
}

static int gemm_impl(int32_t epi, const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N,
                     int32_t K, const void* d_bias, void* d_out, int64_t ldo, float* d_resid, int64_t ldr,
                     float* d_amax_val, int32_t* d_amax_idx, const int32_t* d_m, const int32_t* key0,
                     const int32_t* key1, uint64_t seed, float inv_temp, hm_stream_t stream,
                     const hm::EpiParams* rope = nullptr);

extern "C" int hm_gemm(int32_t epi, const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N,
                       int32_t K, const void* d_bias, void* d_out, int64_t ldo, float* d_resid, int64_t ldr,
                       float* d_amax_val, int32_t* d_amax_idx, const int32_t* d_m, hm_stream_t stream) {
  return gemm_impl(epi, d_x, ldx, d_w, ldw, M, N, K, d_bias, d_out, ldo, d_resid, ldr, d_amax_val, d_amax_idx, d_m,
                   nullptr, nullptr, 0, 0.f, stream);
}

extern "C" int hm_lm_head_sample(const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N,
                                 int32_t K, const int32_t* d_key0, const int32_t* d_key1, uint64_t seed,
                                 float temperature, float* d_amax_val, int32_t* d_amax_idx, const int32_t* d_m,
                                 hm_stream_t stream) {
  if (!(temperature > 0.f)) {
    hm_set_error("hm_lm_head_sample: temperature must be > 0 (use HM_EPI_ARGMAX for greedy)");
    return HM_ERR_INVALID;
  }
  return gemm_impl(HM_EPI_ARGMAX, d_x, ldx, d_w, ldw, M, N, K, nullptr, nullptr, 0, nullptr, 0, d_amax_val,
                   d_amax_idx, d_m, d_key0, d_key1, seed, 1.f / temperature, stream);
}

static int gemm_impl(int32_t epi, const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N,
                     int32_t K, const void* d_bias, void* d_out, int64_t ldo, float* d_resid, int64_t ldr,
                     float* d_amax_val, int32_t* d_amax_idx, const int32_t* d_m, const int32_t* key0,
                     const int32_t* key1, uint64_t seed, float inv_temp, hm_stream_t stream,
                     const hm::EpiParams* rope) {
  if (M <= 0) return HM_OK;
  if (K % hm::BK != 0 || N % 128 != 0) {
    hm_set_error("hm_gemm: K must be a multiple of 64 and N of 128");
    return HM_ERR_INVALID;
  }
  int BN = hm_gemm_bn(N);
  // Plain and fp32 epilogues may narrow the tile when 256-wide tiles would leave SMs idle (decode-sized M):
  // every output element's K reduction is the same sequence of K=16 MMA steps at either width, so a row's
  // bits do not change (tests/test_model_gpu.py::test_gemm_tile_width_is_bit_neutral); SwiGLU's weight
  // interleave and the argmax partials are laid out per hm_gemm_bn(N) and keep it.
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static const int narrow_off = getenv("HM_GEMM_NO_NARROW") != nullptr;   // A/B switch for profiling only
  if (BN == 256 && !narrow_off &&
      (epi == HM_EPI_STORE || epi == HM_EPI_F32 || epi == HM_EPI_RESIDUAL || epi == hm::EPI_ROPE) &&
      ((M + hm::BM - 1) / hm::BM) * ((N + 255) / 256) < g_num_sms)
    BN = 128;
  if (epi == HM_EPI_SWIGLU && N % BN != 0) {
    hm_set_error("hm_gemm: SwiGLU needs N to be a multiple of the tile width (interleave granularity)");
    return HM_ERR_INVALID;
  }
  // CTA pairs for 256-wide tiles when there are enough 256 x 256 tiles to give every pair one (a row's bits
  // are the same in either kernel); HM_GEMM_PAIR=0 turns them off (A/B switch)
  const bool pair = BN == 256 && g_gemm_pair && ((M + 255) / 256) * ((N + 255) / 256) >= hm_cap(g_num_sms, false) / 2;
  CUtensorMap mx, mw;
  if (!make_map(&mx, d_x, M, K, ldx, hm::BM) || !make_map(&mw, d_w, N, K, ldw, pair ? 128 : BN)) {
    hm_set_error("cuTensorMapEncodeTiled failed (alignment: base 16 B, ld multiple of 8 elements)");
    return HM_ERR_INVALID;
  }
  hm::EpiParams p{};
  if (rope) p = *rope;
  p.M = M;
  p.N = N;
  p.K = K;
  p.bias = static_cast<const __nv_bfloat16*>(d_bias);
  p.out = static_cast<__nv_bfloat16*>(d_out);
  p.ldo = (int)ldo;
  p.resid = d_resid;
  p.ldr = (int)ldr;
  p.amax_val = d_amax_val;
  p.amax_idx = d_amax_idx;
  p.n_amax_tiles = N / 128;
  p.m_dev = d_m;
  p.key0 = key0;
  p.key1 = key1;
  p.seed = seed;
  p.inv_temp = inv_temp;
  cudaStream_t st = (cudaStream_t)stream;
  if (pair) {
    switch (epi) {
      case HM_EPI_STORE: return launch_pair<hm::EPI_STORE>(mx, mw, p, st);
      case HM_EPI_SWIGLU: return launch_pair<hm::EPI_SWIGLU>(mx, mw, p, st);
      case HM_EPI_RESIDUAL: return launch_pair<hm::EPI_RESIDUAL>(mx, mw, p, st);
      case HM_EPI_F32: return launch_pair<hm::EPI_F32>(mx, mw, p, st);
      case HM_EPI_ARGMAX: return launch_pair<hm::EPI_ARGMAX>(mx, mw, p, st);
      case hm::EPI_ROPE: return launch_pair<hm::EPI_ROPE>(mx, mw, p, st);
    }
  } else if (BN == 256) {
    switch (epi) {
      case HM_EPI_STORE: return launch<256, 4, hm::EPI_STORE>(mx, mw, p, st);
      case HM_EPI_SWIGLU: return launch<256, 4, hm::EPI_SWIGLU>(mx, mw, p, st);
      case HM_EPI_RESIDUAL: return launch<256, 4, hm::EPI_RESIDUAL>(mx, mw, p, st);
      case HM_EPI_F32: return launch<256, 4, hm::EPI_F32>(mx, mw, p, st);
      case HM_EPI_ARGMAX: return launch<256, 4, hm::EPI_ARGMAX>(mx, mw, p, st);
      case hm::EPI_ROPE: return launch<256, 4, hm::EPI_ROPE>(mx, mw, p, st);
    }
  } else {
    switch (epi) {
      case HM_EPI_STORE: return launch<128, 6, hm::EPI_STORE>(mx, mw, p, st);
      case HM_EPI_SWIGLU: return launch<128, 6, hm::EPI_SWIGLU>(mx, mw, p, st);
      case HM_EPI_RESIDUAL: return launch<128, 6, hm::EPI_RESIDUAL>(mx, mw, p, st);
      case HM_EPI_F32: return launch<128, 6, hm::EPI_F32>(mx, mw, p, st);
      case HM_EPI_ARGMAX: return launch<128, 6, hm::EPI_ARGMAX>(mx, mw, p, st);
      case hm::EPI_ROPE: return launch<128, 6, hm::EPI_ROPE>(mx, mw, p, st);
    }
  }
  hm_set_error("unknown epilogue");
  return HM_ERR_INVALID;
}

extern "C" int hm_gemm_qkv_rope(const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t K,
                                const void* d_bias, int32_t H, int32_t KVH, int32_t hd, const int32_t* d_pos,
                                const int32_t* d_row_slot, const float* d_cos, const float* d_sin, void* d_q,
                                int32_t q_rows, void* d_kcache, void* d_vcache, int64_t slot_stride,
                                int32_t max_len, const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (KVH <= 0 || H % KVH || (hd != 64 && hd != 128) || q_rows < M) {
    hm_set_error("hm_gemm_qkv_rope: H % KVH, hd in {64, 128} and q_rows >= M required");
    return HM_ERR_INVALID;
  }
  hm::EpiParams r{};
  r.pos = d_pos;
  r.row_slot = d_row_slot;
  r.cos_t = d_cos;
  r.sin_t = d_sin;
  r.q_out = static_cast<__nv_bfloat16*>(d_q);
  r.kcache = static_cast<__nv_bfloat16*>(d_kcache);
  r.vcache = static_cast<__nv_bfloat16*>(d_vcache);
  r.slot_stride = slot_stride;
  r.H = H;
  r.KVH = KVH;
  r.hd = hd;
  r.max_len = max_len;
  r.ldq = q_rows;
  return gemm_impl(hm::EPI_ROPE, d_x, ldx, d_w, ldw, M, (H + 2 * KVH) * hd, K, d_bias, nullptr, 0, nullptr, 0,
                   nullptr, nullptr, d_m, nullptr, nullptr, 0, 0.f, stream, &r);
}

extern "C" int hm_argmax_reduce(const float* d_val, const int32_t* d_idx, int32_t M, int32_t n_tiles,
                                const int32_t* d_m, int32_t* d_out, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  int rows_per_block = 8;
  hm_count_launches(1);
  const int blocks = (M + rows_per_block - 1) / rows_per_block;
  hm::k_argmax_reduce<<<blocks < 1184 ? blocks : 1184, 256, 0, (cudaStream_t)stream>>>(
      d_val, d_idx, M, n_tiles, d_m, d_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    hm_set_error(cudaGetErrorString(e));
    return HM_ERR_CUDA;
  }
  return HM_OK;
}
