// K4: causal GQA attention for variable-length query blocks (decode rows,
// verify blocks [last, d_1..d_k], prefill prompts) over a slot-contiguous KV
// cache.  One CTA = (query tile, kv head, sequence); its 64 rows are
// (query i, head j in the GQA group) pairs, so the group shares every K/V
// load.  K/V blocks of 64 keys are double-buffered in XOR-swizzled smem with
// cp.async; QK^T and PV run on mma.sync m16n8k16 bf16 with fp32 accumulate
// and an online softmax in the exp2 domain.
//
// Batch invariance: a row's result depends only on its own query, its
// position and the cache -- KV blocks are visited in the same order from
// position 0 for every row, blocks past a row's position are fully masked
// (exact no-ops), and there is no split-KV whose partition could move with the
// batch composition.
#include <cuda_bf16.h>
#include <stdint.h>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "../../include/hsmodel.h"
#include "hm_ptx.cuh"

void hm_set_error(const char* msg);
bool hm_make_tma_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows);
void hm_count_launches(int64_t n);
int hm_cap(int n_sms, bool attn);

namespace hm {

constexpr int AT_ROWS = 64;   // rows per CTA (4 warps x 16)
constexpr int AT_KEYS = 64;   // keys per block

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// [rows][HD] bf16 tile, 16-byte chunks XOR-swizzled by (row & 7)
template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {
  return row * (HD / 8) + (chunk ^ (row & 7));
}

template <int HD>
__global__ void __launch_bounds__(128) k_attention(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                                                   const __nv_bfloat16* __restrict__ vc, int64_t slot_stride,
                                                   const int32_t* __restrict__ q_off, const int32_t* __restrict__ q_len,
                                                   const int32_t* __restrict__ pos0, const int32_t* __restrict__ kv_slot,
                                                   int H, int KVH, int q_rows, int max_len, float scale_log2,
                                                   __nv_bfloat16* __restrict__ out) {
  constexpr int CH = HD / 8;   // 16-byte chunks per row
  const int tile = blockIdx.x, kvh = blockIdx.y, s = blockIdx.z;
  const int G = H / KVH;
  const int ql = q_len[s];
  const int rows_total = ql * G;
  if (tile * AT_ROWS >= rows_total) return;
  const int qo = q_off[s], p0 = pos0[s];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  extern __shared__ __align__(128) uint8_t sm[];
  uint4* sQ = reinterpret_cast<uint4*>(sm);                       // [64][HD]
  uint4* sK = sQ + AT_ROWS * CH;                                    // [2][64][HD]
  uint4* sV = sK + 2 * AT_KEYS * CH;                                // [2][64][HD]

  // ---- stage Q rows (row r -> query r / G, head kvh * G + r % G)
  for (int c = threadIdx.x; c < AT_ROWS * CH; c += blockDim.x) {
    const int r = c / CH, ch = c % CH;
    const int rr = tile * AT_ROWS + r;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (rr < rows_total) {
      v = reinterpret_cast<const uint4*>(q + ((size_t)(kvh * q_rows + qo) * G + rr) * HD)[ch];   // [KVH][rows][G][hd]
    }
    sQ[swz<HD>(r, ch)] = v;
  }
  // max position among this tile's rows
  const int last_row = min(rows_total, (tile + 1) * AT_ROWS) - 1;
  const int max_pos = p0 + last_row / G;
  const int n_blocks = max_pos / AT_KEYS + 1;
  const __nv_bfloat16* kbase = kc + (size_t)kv_slot[s] * slot_stride + (size_t)kvh * max_len * HD;
  const __nv_bfloat16* vbase = vc + (size_t)kv_slot[s] * slot_stride + (size_t)kvh * max_len * HD;

  auto load_kv = [&](int blk, int buf) {
    for (int c = threadIdx.x; c < AT_KEYS * CH; c += blockDim.x) {
      const int r = c / CH, ch = c % CH;
      const int key = blk * AT_KEYS + r;
      const bool ok = key <= max_pos;
      const size_t off = (size_t)(ok ? key : 0) * HD + ch * 8;
      cp_async16(&sK[buf * AT_KEYS * CH + swz<HD>(r, ch)], kbase + off, ok);
      cp_async16(&sV[buf * AT_KEYS * CH + swz<HD>(r, ch)], vbase + off, ok);
    }
    cp_commit();
  };
  load_kv(0, 0);
  __syncthreads();

  // ---- Q fragments (A operand) for this warp's 16 rows
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int r = warp * 16 + (lane & 15);
    const int ch = kk * 2 + (lane >> 4);
    ldsm_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], &sQ[swz<HD>(r, ch)]);
  }
  // rows owned by this thread in the C layout
  const int r0 = tile * AT_ROWS + warp * 16 + (lane >> 2);
  const int r1 = r0 + 8;
  const int rpos0 = r0 < rows_total ? p0 + r0 / G : -1;   // -1 => padding row (fully masked)
  const int rpos1 = r1 < rows_total ? p0 + r1 / G : -1;

  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int blk = 0; blk < n_blocks; ++blk) {
    const int buf = blk & 1;
    if (blk + 1 < n_blocks) {
      load_kv(blk + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint4* K = sK + buf * AT_KEYS * CH;
    const uint4* V = sV + buf * AT_KEYS * CH;
    // S = Q K^T : 16 x 64 per warp (8 n-tiles of 8 keys)
    float sc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t b0, b1, b2, b3;
        const int key = j * 8 + (lane & 7);
        const int ch = c * 4 + (lane >> 3);
        ldsm_x4(b0, b1, b2, b3, &K[swz<HD>(key, ch)]);
        mma16816(sc[j], qf[2 * c], b0, b1);
        mma16816(sc[j], qf[2 * c + 1], b2, b3);
      }
    }
    // mask + online softmax (log2 domain)
    float bm0 = -INFINITY, bm1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kbase_ = blk * AT_KEYS + j * 8 + 2 * (lane & 3);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = kbase_ + e;
        sc[j][e] = key <= rpos0 ? sc[j][e] * scale_log2 : -INFINITY;
        sc[j][2 + e] = key <= rpos1 ? sc[j][2 + e] * scale_log2 : -INFINITY;
        bm0 = fmaxf(bm0, sc[j][e]);
        bm1 = fmaxf(bm1, sc[j][2 + e]);
      }
    }
    bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 1));
    bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
    bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 1));
    bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
    const float nm0 = fmaxf(m0, bm0), nm1 = fmaxf(m1, bm1);
    const float a0 = nm0 == -INFINITY ? 1.f : exp2f(m0 - nm0);
    const float a1 = nm1 == -INFINITY ? 1.f : exp2f(m1 - nm1);
    const float sub0 = nm0 == -INFINITY ? 0.f : nm0;
    const float sub1 = nm1 == -INFINITY ? 0.f : nm1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j][0] = exp2f(sc[j][0] - sub0);
      sc[j][1] = exp2f(sc[j][1] - sub0);
      sc[j][2] = exp2f(sc[j][2] - sub1);
      sc[j][3] = exp2f(sc[j][3] - sub1);
      rs0 += sc[j][0] + sc[j][1];
      rs1 += sc[j][2] + sc[j][3];
    }
    rs0 += __shfl_xor_sync(0xffffffffu, rs0, 1);
    rs0 += __shfl_xor_sync(0xffffffffu, rs0, 2);
    rs1 += __shfl_xor_sync(0xffffffffu, rs1, 1);
    rs1 += __shfl_xor_sync(0xffffffffu, rs1, 2);
    l0 = l0 * a0 + rs0;
    l1 = l1 * a1 + rs1;
    m0 = nm0;
    m1 = nm1;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= a0;
      o[i][1] *= a0;
      o[i][2] *= a1;
      o[i][3] *= a1;
    }
    // O += P V : P (16 x 64) as A fragments, V via transposed ldmatrix
#pragma unroll
    for (int t = 0; t < 4; ++t) {   // 16 keys per k-step
      uint32_t pa[4];
      pa[0] = pack2(sc[2 * t][0], sc[2 * t][1]);
      pa[1] = pack2(sc[2 * t][2], sc[2 * t][3]);
      pa[2] = pack2(sc[2 * t + 1][0], sc[2 * t + 1][1]);
      pa[3] = pack2(sc[2 * t + 1][2], sc[2 * t + 1][3]);
#pragma unroll
      for (int n = 0; n < HD / 16; ++n) {   // two 8-dim n-tiles per ldmatrix.x4
        uint32_t b0, b1, b2, b3;
        const int key = t * 16 + (lane & 15);
        const int ch = n * 2 + (lane >> 4);
        ldsm_x4_t(b0, b1, b2, b3, &V[swz<HD>(key, ch)]);
        mma16816(o[2 * n], pa, b0, b1);
        mma16816(o[2 * n + 1], pa, b2, b3);
      }
    }
    __syncthreads();
  }

  // ---- normalize + store: row r -> out[(qo + r / G), head kvh * G + r % G, :]
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f;
  const float inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int col = i * 8 + 2 * (lane & 3);
    if (rpos0 >= 0) {
      __nv_bfloat16* dst = out + ((size_t)(qo + r0 / G) * H + kvh * G + r0 % G) * HD + col;
      *reinterpret_cast<uint32_t*>(dst) = pack2(o[i][0] * inv0, o[i][1] * inv0);
    }
    if (rpos1 >= 0) {
      __nv_bfloat16* dst = out + ((size_t)(qo + r1 / G) * H + kvh * G + r1 % G) * HD + col;
      *reinterpret_cast<uint32_t*>(dst) = pack2(o[i][2] * inv1, o[i][3] * inv1);
    }
  }
}

// ---------------------------------------------------------------------------
// v2: KV split across the 4 warps of a CTA.  A CTA owns SL m16 row slices
// (16*SL rows of (query, head-in-group)); each pipeline stage holds 64 keys
// of K and V; warp w processes keys [stage*64 + 16w, +16) for all of the
// CTA's rows with its own online-softmax state, and the 4 partial states are
// merged in warp order at the end.  Compared with v1 this computes 16*SL
// instead of 64 rows per key (30 live rows of a q=5 verify block on GQA-6:
// SL=2; decode: SL=1) and keeps every warp busy.  The key->warp map depends
// only on the key position and the merge order is fixed, so a row's result is
// independent of the batch (bit-exact greedy under speculation).
// NW = 8 (with SL = 2): eight warps, warp w = (key group w & 3, slice w >> 2) -- one 16-row slice per
// warp instead of two, half the registers, so two CTAs (16 warps) fit an SM.  The per-slice source is
// the same as NW = 4's and the rounding is pinned with explicit intrinsics, so a row's bits do not
// depend on NW (or on SL): verify blocks and decode rows still agree bit for bit.
template <int HD, int SL, int NW = 4>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 2 : 1) k_attention2(const __nv_bfloat16* __restrict__ q,
                                                    const __nv_bfloat16* __restrict__ kc,
                                                    const __nv_bfloat16* __restrict__ vc, int64_t slot_stride,
                                                    const int32_t* __restrict__ q_off,
                                                    const int32_t* __restrict__ q_len,
                                                    const int32_t* __restrict__ pos0,
                                                    const int32_t* __restrict__ kv_slot, int H, int KVH,
                                                    int q_rows, int max_len, float scale_log2,
                                                    __nv_bfloat16* __restrict__ out, int n_seq,
                                                    const int32_t* __restrict__ work,
                                                    const __grid_constant__ CUtensorMap tmK,
                                                    const __grid_constant__ CUtensorMap tmV, int use_tma, int flags) {
  constexpr int CH = HD / 8;        // 16-byte chunks per row
  constexpr int ROWS = 16 * SL;
  constexpr int KS = 64;            // keys per stage (4 warps x 16)
  constexpr int NST = 3;            // pipeline stages
  static_assert(NW == 4 || (NW == 8 && SL == 2), "8 warps: one slice each of a 2-slice tile");
  constexpr int SLW = NW == 8 ? 1 : SL;   // slices this warp computes
  const int G = H / KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kg = warp & 3;                                // key group: keys [stage * 64 + 16 kg, +16)
  const int sl_base = NW == 8 ? (warp >> 2) : 0;          // first slice of this warp
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  // TMA 128B-swizzled destinations need 1024-byte alignment (the launch adds 1 KB of slack)
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint4* sK = reinterpret_cast<uint4*>(sm);            // [NST][KS][CH]
  uint4* sV = sK + NST * KS * CH;                        // [NST][KS][CH]
  uint4* sQ = sV + NST * KS * CH;                        // [ROWS][CH]
  __shared__ uint64_t full[NST];                         // TMA stage barriers
  const bool tma = use_tma != 0;
  // K/V tile layout: TMA writes 64-key x 128 B halves with the hardware 128B swizzle
  // (16-byte chunk ^ row%8); the cp.async path uses the equivalent per-row XOR on 256 B rows
  auto kvoff = [&](int r, int ch) -> int {
    return tma ? (ch >> 3) * (KS * 8) + r * 8 + ((ch & 7) ^ (r & 7)) : swz<HD>(r, ch);
  };
  if (tma && threadIdx.x == 0) {
    for (int b = 0; b < NST; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t g_stage = 0;   // CTA-wide count of consumed TMA stages (mbarrier phase tracking)

  // one work item = (sequence, row tile, kv head)
  auto do_tile = [&](const int s, const int kvh, const int tile) {
  const int rows_total = q_len[s] * G;
  const int qo = q_off[s], p0 = pos0[s];

  for (int c = threadIdx.x; c < ROWS * CH; c += blockDim.x) {
    const int r = c / CH, ch = c % CH;
    const int rr = tile * ROWS + r;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (rr < rows_total) {
      v = reinterpret_cast<const uint4*>(q + ((size_t)(kvh * q_rows + qo) * G + rr) * HD)[ch];   // [KVH][rows][G][hd]
    }
    sQ[swz<HD>(r, ch)] = v;
  }
  const int last_row = min(rows_total, (tile + 1) * ROWS) - 1;
  const int max_pos = p0 + last_row / G;
  const int n_stage = max_pos / KS + 1;
  const __nv_bfloat16* kbase = kc + (size_t)kv_slot[s] * slot_stride + (size_t)kvh * max_len * HD;
  const __nv_bfloat16* vbase = vc + (size_t)kv_slot[s] * slot_stride + (size_t)kvh * max_len * HD;

  const int row0 = (kv_slot[s] * KVH + kvh) * max_len;   // first cache row of this (slot, kv head)
  const uint32_t g0 = g_stage;
  auto load_stage = [&](int st) {
    if (tma) {
      // one thread: 2 (HD=64) or 4 (HD=128) TMA boxes of 64 keys x 64 dims, completing on full[buf]
      const int buf = (g0 + st) % NST;
      constexpr uint32_t bytes = 2 * KS * HD * 2;
      mbar_arrive_expect_tx(&full[buf], bytes);
#pragma unroll
      for (int h = 0; h < HD / 64; ++h) {
        // K / V are read once: evict-first in L2 (same policy as the tcgen05 family)
        tma_load_2d_evict_first(&tmK, &full[buf], &sK[(buf * KS) * CH + h * KS * 8], h * 64, row0 + st * KS);
        tma_load_2d_evict_first(&tmV, &full[buf], &sV[(buf * KS) * CH + h * KS * 8], h * 64, row0 + st * KS);
      }
      return;
    }
    const int buf = st % NST;
    for (int c = threadIdx.x; c < KS * CH; c += blockDim.x) {
      const int r = c / CH, ch = c % CH;
      const int key = st * KS + r;
      const bool ok = key <= max_pos;
      const size_t off = (size_t)(ok ? key : 0) * HD + ch * 8;
      cp_async16(&sK[(buf * KS) * CH + swz<HD>(r, ch)], kbase + off, ok);
      cp_async16(&sV[(buf * KS) * CH + swz<HD>(r, ch)], vbase + off, ok);
    }
  };
  __syncthreads();
  // Q fragments are re-read from smem per sub-block (ldmatrix) instead of living in registers:
  // keeps the 32-row variant under 255 registers without spills
#pragma unroll
  for (int i = 0; i < NST - 1; ++i) {
    if (tma) {
      if (threadIdx.x == 0 && i < n_stage) load_stage(i);
    } else {
      if (i < n_stage) load_stage(i);
      cp_commit();
    }
  }
  int rpos[SLW][2];
  // per slice of this warp: live (any row < rows_total; a slice of padding rows only is skipped -- its
  // state is never merged into an output row) and vis_all (keys <= vis_all are visible to all 16 rows,
  // so their blocks skip the mask: the mask is the identity there).  Both warp-uniform, both exact.
  bool live[SLW];
  int vis_all[SLW];
#pragma unroll
  for (int sl = 0; sl < SLW; ++sl) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = tile * ROWS + (sl_base + sl) * 16 + (lane >> 2) + 8 * h;
      rpos[sl][h] = rr < rows_total ? p0 + rr / G : -1;   // -1: padding row, fully masked
    }
    const int first = tile * ROWS + (sl_base + sl) * 16;
    live[sl] = first < rows_total;
    vis_all[sl] = first + 15 < rows_total ? p0 + first / G : -1;
  }
  float o[SLW][HD / 8][4];
  float mrow[SLW][2], lrow[SLW][2];
#pragma unroll
  for (int sl = 0; sl < SLW; ++sl) {
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[sl][i][0] = o[sl][i][1] = o[sl][i][2] = o[sl][i][3] = 0.f;
    mrow[sl][0] = mrow[sl][1] = -INFINITY;
    lrow[sl][0] = lrow[sl][1] = 0.f;
  }

  // The stage loop, instantiated for the number NS of live 16-row slices of this tile (trailing
  // slices of padding rows only are skipped: their state never reaches an output row).  The live
  // slices share every K and V fragment load, and their independent mma/softmax chains interleave.
  // Per slice the arithmetic is identical for every NS and SL (a row's bits do not depend on the tile).
  auto stages = [&](auto ns_tag, bool compute) {
    constexpr int NS = decltype(ns_tag)::value;
    for (int st = 0; st < n_stage; ++st) {
      int buf;
      if (tma) {
        __syncthreads();       // every warp is done with the buffer the next load overwrites
        if (threadIdx.x == 0 && st + NST - 1 < n_stage) load_stage(st + NST - 1);
        buf = (g0 + st) % NST;
        mbar_wait(&full[buf], ((g0 + st) / NST) & 1);
      } else {
        cp_wait<NST - 2>();      // stage st landed (this thread's copies)
        __syncthreads();         // ... and everyone's; stage st-1's buffer is free again
        if (st + NST - 1 < n_stage) load_stage(st + NST - 1);
        cp_commit();
        buf = st % NST;
      }
      const int key0 = st * KS + kg * 16;
      if (!compute || key0 > max_pos) continue;   // warp-uniform
      const uint4* K = sK + (buf * KS) * CH;
      const uint4* V = sV + (buf * KS) * CH;
      float sc[NS][2][4];
#pragma unroll
      for (int sl = 0; sl < NS; ++sl)
#pragma unroll
        for (int j = 0; j < 2; ++j) sc[sl][j][0] = sc[sl][j][1] = sc[sl][j][2] = sc[sl][j][3] = 0.f;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t kb[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
          ldsm_x4(kb[j][0], kb[j][1], kb[j][2], kb[j][3], &K[kvoff(kg * 16 + j * 8 + (lane & 7), c * 4 + (lane >> 3))]);
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          uint32_t qa[2][4];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            ldsm_x4(qa[u][0], qa[u][1], qa[u][2], qa[u][3],
                    &sQ[swz<HD>((sl_base + sl) * 16 + (lane & 15), (2 * c + u) * 2 + (lane >> 4))]);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            mma16816(sc[sl][j], qa[0], kb[j][0], kb[j][1]);
            mma16816(sc[sl][j], qa[1], kb[j][2], kb[j][3]);
          }
        }
      }
      uint32_t pa[NS][4];
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        float bm0 = -INFINITY, bm1 = -INFINITY;
        if ((flags & 4) && key0 + 15 <= vis_all[sl]) {   // block visible to every row: the mask is the identity
#pragma unroll
          for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              sc[sl][j][e] = __fmul_rn(sc[sl][j][e], scale_log2);
              sc[sl][j][2 + e] = __fmul_rn(sc[sl][j][2 + e], scale_log2);
              bm0 = fmaxf(bm0, sc[sl][j][e]);
              bm1 = fmaxf(bm1, sc[sl][j][2 + e]);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int key = key0 + j * 8 + 2 * (lane & 3) + e;
              sc[sl][j][e] = key <= rpos[sl][0] ? __fmul_rn(sc[sl][j][e], scale_log2) : -INFINITY;
              sc[sl][j][2 + e] = key <= rpos[sl][1] ? __fmul_rn(sc[sl][j][2 + e], scale_log2) : -INFINITY;
              bm0 = fmaxf(bm0, sc[sl][j][e]);
              bm1 = fmaxf(bm1, sc[sl][j][2 + e]);
            }
          }
        }
        bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 1));
        bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
        bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 1));
        bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
        const float nm0 = fmaxf(mrow[sl][0], bm0), nm1 = fmaxf(mrow[sl][1], bm1);
        const float a0 = nm0 == -INFINITY ? 1.f : exp2f(__fsub_rn(mrow[sl][0], nm0));
        const float a1 = nm1 == -INFINITY ? 1.f : exp2f(__fsub_rn(mrow[sl][1], nm1));
        const float sub0 = nm0 == -INFINITY ? 0.f : nm0;
        const float sub1 = nm1 == -INFINITY ? 0.f : nm1;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          sc[sl][j][0] = exp2f(__fsub_rn(sc[sl][j][0], sub0));
          sc[sl][j][1] = exp2f(__fsub_rn(sc[sl][j][1], sub0));
          sc[sl][j][2] = exp2f(__fsub_rn(sc[sl][j][2], sub1));
          sc[sl][j][3] = exp2f(__fsub_rn(sc[sl][j][3], sub1));
          rs0 = __fadd_rn(rs0, __fadd_rn(sc[sl][j][0], sc[sl][j][1]));
          rs1 = __fadd_rn(rs1, __fadd_rn(sc[sl][j][2], sc[sl][j][3]));
        }
        rs0 = __fadd_rn(rs0, __shfl_xor_sync(0xffffffffu, rs0, 1));
        rs0 = __fadd_rn(rs0, __shfl_xor_sync(0xffffffffu, rs0, 2));
        rs1 = __fadd_rn(rs1, __shfl_xor_sync(0xffffffffu, rs1, 1));
        rs1 = __fadd_rn(rs1, __shfl_xor_sync(0xffffffffu, rs1, 2));
        lrow[sl][0] = __fmaf_rn(lrow[sl][0], a0, rs0);
        lrow[sl][1] = __fmaf_rn(lrow[sl][1], a1, rs1);
        mrow[sl][0] = nm0;
        mrow[sl][1] = nm1;
        pa[sl][0] = pack2(sc[sl][0][0], sc[sl][0][1]);
        pa[sl][1] = pack2(sc[sl][0][2], sc[sl][0][3]);
        pa[sl][2] = pack2(sc[sl][1][0], sc[sl][1][1]);
        pa[sl][3] = pack2(sc[sl][1][2], sc[sl][1][3]);
        // rescale only when some row's running max moved: skipping a multiply by exactly 1 is exact
        if (!(flags & 1) || __any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
          for (int n = 0; n < HD / 8; ++n) {
            o[sl][n][0] = __fmul_rn(o[sl][n][0], a0);
            o[sl][n][1] = __fmul_rn(o[sl][n][1], a0);
            o[sl][n][2] = __fmul_rn(o[sl][n][2], a1);
            o[sl][n][3] = __fmul_rn(o[sl][n][3], a1);
          }
        }
      }
#pragma unroll
      for (int n = 0; n < HD / 16; ++n) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(b0, b1, b2, b3, &V[kvoff(kg * 16 + (lane & 15), n * 2 + (lane >> 4))]);
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          mma16816(o[sl][2 * n], pa[sl], b0, b1);
          mma16816(o[sl][2 * n + 1], pa[sl], b2, b3);
        }
      }
    }
  };
  if constexpr (SLW == 1) {
    // NW = 8: a warp whose slice is padding only still walks the stages (barriers, TMA issue)
    stages(std::integral_constant<int, 1>{}, live[0] || !(flags & 2));
  } else {
    if ((flags & 2) && !live[1]) stages(std::integral_constant<int, 1>{}, true);
    else stages(std::integral_constant<int, SLW>{}, true);
  }
  cp_wait<0>();
  __syncthreads();
  g_stage = g0 + n_stage;

  // ---- merge the 4 warps' partial states in warp order (smem reuses the K/V ring)
  float* cO = reinterpret_cast<float*>(sm);                  // [4][ROWS][HD]
  float* cM = cO + 4 * ROWS * HD;                            // [4][ROWS]
  float* cL = cM + 4 * ROWS;                                 // [4][ROWS]
#pragma unroll
  for (int sl = 0; sl < SLW; ++sl) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = (sl_base + sl) * 16 + (lane >> 2) + 8 * h;
      float* dst = cO + ((size_t)kg * ROWS + r) * HD;
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        const int col = i * 8 + 2 * (lane & 3);
        dst[col] = o[sl][i][2 * h];
        dst[col + 1] = o[sl][i][2 * h + 1];
      }
      if ((lane & 3) == 0) {
        cM[kg * ROWS + r] = mrow[sl][h];
        cL[kg * ROWS + r] = lrow[sl][h];
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ROWS * (HD / 2); e += blockDim.x) {
    const int r = e / (HD / 2), d = (e % (HD / 2)) * 2;
    const int rr = tile * ROWS + r;
    if (rr >= rows_total) continue;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) mx = fmaxf(mx, cM[w * ROWS + r]);
    float num0 = 0.f, num1 = 0.f, den = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = cM[w * ROWS + r];
      const float sc = mw == -INFINITY ? 0.f : exp2f(__fsub_rn(mw, mx));
      den = __fmaf_rn(cL[w * ROWS + r], sc, den);
      num0 = __fmaf_rn(cO[((size_t)w * ROWS + r) * HD + d], sc, num0);
      num1 = __fmaf_rn(cO[((size_t)w * ROWS + r) * HD + d + 1], sc, num1);
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    __nv_bfloat16* dst = out + ((size_t)(qo + rr / G) * H + kvh * G + rr % G) * HD + d;
    *reinterpret_cast<uint32_t*>(dst) = pack2(num0 * inv, num1 * inv);
  }
  __syncthreads();   // the next item reuses the smem ring / merge buffers
  };

  if (work) {
    // persistent: items enumerated from the per-sequence tile prefix (work[s] = first tile of s)
    const int n_items = work[n_seq] * KVH;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int kvh = it % KVH, j = it / KVH;
      int lo = 0, hi = n_seq;   // last s with work[s] <= j
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (work[mid] <= j) lo = mid; else hi = mid;
      }
      do_tile(lo, kvh, j - work[lo]);
    }
  } else {
    // one CTA per (kv head, sequence) walking the sequence's tiles
    const int kvh = blockIdx.x, s = blockIdx.y;
    for (int tile = 0; tile * ROWS < q_len[s] * G; ++tile) do_tile(s, kvh, tile);
  }
}

// work[s] = sum over earlier sequences of ceil(q_len * G / rows); work[n_seq] = total (single block)
// work[s] = first tile of sequence s (exclusive prefix of ceil(q_len * G / rows)), work[n_seq] = total; with
// tile_seq (tcgen05 family) also tile_seq[t] = the sequence of tile t
__global__ void k_attn_tiles(const int32_t* __restrict__ q_len, int n_seq, int G, int rows, int32_t* __restrict__ work,
                             int32_t* __restrict__ tile_seq) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int base = 0; base < n_seq; base += blockDim.x) {
    const int s = base + threadIdx.x;
    const int t = s < n_seq ? (q_len[s] * G + rows - 1) / rows : 0;
    int incl = t;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int v = lane < nw ? warp_sums[lane] : 0;
      int iv = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, iv, o);
        if (lane >= o) iv += y;
      }
      if (lane < nw) warp_sums[lane] = iv - v;
    }
    __syncthreads();
    const int off = carry + warp_sums[wid] + incl - t;
    if (s < n_seq) work[s] = off;
    if (tile_seq)
      for (int i = 0; i < t; ++i) tile_seq[off + i] = s;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = off + t;
    __syncthreads();
  }
  if (threadIdx.x == 0) work[n_seq] = carry;
}

// tcgen05 attention (hm_attn_tc.cu): the default family (hm_set_attention_family; HM_ATTN_MMA selects
// mma.sync).  It needs a work list and the cache geometry for the TMA maps, else the mma.sync kernels
// run.  Both families are batch invariant, but a run must not mix them (speculative and greedy rows
// must share one kernel family)
constexpr int kTcRows = 128;
constexpr int kTcKeys = 128;   // keys per K/V stage: the TMA box height of the tcgen05 path
inline int tc_tile_rows(int) { return kTcRows; }
template <int HD>
int launch_attn_tc(const void* d_q, const int32_t* d_q_off, const int32_t* d_q_len, const int32_t* d_pos0,
                   const int32_t* d_kv_slot, int32_t n_seq, int32_t H, int32_t KVH, int32_t q_rows, int32_t max_len,
                   float scale_log2, void* d_out, const int32_t* d_work, const CUtensorMap& mq, const CUtensorMap& mk,
                   const CUtensorMap& mv, const CUtensorMap& mk64, const CUtensorMap& mv64, cudaStream_t st);
// attention family: -1 = not chosen yet (environment default), 0 = mma.sync, 1 = tcgen05 (hm_set_attention_family)
inline int& attn_family() {
  static int family = -1;
  return family;
}
inline bool attn_tc_enabled() {
  if (attn_family() < 0)   // default tcgen05; HM_ATTN_MMA / HM_ATTN_V2 select mma.sync (A/B)
    attn_family() = (getenv("HM_ATTN_MMA") != nullptr || getenv("HM_ATTN_V2") != nullptr) ? 0 : 1;
  return attn_family() == 1;
}

// exact work skips of k_attention2 (bit 0: rescale only when a row max moved, bit 1: skip slices
// of padding rows, bit 2: unmasked fast path for fully visible key blocks); HM_ATTN_FLAGS overrides
// the default (all on) for A/B profiling only
inline int attn_flags() {
  static const int f = getenv("HM_ATTN_FLAGS") ? atoi(getenv("HM_ATTN_FLAGS")) : 7;
  return f;
}

template <int HD, int SL>
int launch_attn2(const void* d_q, const void* d_kcache, const void* d_vcache, int64_t slot_stride,
                 const int32_t* d_q_off, const int32_t* d_q_len, const int32_t* d_pos0, const int32_t* d_kv_slot,
                 int32_t n_seq, int32_t max_q_len, int32_t H, int32_t KVH, int32_t max_len, float scale_log2,
                 void* d_out, int32_t* d_work, int32_t n_slots, int work_ready, int32_t q_rows, cudaStream_t st) {
  constexpr int ROWS = 16 * SL;
  const int ring = 2 * 3 * 64 * HD * 2;                  // K + V stages
  const int merge = 4 * ROWS * HD * 4 + 2 * 4 * ROWS * 4;
  const int smem = (ring > merge ? ring : merge) + ROWS * HD * 2 + 1024;
  // K/V caches as 2-D [slots * kv_heads * max_len, hd] bf16 tensors for TMA (rows past the end read as 0)
  CUtensorMap mk, mv;
  memset(&mk, 0, sizeof(mk));
  memset(&mv, 0, sizeof(mv));
  int use_tma = 0;
  if (n_slots > 0 && getenv("HM_ATTN_NO_TMA") == nullptr) {
    const int64_t rows = (int64_t)n_slots * KVH * max_len;
    use_tma = hm_make_tma_map(&mk, d_kcache, rows, HD, HD, 64) && hm_make_tma_map(&mv, d_vcache, rows, HD, HD, 64);
  }
  static int occupancy = 0;
  if (!occupancy) {
    cudaFuncSetAttribute(k_attention2<HD, SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occupancy, k_attention2<HD, SL>, 128, smem);
    if (occupancy < 1) occupancy = 1;
  }
  const int G = H / KVH;
  if (d_work) {
    // persistent CTAs over the (sequence, tile, kv head) work list: no empty CTAs, long verify blocks spread
    static int n_sm = 0;
    if (!n_sm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    if (!work_ready) {
      k_attn_tiles<<<1, 1024, 0, st>>>(d_q_len, n_seq, G, ROWS, d_work, nullptr);
      hm_count_launches(1);
    }
    if constexpr (SL == 2) {
      // verify tiles, opt-in (HM_ATTN_W8): the 8-warp variant (one slice per warp, two CTAs per SM), same
      // bits as NW = 4.  Measured on the real verify mix it is no faster: 46% more instructions (each
      // warp loads its own K/V fragments) cancel the doubled warps (profiles/r01_attention_variants.md)
      static const bool w8 = getenv("HM_ATTN_W8") != nullptr;
      if (w8) {
        static int occ8 = 0;
        if (!occ8) {
          cudaFuncSetAttribute(k_attention2<HD, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ8, k_attention2<HD, 2, 8>, 256, smem);
          if (occ8 < 1) occ8 = 1;
        }
        k_attention2<HD, 2, 8><<<hm_cap(n_sm, true) * occ8, 256, smem, st>>>(
            (const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_kcache, (const __nv_bfloat16*)d_vcache, slot_stride,
            d_q_off, d_q_len, d_pos0, d_kv_slot, H, KVH, q_rows, max_len, scale_log2, (__nv_bfloat16*)d_out, n_seq, d_work,
            mk, mv, use_tma, attn_flags());
        return 0;
      }
    }
    k_attention2<HD, SL><<<hm_cap(n_sm, true) * occupancy, 128, smem, st>>>(
        (const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_kcache, (const __nv_bfloat16*)d_vcache, slot_stride,
        d_q_off, d_q_len, d_pos0, d_kv_slot, H, KVH, q_rows, max_len, scale_log2, (__nv_bfloat16*)d_out, n_seq, d_work,
        mk, mv, use_tma, attn_flags());
  } else {
    dim3 grid(KVH, n_seq);
    k_attention2<HD, SL><<<grid, 128, smem, st>>>((const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_kcache,
                                                  (const __nv_bfloat16*)d_vcache, slot_stride, d_q_off, d_q_len,
                                                  d_pos0, d_kv_slot, H, KVH, q_rows, max_len, scale_log2,
                                                  (__nv_bfloat16*)d_out, n_seq, nullptr, mk, mv, use_tma, attn_flags());
  }
  return 0;
}

}  // namespace hm

// Attention kernel family for the forwards that follow (process-wide): 0 = mma.sync, 1 = tcgen05.  Both
// are batch invariant, but rows computed by different families differ in their last bits, so one
// rollout (and the greedy run it is compared with) must use one family.
extern "C" int hm_set_attention_family(int32_t family) {
  if (family != 0 && family != 1) { hm_set_error("attention family must be 0 (mma.sync) or 1 (tcgen05)"); return HM_ERR_INVALID; }
  hm::attn_family() = family;
  return HM_OK;
}
extern "C" int hm_attention_family(void) { return hm::attn_tc_enabled() ? 1 : 0; }

// Work list of the persistent attention kernel, computed once per forward (q_len is the same for
// every layer): work[s] = first tile of sequence s, work[n_seq] = total tiles.
extern "C" int64_t hm_attention_work_size(int32_t n_seq, int32_t max_q_len, int32_t H, int32_t KVH) {
  if (n_seq <= 0 || max_q_len <= 0 || KVH <= 0 || H % KVH) return 0;
  const int G = H / KVH;
  return (int64_t)n_seq + 1 + (int64_t)n_seq * (((int64_t)max_q_len * G + hm::kTcRows - 1) / hm::kTcRows);
}

extern "C" int hm_attention_plan(const int32_t* d_q_len, int32_t n_seq, int32_t max_q_len, int32_t H, int32_t KVH,
                                 int32_t* d_work, hm_stream_t stream) {
  if (n_seq <= 0) return HM_OK;
  if (H % KVH) { hm_set_error("H % KVH"); return HM_ERR_INVALID; }
  const int G = H / KVH;
  // must match the tile height chosen in hm_attention (which re-plans if it cannot take the tcgen05 path)
  const bool tc = hm::attn_tc_enabled();
  const int rows = tc ? hm::tc_tile_rows(G) : (max_q_len * G <= 16 ? 16 : 32);
  hm::k_attn_tiles<<<1, 1024, 0, (cudaStream_t)stream>>>(d_q_len, n_seq, G, rows, d_work,
                                                         tc ? d_work + n_seq + 1 : nullptr);
  hm_count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { hm_set_error(cudaGetErrorString(e)); return HM_ERR_CUDA; }
  return HM_OK;
}

extern "C" int hm_attention(const void* d_q, const void* d_kcache, const void* d_vcache, int64_t slot_stride,
                            const int32_t* d_q_off, const int32_t* d_q_len, const int32_t* d_pos0,
                            const int32_t* d_kv_slot, int32_t n_seq, int32_t max_q_len, int32_t H, int32_t KVH,
                            int32_t hd, int32_t max_len, float scale, void* d_out, int32_t* d_work,
                            int32_t work_ready, int32_t n_slots, int32_t q_rows, hm_stream_t stream) {
  if (n_seq <= 0 || max_q_len <= 0) return HM_OK;
  if (H % KVH) { hm_set_error("H % KVH"); return HM_ERR_INVALID; }
  if (q_rows <= 0) { hm_set_error("hm_attention: q_rows (row stride of d_q's kv-group planes) must be > 0"); return HM_ERR_INVALID; }
  const int G = H / KVH;
  dim3 grid((max_q_len * G + hm::AT_ROWS - 1) / hm::AT_ROWS, KVH, n_seq);
  const float scale_log2 = scale * 1.4426950408889634f;
  cudaStream_t st = (cudaStream_t)stream;
  if (hm::attn_tc_enabled()) {
    // tcgen05 path: needs the persistent work list and the cache and q geometry for the TMA maps; its packed
    // item words hold s in 20 bits, the tile in 8 and the kv head in 4
    if (n_seq >= (1 << 20) || KVH > 16 || ((int64_t)max_q_len * G + hm::kTcRows - 1) / hm::kTcRows > 256) {
      hm_set_error("hm_attention: n_seq, KVH or max_q_len beyond the tcgen05 kernel's limits");
      return HM_ERR_INVALID;
    }
    CUtensorMap mq, mk, mv, mk64, mv64;   // 16-row Q blocks; 128-key and trimmed 64-key K/V stages
    const int64_t rows = (int64_t)n_slots * KVH * max_len;
    if (d_work && n_slots > 0 && (hd == 128 || hd == 64) &&
        hm_make_tma_map(&mq, d_q, (int64_t)KVH * q_rows * G, hd, hd, 16) &&
        hm_make_tma_map(&mk, d_kcache, rows, hd, hd, hm::kTcKeys) &&
        hm_make_tma_map(&mv, d_vcache, rows, hd, hd, hm::kTcKeys) &&
        hm_make_tma_map(&mk64, d_kcache, rows, hd, hd, hm::kTcKeys / 2) &&
        hm_make_tma_map(&mv64, d_vcache, rows, hd, hd, hm::kTcKeys / 2)) {
      if (!work_ready) {
        hm::k_attn_tiles<<<1, 1024, 0, st>>>(d_q_len, n_seq, G, hm::tc_tile_rows(G), d_work, d_work + n_seq + 1);
        hm_count_launches(1);
      }
      if (hd == 128)
        hm::launch_attn_tc<128>(d_q, d_q_off, d_q_len, d_pos0, d_kv_slot, n_seq, H, KVH, q_rows, max_len, scale_log2, d_out,
                                d_work, mq, mk, mv, mk64, mv64, st);
      else
        hm::launch_attn_tc<64>(d_q, d_q_off, d_q_len, d_pos0, d_kv_slot, n_seq, H, KVH, q_rows, max_len, scale_log2, d_out,
                               d_work, mq, mk, mv, mk64, mv64, st);
      hm_count_launches(1);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { hm_set_error(cudaGetErrorString(e)); return HM_ERR_CUDA; }
      return HM_OK;
    }
    work_ready = 0;   // a plan made for the tensor-core tiles does not fit the fallback's tile height
  }
  const bool v1 = getenv("HM_ATTN_V1") != nullptr;   // A/B switch for profiling only
  if (!v1 && (hd == 128 || hd == 64)) {
    // rows per CTA tile: 16 when a whole (sequence, kv head) block fits, else 32
    const bool one = max_q_len * G <= 16;
    if (hd == 128) {
      if (one) hm::launch_attn2<128, 1>(d_q, d_kcache, d_vcache, slot_stride, d_q_off, d_q_len, d_pos0, d_kv_slot,
                                        n_seq, max_q_len, H, KVH, max_len, scale_log2, d_out, d_work, n_slots, work_ready, q_rows, st);
      else hm::launch_attn2<128, 2>(d_q, d_kcache, d_vcache, slot_stride, d_q_off, d_q_len, d_pos0, d_kv_slot,
                                    n_seq, max_q_len, H, KVH, max_len, scale_log2, d_out, d_work, n_slots, work_ready, q_rows, st);
    } else {
      if (one) hm::launch_attn2<64, 1>(d_q, d_kcache, d_vcache, slot_stride, d_q_off, d_q_len, d_pos0, d_kv_slot,
                                       n_seq, max_q_len, H, KVH, max_len, scale_log2, d_out, d_work, n_slots, work_ready, q_rows, st);
      else hm::launch_attn2<64, 2>(d_q, d_kcache, d_vcache, slot_stride, d_q_off, d_q_len, d_pos0, d_kv_slot,
                                   n_seq, max_q_len, H, KVH, max_len, scale_log2, d_out, d_work, n_slots, work_ready, q_rows, st);
    }
  } else if (hd == 128) {
    const int smem = (hm::AT_ROWS + 4 * hm::AT_KEYS) * 128 * 2;
    static bool set = false;
    if (!set) { cudaFuncSetAttribute(hm::k_attention<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); set = true; }
    hm::k_attention<128><<<grid, 128, smem, st>>>((const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_kcache,
                                                  (const __nv_bfloat16*)d_vcache, slot_stride, d_q_off, d_q_len,
                                                  d_pos0, d_kv_slot, H, KVH, q_rows, max_len, scale_log2,
                                                  (__nv_bfloat16*)d_out);
  } else if (hd == 64) {
    const int smem = (hm::AT_ROWS + 4 * hm::AT_KEYS) * 64 * 2;
    hm::k_attention<64><<<grid, 128, smem, st>>>((const __nv_bfloat16*)d_q, (const __nv_bfloat16*)d_kcache,
                                                 (const __nv_bfloat16*)d_vcache, slot_stride, d_q_off, d_q_len,
                                                 d_pos0, d_kv_slot, H, KVH, q_rows, max_len, scale_log2,
                                                 (__nv_bfloat16*)d_out);
  } else {
    hm_set_error("attention: head dim must be 64 or 128");
    return HM_ERR_INVALID;
  }
  hm_count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { hm_set_error(cudaGetErrorString(e)); return HM_ERR_CUDA; }
  return HM_OK;
}
