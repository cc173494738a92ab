// K4 on the 5th-gen tensor cores: causal GQA attention for variable-length
// query blocks (decode rows, verify blocks [last, d_1..d_k], prefill chunks)
// over the slot-contiguous KV cache, with both products on tcgen05 and the
// accumulators in TMEM.
//
// Work item = (sequence, kv head, 128-row tile) from the persistent work list
// (hm_attention_plan); its rows are the (query i, head j of the GQA group)
// pairs, so a verify block of up to 21 queries (GQA-6) is one item and its
// KV stream is read from HBM once.  One CTA per SM:
//   warp 0   TMA producer: K and V stages (64 keys) into separate 4-deep
//            rings, K running ahead of V (K is released by S, V by P.V)
//   warp 1   MMA issuer (one thread): S_j = Q K_j^T (M=128, N=64, K=hd) into
//            a 3-deep TMEM S ring, up to three stages ahead of the softmax;
//            O += P_j V_j (M=128, N=hd, K=64) with P read from its own
//            double-buffered TMEM columns and V as an MN-major operand
//   warps 2-5 softmax / correction / epilogue: thread = tile row = TMEM
//            lane; a whole row of 64 scores per thread (no shuffles), P
//            written to TMEM as packed bf16.  Warps whose 32 rows are all
//            padding only keep the barrier cadence.
// TMEM (512 columns): S ring [0, 192), P [192, 256), O [256, 256 + hd).
// Online softmax with a per-row lazy reference max: O and l are rescaled
// only when a block max exceeds the reference by more than 8 (log2 units,
// so P <= 256); the decision is per row, so every row's arithmetic depends
// on its own query, position and the cache only -- a row computed in a
// verify block is bit-identical to the same row decoded alone (greedy under
// speculation stays bit-exact with greedy decoding).
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdio>
#include <cstdlib>

#include "../../include/hsmodel.h"
#include "hm_ptx.cuh"

void hm_set_error(const char* msg);
void hm_count_launches(int64_t n);

namespace hm {

template <int HD>
struct TcAttn {
  static constexpr int ROWS = 128;                    // UMMA M: tile rows
  static constexpr int KS = 64;                       // keys per stage (UMMA N of S, K of P.V)
  static constexpr int NSK = 4, NSV = 4;              // K / V smem ring depths
  static constexpr int NS = 3, NP = 2;                // TMEM S ring / P buffers
  static constexpr int QB = ROWS * HD * 2;            // Q tile: [HD/64][ROWS][128 B], 128B-swizzled
  static constexpr int KVB = KS * HD * 2;             // one K or V stage: [HD/64][KS][128 B]
  // V slot: the stage's HD/64 column groups plus a constant group whose first column is 1.0, so
  // P.V with N = HD + 16 also accumulates the row sum l = sum_k P[k] in O column HD
  static constexpr int VSB = KVB + KS * 128;
  static constexpr int NO = HD + 16;                  // UMMA N of P.V
  static constexpr int SMEM = QB + NSK * KVB + NSV * VSB + 1024;   // QB: the next item's Q, staged
  static constexpr int TMEM_COLS = 512;
  // S ring [0, 192), P [192, 256), O and l [256, 256 + HD + 16) (+16 spare), Q (bf16 pairs) [448, 448 + HD/2)
  static constexpr uint32_t COL_S = 0, COL_P = 192, COL_O = 256, COL_Q = 448;
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

#ifdef HM_TC_WATCHDOG
// debugging aid: a wait that spins too long reports which barrier and traps instead of hanging
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, int id, int gs) {
  for (long long i = 0; i < (1ll << 28); ++i)
    if (mbar_test(bar, parity)) return;
  printf("attn_tc watchdog: block %d thread %d barrier %d parity %u stage %d\n", blockIdx.x, threadIdx.x, id, parity,
         gs);
  __trap();
}
#define MBAR_WAIT(bar, par, id, gs) mbar_wait_wd(bar, par, id, gs)
#else
#define MBAR_WAIT(bar, par, id, gs) mbar_wait(bar, par)
#endif

#ifdef HM_TC_TRACE
// debugging aid: clock64 per (event, stage) of CTA 0, read back with hm_debug_attn_trace
__device__ long long g_tc_trace[8 * 512];
#define TC_TRACE(ev, gs) \
  do { if (blockIdx.x == 0 && (gs) < 512) g_tc_trace[(ev) * 512 + (gs)] = clock64(); } while (0)
#else
#define TC_TRACE(ev, gs) do { } while (0)
#endif

template <int HD>
__global__ void __launch_bounds__(320, 1) k_attn_tc(const __nv_bfloat16* __restrict__ q,
                                                    const int32_t* __restrict__ q_off,
                                                    const int32_t* __restrict__ q_len,
                                                    const int32_t* __restrict__ pos0,
                                                    const int32_t* __restrict__ kv_slot, int H, int KVH,
                                                    int max_len, float scale_log2, __nv_bfloat16* __restrict__ out,
                                                    int n_seq, const int32_t* __restrict__ work,
                                                    const __grid_constant__ CUtensorMap tmK,
                                                    const __grid_constant__ CUtensorMap tmV) {
  using C = TcAttn<HD>;
  constexpr int ROWS = C::ROWS, KS = C::KS, NSK = C::NSK, NSV = C::NSV, NS = C::NS, NP = C::NP;
  const int G = H / KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sm + C::QB;              // [NSK][KVB] (after the Q staging buffer)
  uint8_t* sV = sK + NSK * C::KVB;       // [NSV][VSB]
  // the constant "ones" group of every V slot: key row k, element 0 = 1.0 (128B-swizzled like TMA writes)
  for (int i = threadIdx.x; i < NSV * KS * 8; i += blockDim.x) {
    const int slot = i / (KS * 8), k = (i / 8) % KS, chunk = i % 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if ((chunk ^ (k & 7)) == 0) v.x = 0x3F80u;   // bf16 1.0 in the low half: element 0 of the row
    *reinterpret_cast<uint4*>(sV + slot * C::VSB + C::KVB + k * 128 + chunk * 16) = v;
  }
  fence_proxy_async_smem();
  __shared__ uint64_t k_full[NSK], k_empty[NSK], v_full[NSV], v_empty[NSV];
  __shared__ uint64_t s_full[NS], s_free[NS], p_full[NP], p_free[NP], o_ready, q_full[2], o_free, m_ready[2];
  __shared__ float m_sh[ROWS];   // per-row lazy reference max after the latest stage (handed between the sets)
  __shared__ uint32_t tmem_base;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSK; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    for (int i = 0; i < NP; ++i) {
      mbar_init(&p_full[i], 4);
      mbar_init(&p_free[i], 1);
    }
    mbar_init(&o_ready, 1);
    mbar_init(&q_full[0], 4);
    mbar_init(&q_full[1], 4);
    mbar_init(&o_free, 4);
    mbar_init(&m_ready[0], 4);
    mbar_init(&m_ready[1], 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int n_items = work[n_seq] * KVH;
  auto locate = [&](int it, int& s, int& kvh, int& tile) {
    kvh = it % KVH;
    const int j = it / KVH;
    int lo = 0, hi = n_seq;   // last s with work[s] <= j
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (work[mid] <= j) lo = mid; else hi = mid;
    }
    s = lo;
    tile = j - work[lo];
  };
  // stages of an item: keys [0, max position of its last live row]
  auto item_stages = [&](int s, int tile) {
    const int last_row = min(q_len[s] * G, (tile + 1) * ROWS) - 1;
    return (pos0[s] + last_row / G) / KS + 1;
  };

  if (warp == 0) {
    // ---------------- TMA producer: two cursors (K ahead of V), never blocking on one ring for the other
    if (lane == 0) {
      struct Cur {
        int it, st, nst, row0;
        uint32_t g;
      };
      Cur ck{(int)blockIdx.x - (int)gridDim.x, 0, 0, 0, 0u}, cv = ck;
      auto advance = [&](Cur& c) {   // move to a stage to load; false when the CTA's items are exhausted
        while (c.st >= c.nst) {
          c.it += gridDim.x;
          if (c.it >= n_items) return false;
          int s, kvh, tile;
          locate(c.it, s, kvh, tile);
          c.nst = item_stages(s, tile);
          c.row0 = (kv_slot[s] * KVH + kvh) * max_len;
          c.st = 0;
        }
        return true;
      };
      bool kmore = advance(ck), vmore = advance(cv);
      while (kmore || vmore) {
        const uint32_t issued = ck.g + cv.g;
        if (kmore) {
          const int slot = ck.g % NSK;
          if (ck.g < (uint32_t)NSK || mbar_test(&k_empty[slot], ((ck.g / NSK) - 1) & 1)) {
            mbar_arrive_expect_tx(&k_full[slot], C::KVB);
#pragma unroll
            for (int hb = 0; hb < HD / 64; ++hb)
              tma_load_2d(&tmK, &k_full[slot], sK + slot * C::KVB + hb * KS * 128, hb * 64, ck.row0 + ck.st * KS);
            ++ck.st;
            ++ck.g;
            kmore = advance(ck);
          }
        }
        if (vmore) {
          const int slot = cv.g % NSV;
          if (cv.g < (uint32_t)NSV || mbar_test(&v_empty[slot], ((cv.g / NSV) - 1) & 1)) {
            mbar_arrive_expect_tx(&v_full[slot], C::KVB);
#pragma unroll
            for (int hb = 0; hb < HD / 64; ++hb)
              tma_load_2d(&tmV, &v_full[slot], sV + slot * C::VSB + hb * KS * 128, hb * 64, cv.row0 + cv.st * KS);
            ++cv.st;
            ++cv.g;
            vmore = advance(cv);
          }
        }
        if (ck.g + cv.g == issued) __nanosleep(64);   // both rings full: back off (shares an SMSP with a softmax warp)
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t id_s = idesc_bf16(ROWS, KS);                     // Q, K both K-major
      const uint32_t id_pv = idesc_bf16(ROWS, C::NO) | (1u << 16);    // [V | ones]: MN-major B operand
      uint32_t g = 0, items = 0;
      uint64_t kdesc[NSK], vdesc[NSV];   // base smem descriptors of the K and V ring slots
#pragma unroll
      for (int i = 0; i < NSK; ++i) kdesc[i] = smem_desc_sw128(sK + i * C::KVB);
#pragma unroll
      for (int i = 0; i < NSV; ++i) vdesc[i] = smem_desc_sw128_mn(sV + i * C::VSB, KS * 128);
      auto issue_s = [&](uint32_t gs) {
        const int slot = gs % NSK, b = gs % NS;
        MBAR_WAIT(&k_full[slot], (gs / NSK) & 1, 1, gs);
        TC_TRACE(4, gs);
        if (gs >= (uint32_t)NS) MBAR_WAIT(&s_free[b], ((gs / NS) - 1) & 1, 2, gs);   // softmax has read S_{gs-NS}
        tc_fence_after();
        // A = Q from TMEM (16 elements = 8 packed columns per K step): only K is read from smem.  The K
        // descriptors differ from the slot's base descriptor by constant start-address offsets (16-byte
        // units), so each issue is one add -- rebuilding a descriptor per MMA costs more than the MMA.
        const uint64_t kd0 = kdesc[slot];
        const uint32_t d_s = tbase + C::COL_S + b * KS, a_q = tbase + C::COL_Q;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_f16_ts(d_s, a_q + kk * 8, kd0 + (uint64_t)(((kk >> 2) * KS * 128 + (kk & 3) * 32) >> 4), id_s,
                      kk > 0 ? 1u : 0u);
        umma_commit(&k_empty[slot]);
        umma_commit(&s_full[b]);
        TC_TRACE(0, gs);
      };
      auto stages_of = [&](int it) {
        int s, kvh, tile;
        locate(it, s, kvh, tile);
        return item_stages(s, tile);
      };
      int n_stage = (int)blockIdx.x < n_items ? stages_of(blockIdx.x) : 0;
      for (int it = blockIdx.x; it < n_items; ++items) {
        const int it_next = it + gridDim.x;
        MBAR_WAIT(&q_full[0], items & 1, 3, (int)g);   // this item's Q is in TMEM
        tc_fence_after();
        for (int i = 0; i < NS && i < n_stage; ++i) issue_s(g + i);
        const int n_next = it_next < n_items ? stages_of(it_next) : 0;   // its loads overlap the S MMAs
        if (items > 0) {   // the previous item's epilogue has read O
          MBAR_WAIT(&o_free, (items - 1) & 1, 4, (int)g);
          tc_fence_after();
        }
        for (int st = 0; st < n_stage; ++st) {
          const uint32_t gs = g + st;
          const int vslot = gs % NSV, pb = gs & 1;
          MBAR_WAIT(&p_full[pb], (gs >> 1) & 1, 5, gs);
          TC_TRACE(1, gs);
          MBAR_WAIT(&v_full[vslot], (gs / NSV) & 1, 6, gs);
          TC_TRACE(5, gs);
          tc_fence_after();
          const uint64_t vd0 = vdesc[vslot];
          const uint32_t a_p = tbase + C::COL_P + pb * 32, d_o = tbase + C::COL_O;
#pragma unroll
          for (int kk = 0; kk < KS / 16; ++kk)   // 16 keys = 2 K groups of 8 rows x 128 B per step
            umma_f16_ts(d_o, a_p + kk * 8, vd0 + (uint64_t)(kk * 2048 >> 4), id_pv, (st > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&v_empty[vslot]);
          umma_commit(&p_free[pb]);
          if (st == n_stage - 1) umma_commit(&o_ready);   // the item's O is complete
          if (st + NS < n_stage) issue_s(gs + NS);
        }
        g += n_stage;
        it = it_next;
        n_stage = n_next;
      }
    }
  } else {
    // ---------------- softmax / correction / epilogue: thread = tile row = TMEM lane
    // TMEM lane (= UMMA row = Q smem row) tl; tile row (tl + 64) mod 128, so the first 64 tile rows --
    // all of a decode or short verify block -- sit on warps 2 and 3, whose SM sub-partitions do not
    // also host the producer and MMA warps
    const int quarter = warp & 3;
    const int set = (warp - 2) >> 2;   // softmax set: stages with (global stage & 1) == set
    const int tl = quarter * 32 + lane;
    const int row = (tl + 64) & (ROWS - 1);
    const uint32_t t_lane = tbase + ((uint32_t)(quarter * 32) << 16);
    struct Item {
      int s, kvh, tile, rows_total, rows_here, qo, p0, n_stage;
    };
    auto item_info = [&](int it) {
      Item x;
      locate(it, x.s, x.kvh, x.tile);
      x.rows_total = q_len[x.s] * G;
      x.rows_here = min(x.rows_total - x.tile * ROWS, ROWS);
      x.qo = q_off[x.s];
      x.p0 = pos0[x.s];
      x.n_stage = item_stages(x.s, x.tile);
      return x;
    };
    // Q: this thread's row of an item is staged in smem early (global latency off the critical path),
    // then moved into the TMEM Q columns -- one packed bf16 pair per column -- once the previous
    // item's products are done, and handed to the MMA warp on q_full (zeros for padding rows)
    auto stage_q = [&](const Item& x) {
      const bool lv = row < x.rows_here;
      const int r2 = x.tile * ROWS + row;
      const uint4* src = reinterpret_cast<const uint4*>(
          q + ((size_t)(x.qo + (lv ? r2 / G : 0)) * H + x.kvh * G + (lv ? r2 % G : 0)) * HD);
#pragma unroll
      for (int ch = 0; ch < HD / 8; ++ch) {
        const uint4 v = lv ? src[ch] : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(sQ + (ch >> 3) * ROWS * 128 + tl * 128 + (((ch & 7) ^ (tl & 7)) << 4)) = v;
      }
    };
    auto commit_q = [&]() {
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        uint32_t w[32];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint4 v = *reinterpret_cast<const uint4*>(sQ + c * ROWS * 128 + tl * 128 + ((k ^ (tl & 7)) << 4));
          w[4 * k + 0] = v.x;
          w[4 * k + 1] = v.y;
          w[4 * k + 2] = v.z;
          w[4 * k + 3] = v.w;
        }
        tmem_st32(t_lane + C::COL_Q + c * 32, w);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_full[0]);
    };
    uint32_t g = 0, items = 0;
    Item cur;
    if ((int)blockIdx.x < n_items) {
      cur = item_info(blockIdx.x);
      if (set == 0) {
        stage_q(cur);
        commit_q();
      }
    }
    for (int it = blockIdx.x; it < n_items; ++items) {
      const int it_next = it + gridDim.x;
      Item nxt;
      if (it_next < n_items) {
        nxt = item_info(it_next);
        if (set == 0) stage_q(nxt);   // this thread re-reads only its own staged row: no barrier needed
      }
      const int kvh = cur.kvh, tile = cur.tile, rows_here = cur.rows_here;
      const int qo = cur.qo, p0 = cur.p0, n_stage = cur.n_stage;
      const bool live = row < rows_here;
      const bool warp_live = ((tl - lane + 64) & (ROWS - 1)) < rows_here;   // warp-uniform
      const int rr = tile * ROWS + row;
      const int rpos = live ? p0 + rr / G : -1;          // -1: padding row, fully masked
      // the two softmax sets take alternate stages; the per-row lazy reference max (log2 units) passes
      // from one to the other through m_sh, ordered by m_ready (l accumulates in O column HD)
      for (int st = 0; st < n_stage; ++st) {
        const uint32_t gs = g + st;
        if ((int)(gs & 1) != set) continue;
        const int b = gs % NS, pb = gs & 1;
        MBAR_WAIT(&s_full[b], (gs / NS) & 1, 7, gs);
        if (warp_live && lane == 0) TC_TRACE(2, gs);
        tc_fence_after();
        float sc[64];
        if (warp_live) {
          tmem_ld32(t_lane + C::COL_S + b * KS, sc);
          tmem_ld32(t_lane + C::COL_S + b * KS + 32, sc + 32);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[b]);   // S_gs is in registers: the MMA may refill the buffer
        if (warp_live) {
          const int key0 = st * KS;
          float mx[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) mx[i] = -INFINITY;
          // raw scores; the log2-domain scale is folded into the exponent's fma (scale > 0, so the
          // block max of the scaled scores is the scaled max, exactly)
          if (__all_sync(0xffffffffu, !live || key0 + KS - 1 <= rpos)) {   // no live row needs a mask
#pragma unroll
            for (int i = 0; i < 64; ++i) mx[i & 7] = fmaxf(mx[i & 7], sc[i]);
          } else {
            const int nv = rpos - key0;   // keys key0 + i, i <= nv, are visible to this row
#pragma unroll
            for (int i = 0; i < 64; ++i) {
              sc[i] = i <= nv ? sc[i] : -INFINITY;
              mx[i & 7] = fmaxf(mx[i & 7], sc[i]);
            }
          }
          const float bmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                   fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * scale_log2;
          // the reference after stage gs-1 (the other set's); -inf at the item's first stage
          if (gs >= 1) MBAR_WAIT(&m_ready[(gs - 1) & 1], ((gs - 1) >> 1) & 1, 12, gs);
          const float m_ref = st > 0 ? m_sh[tl] : -INFINITY;
          float m_new = m_ref;
          bool resc = false;
          if (bmax > -INFINITY) {
            if (m_ref == -INFINITY) {
              m_new = bmax;   // first visible block: O and l are still 0
            } else if (bmax > m_ref + 8.f) {
              m_new = bmax;
              resc = true;
            }
          }
          m_sh[tl] = m_new;
          __syncwarp();
          if (lane == 0) mbar_arrive(&m_ready[gs & 1]);
          if (__any_sync(0xffffffffu, resc)) {
            // O holds P.V through stage gs-1 once P_{gs-1}.V_{gs-1} is done; scale this warp's rows
            // (factor 1 for the others: an exact no-op)
            MBAR_WAIT(&p_free[(gs - 1) & 1], ((gs - 1) >> 1) & 1, 8, gs);
            tc_fence_after();
            const float f = resc ? ex2f(m_ref - m_new) : 1.f;
#pragma unroll
            for (int c = 0; c <= HD / 32; ++c) {   // O columns [0, HD) and l (column HD; 16 spare columns ride along)
              float o[32];
              tmem_ld32(t_lane + C::COL_O + c * 32, o);
              uint32_t u[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(o[i] * f);
              tmem_st32(t_lane + C::COL_O + c * 32, u);
            }
            tmem_wait_st();
          }
          const float sub = m_new == -INFINITY ? 0.f : m_new;
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i)
            pk[i] = pack2(ex2f(fmaf(sc[2 * i], scale_log2, -sub)), ex2f(fmaf(sc[2 * i + 1], scale_log2, -sub)));
          // P buffer pb was last read by P_{gs-2}.V_{gs-2}
          if (gs >= 2) MBAR_WAIT(&p_free[pb], ((gs >> 1) - 1) & 1, 9, gs);
          tc_fence_after();
          tmem_st32(t_lane + C::COL_P + pb * 32, pk);
          tmem_wait_st();
        } else {
          // padding-only warps keep the cadence: an early arrival on m_ready or p_full for stage gs could
          // land in the phase of stage gs-2 while a slower warp has not yet arrived for it
          if (gs >= 1) MBAR_WAIT(&m_ready[(gs - 1) & 1], ((gs - 1) >> 1) & 1, 12, gs);
          __syncwarp();
          if (lane == 0) mbar_arrive(&m_ready[gs & 1]);
          if (gs >= 2) MBAR_WAIT(&p_free[pb], ((gs >> 1) - 1) & 1, 11, gs);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
        if (warp_live && lane == 0) TC_TRACE(3, gs);
      }
      // epilogue (set 0): O / l for the live rows
      if (set == 0) {
      MBAR_WAIT(&o_ready, items & 1, 10, (int)g);
      tc_fence_after();
      // every product of this item is done: the next item's Q can replace this one in TMEM, and the MMA
      // warp starts its S products while this epilogue reads O
      if (it_next < n_items) commit_q();
      if (warp_live) {
        float lv[32];
        tmem_ld32(t_lane + C::COL_O + HD, lv);   // l = sum of the bf16 P the tensor core accumulated
        const float inv = lv[0] > 0.f ? 1.f / lv[0] : 0.f;
        __nv_bfloat16* dst = out + ((size_t)(qo + (live ? rr / G : 0)) * H + kvh * G + (live ? rr % G : 0)) * HD;
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          float o[32];
          tmem_ld32(t_lane + C::COL_O + c * 32, o);
          if (live) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 w;
              w.x = pack2(o[8 * v + 0] * inv, o[8 * v + 1] * inv);
              w.y = pack2(o[8 * v + 2] * inv, o[8 * v + 3] * inv);
              w.z = pack2(o[8 * v + 4] * inv, o[8 * v + 5] * inv);
              w.w = pack2(o[8 * v + 6] * inv, o[8 * v + 7] * inv);
              *reinterpret_cast<uint4*>(dst + c * 32 + 8 * v) = w;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free);
      }
      g += n_stage;
      it = it_next;
      cur = nxt;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tbase);
  }
}

template <int HD>
int launch_attn_tc(const void* d_q, const int32_t* d_q_off, const int32_t* d_q_len, const int32_t* d_pos0,
                   const int32_t* d_kv_slot, int32_t n_seq, int32_t H, int32_t KVH, int32_t max_len, float scale_log2,
                   void* d_out, const int32_t* d_work, const CUtensorMap& mk, const CUtensorMap& mv,
                   cudaStream_t st) {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_attn_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcAttn<HD>::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, dev);   // one CTA per SM (512 TMEM columns)
    if (getenv("HM_TC_GRID")) grid = atoi(getenv("HM_TC_GRID"));          // debugging only
  }
  k_attn_tc<HD><<<grid, 320, TcAttn<HD>::SMEM, st>>>((const __nv_bfloat16*)d_q, d_q_off, d_q_len, d_pos0, d_kv_slot,
                                                      H, KVH, max_len, scale_log2, (__nv_bfloat16*)d_out, n_seq,
                                                      d_work, mk, mv);
  return 0;
}

#ifdef HM_TC_TRACE
extern "C" int hm_debug_attn_trace(long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_tc_trace, sizeof(g_tc_trace));
}
#endif

template int launch_attn_tc<64>(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, int32_t,
                                int32_t, int32_t, int32_t, float, void*, const int32_t*, const CUtensorMap&,
                                const CUtensorMap&, cudaStream_t);
template int launch_attn_tc<128>(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, int32_t,
                                 int32_t, int32_t, int32_t, float, void*, const int32_t*, const CUtensorMap&,
                                 const CUtensorMap&, cudaStream_t);

}  // namespace hm
