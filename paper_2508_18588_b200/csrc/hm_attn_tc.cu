// K4 on the 5th-gen tensor cores: causal GQA attention for variable-length
// query blocks (decode rows, verify blocks [last, d_1..d_k], prefill chunks)
// over the slot-contiguous KV cache, with both products on tcgen05 and the
// accumulators in TMEM.
//
// Work item = (sequence, kv head, 128-row tile) from the persistent work list
// (hm_attention_plan); its rows are the (query i, head j of the GQA group)
// pairs, so a verify block of up to 21 queries (GQA-6) is one item and its
// KV stream is read from HBM once.  One CTA per SM, 10 warps:
//   warp 0   TMA producer: K and V stages of 128 keys into separate 3-deep
//            rings, K running ahead of V (K is released by S, V by P.V)
//   warp 1   MMA issuer (one thread): S_j = Q K_j^T (M=128, N=128, K=hd, Q
//            read from TMEM) into a 2-deep TMEM S ring; O += P_j V_j (M=128,
//            N=hd, K=128) with P written by the softmax over the first half of
//            S_j's columns and V as an MN-major operand.  Measured on B200
//            (tools/dbg/umma_bench*.cu): an M=128 UMMA costs 45/64/128 cycles
//            at N=64/128/256, so 128-key stages halve the issue cost per key.
//   warps 2-9 softmax: two sets of four warps take alternate stages; in a
//            set, warp w owns TMEM lane quarter w % 4 and reads it as two
//            16-lane halves with tcgen05.ld.16x256b, so thread t holds rows
//            t/4 and t/4 + 8 of the half and 32 of the stage's keys -- a
//            decode block's few live rows get 4 threads each.  The packed P
//            pairs are exactly the tcgen05.st.16x128b fragment.
// Online softmax with a per-row lazy reference max: O and l are rescaled
// only when a block max exceeds the reference by more than 8 (log2 units,
// so P <= 256); the reference passes between the sets through shared
// memory.  Every decision is per row, so a row's arithmetic depends only on
// its own query, position and the cache -- a row computed in a verify block
// is bit-identical to the same row decoded alone (greedy under speculation
// stays bit-exact with greedy decoding).

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
  static constexpr int KS = 128;                      // keys per stage (UMMA N of S, K of P.V)
  static constexpr int NSK = 2, NSV = 3;              // K / V smem ring depths
  static constexpr int NS = 3;                        // TMEM S ring (P aliases the first KS/2 columns)
  static constexpr int QB = ROWS * HD * 2;            // Q tile: [HD/64][ROWS][128 B], 128B-swizzled
  static constexpr int KVB = KS * HD * 2;             // one K or V stage: [HD/64][KS][128 B]
  static constexpr int SMEM = 2 * QB + (NSK + NSV) * KVB + 1024;   // Q double-buffered across items
  static constexpr int TMEM_COLS = 512;
  // S ring [0, 384) (P = packed bf16 pairs over the first KS/2 columns of its S buffer), O [384, 384 + HD)
  static constexpr uint32_t COL_S = 0, COL_O = 384;
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
// 16x256b.x16: 16 lanes x 128 columns (r[4i + 0/1] = (a, 8i + 2q + 0/1), r[4i + 2/3] = (b, ...))
__device__ __forceinline__ void tmem_ld_16x256b_x16(uint32_t taddr, uint32_t* r) {
  tmem_ld_16x256b_x8(taddr, r);
  tmem_ld_16x256b_x8(taddr + 64, r + 32);
}
// 16x128b.x16: 16 lanes x 64 columns (r[2i] = (a, 4i + q), r[2i + 1] = (b, 4i + q))
__device__ __forceinline__ void tmem_st_16x128b_x16(uint32_t taddr, const uint32_t* r) {
  tmem_st_16x128b_x8(taddr, r);
  tmem_st_16x128b_x8(taddr + 32, r + 16);
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
                                                    const __grid_constant__ CUtensorMap tmV,
                                                    const __grid_constant__ CUtensorMap tmK64,
                                                    const __grid_constant__ CUtensorMap tmV64) {
  using C = TcAttn<HD>;
  constexpr int ROWS = C::ROWS, KS = C::KS, NSK = C::NSK, NSV = C::NSV, NS = C::NS;
  const int G = H / KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                      // [2][QB]: Q tiles by item parity
  uint8_t* sK = sm + 2 * C::QB;          // [NSK][KVB]
  uint8_t* sV = sK + NSK * C::KVB;       // [NSV][KVB]
  __shared__ uint64_t k_full[NSK], k_empty[NSK], v_full[NSV], v_empty[NSV];
  __shared__ uint64_t s_full[NS], p_full[NS], p_done[NS], o_ready, q_full[2], o_free, m_ready[2], l_ready[2];
  __shared__ float m_sh[ROWS];       // per-row lazy reference max after the latest stage (handed between the sets)
  __shared__ float l_sh[2 * ROWS];   // per-row sum of P, gathered for the epilogue (by item parity)
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
      mbar_init(&p_full[i], 4);
      mbar_init(&p_done[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&m_ready[i], 4);
      mbar_init(&l_ready[i], 4);
      mbar_init(&q_full[i], 4);
    }
    mbar_init(&o_ready, 1);
    mbar_init(&o_free, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&tmem_base);
  // A trimmed last stage loads only its first 64 keys; the rest of the slot keeps earlier contents, which
  // are masked (K) or multiplied by P = 0 (V) -- zero the rings once so they are finite from the start.
  for (int i = threadIdx.x; i < (NSK + NSV) * C::KVB / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sK)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
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
        bool half_last;   // the item's last stage needs at most its first 64 keys
        uint32_t g;
      };
      Cur ck{(int)blockIdx.x - (int)gridDim.x, 0, 0, 0, false, 0u}, cv = ck;
      auto advance = [&](Cur& c) {   // move to a stage to load; false when the CTA's items are exhausted
        while (c.st >= c.nst) {
          c.it += gridDim.x;
          if (c.it >= n_items) return false;
          int s, kvh, tile;
          locate(c.it, s, kvh, tile);
          c.nst = item_stages(s, tile);
          const int last_row = min(q_len[s] * G, (tile + 1) * ROWS) - 1;
          c.half_last = (pos0[s] + last_row / G) % KS < KS / 2;
          c.row0 = (kv_slot[s] * KVH + kvh) * max_len;
          c.st = 0;
        }
        return true;
      };
      // one K or V stage; the item's last stage is trimmed to a 64-key box when that covers it (decode rows
      // would otherwise over-read ~64 keys per item, ~3% of the KV stream)
      auto load = [&](const Cur& c, const CUtensorMap* full_map, const CUtensorMap* half_map, uint64_t* bar,
                      uint8_t* dst) {
        const bool half = c.half_last && c.st == c.nst - 1;
        mbar_arrive_expect_tx(bar, half ? C::KVB / 2 : C::KVB);
#pragma unroll
        for (int hb = 0; hb < HD / 64; ++hb)
          tma_load_2d(half ? half_map : full_map, bar, dst + hb * KS * 128, hb * 64, c.row0 + c.st * KS);
      };
      bool kmore = advance(ck), vmore = advance(cv);
      while (kmore || vmore) {
        const uint32_t issued = ck.g + cv.g;
        if (kmore) {
          const int slot = ck.g % NSK;
          if (ck.g < (uint32_t)NSK || mbar_test(&k_empty[slot], ((ck.g / NSK) - 1) & 1)) {
            load(ck, &tmK, &tmK64, &k_full[slot], sK + slot * C::KVB);
            ++ck.st;
            ++ck.g;
            kmore = advance(ck);
          }
        }
        if (vmore) {
          const int slot = cv.g % NSV;
          if (cv.g < (uint32_t)NSV || mbar_test(&v_empty[slot], ((cv.g / NSV) - 1) & 1)) {
            load(cv, &tmV, &tmV64, &v_full[slot], sV + slot * C::KVB);
            ++cv.st;
            ++cv.g;
            vmore = advance(cv);
          }
        }
        if (ck.g + cv.g == issued) __nanosleep(64);   // both rings full: back off (shares an SMSP with softmax warps)
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t id_s = idesc_bf16(ROWS, KS);                     // A = Q, B = K (both K-major smem)
      const uint32_t id_pv = idesc_bf16(ROWS, HD) | (1u << 16);       // A = P (TMEM), B = V (MN-major smem)
      uint64_t kdesc[NSK], vdesc[NSV], qdesc[2];   // base descriptors (per-step offsets are constants)
#pragma unroll
      for (int i = 0; i < NSK; ++i) kdesc[i] = smem_desc_sw128(sK + i * C::KVB);
#pragma unroll
      for (int i = 0; i < NSV; ++i) vdesc[i] = smem_desc_sw128_mn(sV + i * C::KVB, KS * 128);
      qdesc[0] = smem_desc_sw128(sQ);
      qdesc[1] = smem_desc_sw128(sQ + C::QB);
      uint32_t g = 0, items = 0;
      auto issue_s = [&](uint32_t gs) {
        const int slot = gs % NSK, b = gs % NS;
        MBAR_WAIT(&k_full[slot], (gs / NSK) & 1, 1, gs);
        TC_TRACE(4, gs);
        // S buffer b last held S_{gs-NS} and P_{gs-NS}: wait until P_{gs-NS}.V_{gs-NS} has read it
        if (gs >= (uint32_t)NS) MBAR_WAIT(&p_done[b], ((gs / NS) - 1) & 1, 2, gs);
        tc_fence_after();
        const uint64_t kd0 = kdesc[slot], qd0 = qdesc[items & 1];
        const uint32_t d_s = tbase + C::COL_S + b * KS;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off_q = ((kk >> 2) * ROWS * 128 + (kk & 3) * 32) >> 4;
          const uint32_t off_k = ((kk >> 2) * KS * 128 + (kk & 3) * 32) >> 4;
          umma_f16(d_s, qd0 + off_q, kd0 + off_k, id_s, kk > 0 ? 1u : 0u);
        }
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
        MBAR_WAIT(&q_full[items & 1], (items >> 1) & 1, 3, (int)g);   // this item's Q tile is in smem
        tc_fence_after();
        // S runs NS - 1 stages ahead of P.V: the buffer S_{j+2} overwrites held P_{j-1}, whose P.V was
        // queued a stage earlier, so the issuing thread rarely waits (S_{j+3} would wait for P_j.V_j)
        for (int i = 0; i < NS - 1 && i < n_stage; ++i) issue_s(g + i);
        const int n_next = it_next < n_items ? stages_of(it_next) : 0;   // its loads overlap the S MMAs
        if (items > 0) {   // the previous item's epilogue has read O
          MBAR_WAIT(&o_free, (items - 1) & 1, 4, (int)g);
          tc_fence_after();
        }
        for (int st = 0; st < n_stage; ++st) {
          const uint32_t gs = g + st;
          const int vslot = gs % NSV, b = gs % NS;
          MBAR_WAIT(&p_full[b], (gs / NS) & 1, 5, gs);
          TC_TRACE(1, gs);
          MBAR_WAIT(&v_full[vslot], (gs / NSV) & 1, 6, gs);
          TC_TRACE(5, gs);
          tc_fence_after();
          const uint64_t vd0 = vdesc[vslot];
          const uint32_t a_p = tbase + C::COL_S + b * KS, d_o = tbase + C::COL_O;
#pragma unroll
          for (int kk = 0; kk < KS / 16; ++kk)   // 16 keys = 2 K groups of 8 rows x 128 B per step
            umma_f16_ts(d_o, a_p + kk * 8, vd0 + (uint64_t)(kk * 2048 >> 4), id_pv, (st > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&v_empty[vslot]);
          umma_commit(&p_done[b]);
          if (st == n_stage - 1) umma_commit(&o_ready);   // the item's O is complete
          if (st + NS - 1 < n_stage) issue_s(gs + NS - 1);
        }
        g += n_stage;
        it = it_next;
        n_stage = n_next;
      }
    }
  } else {
    // ---------------- softmax / correction / epilogue
    // TMEM lane (= UMMA row = Q row) tl of tile row r: 16-row block rb = r / 16 goes to lane quarter
    // (2 + rb) % 4, half rb / 4.  The first halves of all four quarters fill first, so a tile of up to 64
    // rows (a verify block of <= 10 queries at GQA-6) spreads over four softmax warps per set, one 16-lane
    // half each; decode rows sit on quarter 2, whose SM sub-partition does not also host the producer and
    // MMA warps.  Softmax fragment: half h of the quarter, thread t: lanes a = 16h + t/4 and b = a + 8 (of
    // the quarter), keys 8i + 2q + {0,1}, q = t % 4.
    const int quarter = warp & 3;
    const int set = (warp - 2) >> 2;   // this set takes the stages with (global stage & 1) == set
    const int tl = quarter * 32 + lane;
    auto row_of_lane = [&](int ln) {   // inverse of the lane map above
      const int rb = (((ln >> 5) + 2) & 3) + ((ln >> 4) & 1) * 4;
      return rb * 16 + (ln & 15);
    };
    const int row = row_of_lane(tl);
    const uint32_t t_lane = tbase + ((uint32_t)(quarter * 32) << 16);
    const int q4 = lane & 3;
    auto trow_of = [&](int h, int ab) { return row_of_lane(quarter * 32 + 16 * h + (lane >> 2) + 8 * ab); };
    auto lane_of = [&](int h, int ab) { return quarter * 32 + 16 * h + (lane >> 2) + 8 * ab; };
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
    // Q: set 0 writes this thread's row of an item into the item's smem Q tile (128B-swizzled, K-major:
    // the S products' A operand) and hands it over on q_full[buffer]; zeros for padding rows
    auto write_q = [&](const Item& x, int qbuf) {
      const bool lv = row < x.rows_here;
      const int r2 = x.tile * ROWS + row;
      const uint4* src = reinterpret_cast<const uint4*>(
          q + ((size_t)(x.qo + (lv ? r2 / G : 0)) * H + x.kvh * G + (lv ? r2 % G : 0)) * HD);
      uint8_t* dq = sQ + qbuf * C::QB;
#pragma unroll
      for (int ch = 0; ch < HD / 8; ++ch) {
        const uint4 v = lv ? src[ch] : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(dq + (ch >> 3) * ROWS * 128 + tl * 128 + (((ch & 7) ^ (tl & 7)) << 4)) = v;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_full[qbuf]);
    };
    uint32_t g = 0, items = 0;
    Item cur;
    if ((int)blockIdx.x < n_items) {
      cur = item_info(blockIdx.x);
      if (set == 0) write_q(cur, 0);
    }
    for (int it = blockIdx.x; it < n_items; ++items) {
      // the next item's Q goes into the other buffer now, so the MMA warp can start its S products while
      // this item's epilogue runs (that buffer was last read by the previous item's S products, all done)
      const int it_next = it + gridDim.x;
      Item nxt;
      if (it_next < n_items) {
        nxt = item_info(it_next);
        if (set == 0) write_q(nxt, (items + 1) & 1);
      }
      const int rows_here = cur.rows_here, n_stage = cur.n_stage;
      int hpos[2][2];   // position of row (half, a/b); -1: padding row, fully masked
      bool hlive[2];    // the half holds a live row (warp-uniform)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        hlive[h] = row_of_lane(quarter * 32 + 16 * h) < rows_here;   // first row of the half's 16-row block
#pragma unroll
        for (int ab = 0; ab < 2; ++ab) {
          const int tr = trow_of(h, ab);
          hpos[h][ab] = tr < rows_here ? cur.p0 + (cur.tile * ROWS + tr) / G : -1;
        }
      }
      float lsum[2][2] = {{0.f, 0.f}, {0.f, 0.f}};   // this thread's part of each row's sum of P
      for (int st = 0; st < n_stage; ++st) {
        const uint32_t gs = g + st;
        if ((int)(gs & 1) != set) continue;
        const int b = gs % NS;
        const uint32_t t_s = t_lane + C::COL_S + b * KS;
        MBAR_WAIT(&s_full[b], (gs / NS) & 1, 7, gs);
        tc_fence_after();
        if (quarter == 2 && lane == 0) TC_TRACE(2, gs);
        const int key0 = st * KS;
        // the reference after stage gs-1 (the other set's); -inf at the item's first stage
        if (gs >= 1) MBAR_WAIT(&m_ready[(gs - 1) & 1], ((gs - 1) >> 1) & 1, 12, gs);
        float fac[2][2] = {{1.f, 1.f}, {1.f, 1.f}};
        bool resc_any = false;
        uint32_t pk[2][32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!hlive[h]) continue;
          uint32_t sv[64];
          tmem_ld_16x256b_x16(t_s + ((uint32_t)(16 * h) << 16), sv);
          tmem_wait_ld();
          float* sc = reinterpret_cast<float*>(sv);   // sc[4i + 2ab + e]: row ab, key key0 + 8i + 2q + e
          if (!__all_sync(0xffffffffu, key0 + KS - 1 <= hpos[h][0] && key0 + KS - 1 <= hpos[h][1])) {
#pragma unroll
            for (int ab = 0; ab < 2; ++ab) {
              const int nv = hpos[h][ab] - key0;   // keys key0 + k, k <= nv, are visible to the row
#pragma unroll
              for (int i = 0; i < KS / 8; ++i)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                  if (8 * i + 2 * q4 + e > nv) sc[4 * i + 2 * ab + e] = -INFINITY;
            }
          }
#pragma unroll
          for (int ab = 0; ab < 2; ++ab) {
            // raw-score row max over the 4 threads of the row; the log2-domain scale is folded into the
            // exponent's fma (scale > 0: the max of the scaled scores is the scaled max, exactly)
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int i = 0; i < KS / 8; ++i) {
              mx0 = fmaxf(mx0, sc[4 * i + 2 * ab]);
              mx1 = fmaxf(mx1, sc[4 * i + 2 * ab + 1]);
            }
            float mx = fmaxf(mx0, mx1);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float bmax = mx * scale_log2;
            const int ln = lane_of(h, ab);
            const float m_ref = st > 0 ? m_sh[ln] : -INFINITY;
            float m_new = m_ref;
            if (bmax > -INFINITY) {
              if (m_ref == -INFINITY) {
                m_new = bmax;   // first visible block: O and l are still 0
              } else if (bmax > m_ref + 8.f) {
                m_new = bmax;
                fac[h][ab] = ex2f(m_ref - m_new);
                resc_any = true;
              }
            }
            if (q4 == 0) m_sh[ln] = m_new;
            const float sub = m_new == -INFINITY ? 0.f : m_new;
            float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
            for (int i = 0; i < KS / 8; ++i) {
              const float p0 = ex2f(fmaf(sc[4 * i + 2 * ab], scale_log2, -sub));
              const float p1 = ex2f(fmaf(sc[4 * i + 2 * ab + 1], scale_log2, -sub));
              ls0 += p0;
              ls1 += p1;
              pk[h][2 * i + ab] = pack2(p0, p1);
            }
            lsum[h][ab] = fmaf(lsum[h][ab], fac[h][ab], ls0 + ls1);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&m_ready[gs & 1]);
        if (__any_sync(0xffffffffu, resc_any)) {
          // O holds P.V through stage gs-1 once P_{gs-1}.V_{gs-1} is done: scale the rows whose
          // reference moved (factor 1 for the others: an exact no-op)
          MBAR_WAIT(&p_done[(gs - 1) % NS], ((gs - 1) / NS) & 1, 8, gs);
          tc_fence_after();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (!hlive[h]) continue;
            const uint32_t t_o = t_lane + ((uint32_t)(16 * h) << 16) + C::COL_O;
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
              uint32_t o[32];
              tmem_ld_16x256b_x8(t_o + c * 64, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * fac[h][(i >> 1) & 1]);
              tmem_st_16x256b_x8(t_o + c * 64, o);
            }
          }
          tmem_wait_st();
        }
        // P over the first KS/2 columns of S_gs (this set has read them; the MMA warp reads P next)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (hlive[h]) tmem_st_16x128b_x16(t_s + ((uint32_t)(16 * h) << 16), pk[h]);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        if (quarter == 2 && lane == 0) TC_TRACE(3, gs);
      }
      // gather each row's sum of P (the 4 threads of a row, both sets) into l_sh
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int ab = 0; ab < 2; ++ab) {
          float v = lsum[h][ab];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          lsum[h][ab] = v;
        }
      float* lbuf = l_sh + (items & 1) * ROWS;   // per item parity: set 1 may run an item ahead of set 0
      if (set == 1) {
        // hand this set's sums of P over to set 0's epilogue
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ab = 0; ab < 2; ++ab)
            if (q4 == 0) lbuf[lane_of(h, ab)] = lsum[h][ab];
        __syncwarp();
        if (lane == 0) mbar_arrive(&l_ready[items & 1]);
      } else {
        // epilogue (set 0), once every product of the item is done: O / l for the live rows
        MBAR_WAIT(&o_ready, items & 1, 10, (int)g);
        tc_fence_after();
        MBAR_WAIT(&l_ready[items & 1], (items >> 1) & 1, 13, (int)g);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ab = 0; ab < 2; ++ab)
            if (q4 == 0) lbuf[lane_of(h, ab)] += lsum[h][ab];
        __syncwarp();
        const bool live = row < rows_here;
        if (hlive[0] || hlive[1]) {   // the warp holds a live row
          const float lrow = lbuf[tl];
          const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
          const int rr = cur.tile * ROWS + row;
          __nv_bfloat16* dst =
              out + ((size_t)(cur.qo + (live ? rr / G : 0)) * H + cur.kvh * G + (live ? rr % G : 0)) * HD;
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
                   const CUtensorMap& mk64, const CUtensorMap& mv64, cudaStream_t st) {
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
                                                      d_work, mk, mv, mk64, mv64);
  return 0;
}

#ifdef HM_TC_TRACE
extern "C" int hm_debug_attn_trace(long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_tc_trace, sizeof(g_tc_trace));
}
#endif

template int launch_attn_tc<64>(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, int32_t,
                                int32_t, int32_t, int32_t, float, void*, const int32_t*, const CUtensorMap&,
                                const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, cudaStream_t);
template int launch_attn_tc<128>(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, int32_t,
                                 int32_t, int32_t, int32_t, float, void*, const int32_t*, const CUtensorMap&,
                                 const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, cudaStream_t);

}  // namespace hm
