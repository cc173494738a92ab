// K4 on the 5th-gen tensor cores: causal GQA attention for variable-length
// query blocks (decode rows, verify blocks [last, d_1..d_k], prefill chunks)
// over the slot-contiguous KV cache, with both products on tcgen05 and the
// accumulators in TMEM.
//
// Work item = (sequence, kv head, 128-row tile) from the persistent work list
// (hm_attention_plan); its rows are the (query i, head j of the GQA group)
// pairs, so a verify block of up to 21 queries (GQA-6) is one item and its KV
// stream is read from HBM once.  One CTA per SM,
// 10 warps:
//   warp 0   TMA producer: the item's Q boxes (one per 16-row block, into a
//            double-buffered tile), K and V stages of 128 keys into separate
//            2- and 3-deep rings, K running ahead of V (K is released by S,
//            V by P.V, Q by the item's last S)
//   warp 1   MMA issuer (one thread): S_j = Q K_j^T (M=128, N=128, K=hd)
//            into a 3-deep TMEM S ring, two stages ahead of O += P_j V_j
//            (M=128, N=hd, K=128) with P written by the softmax over the
//            first half of S_j's columns and V as an MN-major operand.
//            Measured on B200 (tools/dbg/umma_bench*.cu): an M=128 UMMA costs
//            45/64/128 cycles at N=64/128/256, so 128-key stages halve the
//            issue cost per key.
//   warps 2-9 softmax: two sets of four warps take alternate stages; in a
//            set, warp w owns TMEM lane quarter w % 4 and reads it as two
//            16-lane halves with tcgen05.ld.16x256b, so thread t holds rows
//            t/4 and t/4 + 8 of the half and 32 of the stage's keys -- a
//            decode block's few live rows get 4 threads each.  The packed P
//            pairs are exactly the tcgen05.st.16x128b fragment.
// The per-CTA item list is located once per 32 items (one item per lane,
// read back by shuffles), so no warp waits on a global load at an item
// boundary.
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
int hm_cap(int n_sms, bool attn);

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
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {   // zero-fills if !valid
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
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
// debugging aid: a wait that spins too long reports which barrier (and what every warp of the CTA waits on)
// and traps instead of hanging
__shared__ int g_wd_state[10][3];
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, int id, int gs) {
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    g_wd_state[w][0] = id;
    g_wd_state[w][1] = gs;
    g_wd_state[w][2] = (int)parity;
  }
  for (long long i = 0; i < (1ll << 28); ++i)
    if (mbar_test(bar, parity)) {
      if ((threadIdx.x & 31) == 0) g_wd_state[w][0] = -id;
      return;
    }
  if ((threadIdx.x & 31) == 0) {
    printf("attn_tc watchdog: block %d warp %d barrier %d parity %u stage %d | %d:%d/%d/%d %d:%d/%d/%d %d:%d/%d/%d %d:%d/%d/%d %d:%d/%d/%d %d:%d/%d/%d %d:%d/%d/%d %d:%d/%d/%d\n",
           blockIdx.x, w, id, parity, gs, 0, g_wd_state[0][0], g_wd_state[0][1], g_wd_state[0][2], 1,
           g_wd_state[1][0], g_wd_state[1][1], g_wd_state[1][2], 2, g_wd_state[2][0], g_wd_state[2][1],
           g_wd_state[2][2], 3, g_wd_state[3][0], g_wd_state[3][1], g_wd_state[3][2], 6, g_wd_state[6][0],
           g_wd_state[6][1], g_wd_state[6][2], 7, g_wd_state[7][0], g_wd_state[7][1], g_wd_state[7][2], 4,
           g_wd_state[4][0], g_wd_state[4][1], g_wd_state[4][2], 5, g_wd_state[5][0], g_wd_state[5][1],
           g_wd_state[5][2]);
  }
  __trap();
}
#define MBAR_WAIT(bar, par, id, gs) mbar_wait_wd(bar, par, id, gs)
#define WD_NOTE(id, gs) do { if ((threadIdx.x & 31) == 0) { g_wd_state[threadIdx.x >> 5][0] = (id); g_wd_state[threadIdx.x >> 5][1] = (gs); } } while (0)
#else
#define MBAR_WAIT(bar, par, id, gs) mbar_wait(bar, par)
#define WD_NOTE(id, gs) do { } while (0)
#endif

#ifndef HM_TC_BACKOFF_NS
#define HM_TC_BACKOFF_NS 64   // producer back-off when every ring is full
#endif

#ifdef HM_TC_TRACE
// debugging aid: clock64 per (event, stage) of CTA 0, read back with hm_debug_attn_trace
__device__ long long g_tc_trace[16 * 512];
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
                                                    int q_rows, int max_len, float scale_log2, __nv_bfloat16* __restrict__ out,
                                                    int n_seq, const int32_t* __restrict__ work,
                                                    const __grid_constant__ CUtensorMap tmQ,
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
  __shared__ uint64_t s_full[NS], p_full[NS], p_done[NS], o_ready[2], q_full[2], q_empty[2], o_free, m_ready[2],
      l_ready[2];
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
#ifdef HM_TC_QCPASYNC
      mbar_init(&q_full[i], 4);
#else
      mbar_init(&q_full[i], 1);
#endif
      mbar_init(&q_empty[i], 1);
      mbar_init(&o_ready[i], 1);
    }
    mbar_init(&o_free, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&tmem_base);
  // A trimmed last stage loads only its first 64 keys; the rest of the slot keeps earlier contents, which
  // are masked (K) or multiplied by P = 0 (V); Q lanes that no query box covers keep theirs, masked rows --
  // zero the Q tiles and the rings once so they are finite from the start.
  for (int i = threadIdx.x; i < (2 * C::QB + (NSK + NSV) * C::KVB) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sQ)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int n_items = work[n_seq] * KVH;
  const int n_mine = n_items > (int)blockIdx.x ? (n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int32_t* tile_seq = work + n_seq + 1;   // hm_attention_plan: sequence of each tile
  // Q tile layout: tile row r (query r / G, head r % G of the item's kv group; rows past the item's are
  // padding) sits in TMEM lane / smem row 32 * ((2 + rb) % 4) + 16 * (rb / 4) + r % 16, rb = r / 16.  The
  // first halves of all four lane quarters fill first, so a verify block of up to 64 rows (10 queries at
  // GQA-6) keeps four softmax warps per set busy with one 16-lane half each, and a decode row sits on
  // quarter 2, whose SM sub-partition does not also host the producer and MMA warps.  d_q is kv-group-major
  // ([KVH][q_rows][G][hd]), so each 16-row block is one 2-D TMA box.
  auto block_lane = [](int rb) { return ((2 + rb) & 3) * 32 + (rb >> 2) * 16; };
  auto locate = [&](int it, int& s, int& kvh, int& tile) {
    kvh = it % KVH;
    const int j = it / KVH;
    s = tile_seq[j];
    tile = j - work[s];
  };
  // rows of an item's tile
  auto tile_rows = [&](int qlen, int tile) { return min(qlen * G - tile * ROWS, ROWS); };
  // This CTA's items k = 0, 1, ... (work item blockIdx.x + k * gridDim.x) are located 32 at a time, one per
  // lane, and read back with a shuffle, so no warp waits on a global load at an item boundary (under a
  // saturated HBM one round trip costs thousands of cycles).  Item word: s << 12 | tile << 4 | kvh
  // (hm_attention checks the field widths).
  struct Tab {
    int base;             // CTA-local index of the item held by lane 0
    uint32_t word, nst;   // this lane's item: word, stage count
    int row0, half;       // (producer) first cache row of its K/V head; last stage fits a 64-key box
    int qrow, nrows;      // (producer) first Q row of the tile in d_q's 2-D view; rows in the tile
  };
  auto fill = [&](Tab& t, int base) {
    t.base = base;
    t.word = 0u;
    t.nst = 0u;
    t.row0 = 0;
    t.half = 0;
    t.qrow = 0;
    t.nrows = 0;
    if (base + lane < n_mine) {
      int s, kvh, tile;
      locate((int)blockIdx.x + (base + lane) * (int)gridDim.x, s, kvh, tile);
      const int nr = tile_rows(q_len[s], tile);
      const int lastpos = pos0[s] + (tile * ROWS + nr - 1) / G;   // the key range ends at its last row
      t.word = (uint32_t)s << 12 | (uint32_t)tile << 4 | (uint32_t)kvh;
      t.nst = (uint32_t)(lastpos / KS + 1);
      t.row0 = (kv_slot[s] * KVH + kvh) * max_len;
      t.half = lastpos % KS < KS / 2;
      t.qrow = (kvh * q_rows + q_off[s]) * G + tile * ROWS;
      t.nrows = nr;
    }
  };
  // warp-uniform k, k >= t.base (items are visited in order); refills when k leaves the window
  auto lookup = [&](Tab& t, int k, int& s, int& kvh, int& tile, int& nst) {
    if (k >= t.base + 32) fill(t, k);
    const uint32_t w = __shfl_sync(0xffffffffu, t.word, k - t.base);
    nst = (int)__shfl_sync(0xffffffffu, t.nst, k - t.base);
    s = (int)(w >> 12);
    tile = (int)((w >> 4) & 255u);
    kvh = (int)(w & 15u);
  };

  if (warp == 0) {
    // ---------------- TMA producer (the whole warp walks the items; lane 0 issues): two cursors (K ahead of
    // V), never blocking on one ring for the other
    struct Cur {
      int k, st, nst, row0;
      bool half_last;   // the item's last stage needs at most its first 64 keys
      uint32_t g;
      Tab tab;
    };
    Cur ck;
    ck.k = -1;
    ck.st = ck.nst = ck.row0 = 0;
    ck.half_last = false;
    ck.g = 0u;
    fill(ck.tab, 0);
    Cur cv = ck;
    auto advance = [&](Cur& c) {   // move to a stage to load; false when the CTA's items are exhausted
      while (c.st >= c.nst) {
        if (++c.k >= n_mine) return false;
        int s, kvh, tile;
        lookup(c.tab, c.k, s, kvh, tile, c.nst);
        c.half_last = __shfl_sync(0xffffffffu, c.tab.half, c.k - c.tab.base) != 0;
        c.row0 = __shfl_sync(0xffffffffu, c.tab.row0, c.k - c.tab.base);
        if (&c == &ck && lane == 0) TC_TRACE(14, c.k);
        c.st = 0;
      }
      return true;
    };
    // one K or V stage; the item's last stage is trimmed to a 64-key box when that covers it (decode rows
    // would otherwise over-read ~64 keys per item, ~3% of the KV stream)
    auto load = [&](const Cur& c, const CUtensorMap* full_map, const CUtensorMap* half_map, uint64_t* bar,
                    uint8_t* dst) {
      if (lane != 0) return;
      const bool half = c.half_last && c.st == c.nst - 1;
      mbar_arrive_expect_tx(bar, half ? C::KVB / 2 : C::KVB);
#pragma unroll
      for (int hb = 0; hb < HD / 64; ++hb)
#ifndef HM_TC_KV_L2_NORMAL   // the K/V stream is read once: evict-first in L2, so it does not push out the
                              // tile's Q, the outputs and the next kernels' operands (-4% verify, -2% decode)
        tma_load_2d_evict_first(half ? half_map : full_map, bar, dst + hb * KS * 128, hb * 64, c.row0 + c.st * KS);
#else
        tma_load_2d(half ? half_map : full_map, bar, dst + hb * KS * 128, hb * 64, c.row0 + c.st * KS);
#endif
    };
    // slot free? (lane 0 polls, the warp follows)
    auto ready = [&](uint64_t* bar, uint32_t parity) {
      return __shfl_sync(0xffffffffu, lane == 0 ? (int)mbar_test(bar, parity) : 0, 0) != 0;
    };
    // Q tiles: item kq's tile goes into buffer kq & 1 once item kq - 2's S products are done; one 16-row
    // box per block (rows past the tile's read the next rows of d_q or zeros past its end: masked padding)
#ifdef HM_TC_QCPASYNC   // A/B variant: set 0 copies Q with cp.async (softmax section)
    int kq = n_mine;
#else
    int kq = 0;
#endif
    Tab tq;
    fill(tq, 0);
    auto load_q = [&]() {
      int s, kvh, tile, nst;
      lookup(tq, kq, s, kvh, tile, nst);
      const int qrow = __shfl_sync(0xffffffffu, tq.qrow, kq - tq.base);
      const int nblk = (__shfl_sync(0xffffffffu, tq.nrows, kq - tq.base) + 15) / 16;
      if (lane == 0) {
        uint64_t* bar = &q_full[kq & 1];
        mbar_arrive_expect_tx(bar, nblk * 16 * 128 * (HD / 64));
        uint8_t* dq = sQ + (kq & 1) * C::QB;
        for (int rb = 0; rb < nblk; ++rb)
#pragma unroll
          for (int hb = 0; hb < HD / 64; ++hb)
            tma_load_2d(&tmQ, bar, dq + hb * ROWS * 128 + block_lane(rb) * 128, hb * 64, qrow + rb * 16);
      }
      ++kq;
    };
    bool kmore = advance(ck), vmore = advance(cv);
    while (kmore || vmore || kq < n_mine) {
      const uint32_t issued = ck.g + cv.g + kq;
      WD_NOTE(100 + kq, (int)(ck.g * 1000 + cv.g));
      if (kq < n_mine && (kq < 2 || ready(&q_empty[kq & 1], ((kq - 2) >> 1) & 1))) load_q();
      if (kmore) {
        const int slot = ck.g % NSK;
        if (ck.g < (uint32_t)NSK || ready(&k_empty[slot], ((ck.g / NSK) - 1) & 1)) {
          load(ck, &tmK, &tmK64, &k_full[slot], sK + slot * C::KVB);
          ++ck.st;
          ++ck.g;
          kmore = advance(ck);
        }
      }
      if (vmore) {
        const int slot = cv.g % NSV;
        if (cv.g < (uint32_t)NSV || ready(&v_empty[slot], ((cv.g / NSV) - 1) & 1)) {
          load(cv, &tmV, &tmV64, &v_full[slot], sV + slot * C::KVB);
          ++cv.st;
          ++cv.g;
          vmore = advance(cv);
        }
      }
      if (ck.g + cv.g + kq == issued) __nanosleep(HM_TC_BACKOFF_NS);   // rings full: back off (shares an SMSP with softmax warps)
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (the whole warp walks the items; lane 0 issues)
    const bool leader = lane == 0;
    const uint32_t id_s = idesc_bf16(ROWS, KS);                     // A = Q, B = K (both K-major smem)
    const uint32_t id_pv = idesc_bf16(ROWS, HD) | (1u << 16);       // A = P (TMEM), B = V (MN-major smem)
    uint64_t kdesc[NSK], vdesc[NSV], qdesc[2];   // base descriptors (per-step offsets are constants)
#pragma unroll
    for (int i = 0; i < NSK; ++i) kdesc[i] = smem_desc_sw128(sK + i * C::KVB);
#pragma unroll
    for (int i = 0; i < NSV; ++i) vdesc[i] = smem_desc_sw128_mn(sV + i * C::KVB, KS * 128);
    qdesc[0] = smem_desc_sw128(sQ);
    qdesc[1] = smem_desc_sw128(sQ + C::QB);
    // S products run NS - 1 = 2 stages ahead of P.V as one stream across items (an item's first S products
    // are queued while the previous item's last P.V run): S_{j+2} overwrites the buffer of P_{j-1}, whose P.V
    // was queued a stage earlier, so the issuing thread rarely waits (S_{j+3} would wait for P_j.V_j)
    Tab tab_s, tab_p;
    fill(tab_s, 0);
    tab_p = tab_s;
    int s_, kvh_, tile_;
    int ks = 0, ss = 0, ns_s = 0;   // S cursor: item, stage in item, item's stage count
    uint32_t gS = 0;                // global index of the next S
    if (n_mine > 0) lookup(tab_s, 0, s_, kvh_, tile_, ns_s);
    auto issue_next_s = [&]() {
      if (ks >= n_mine) return;
      const uint32_t gs = gS;
      if (ss == 0) {   // the item's Q tile is in smem
        MBAR_WAIT(&q_full[ks & 1], (ks >> 1) & 1, 3, (int)gs);
        if (lane == 0) TC_TRACE(15, ks);
      }
      const int slot = gs % NSK, b = gs % NS;
      MBAR_WAIT(&k_full[slot], (gs / NSK) & 1, 1, gs);
      TC_TRACE(4, gs);
      // S buffer b last held S_{gs-NS} and P_{gs-NS}: wait until P_{gs-NS}.V_{gs-NS} has read it
      if (gs >= (uint32_t)NS) MBAR_WAIT(&p_done[b], ((gs / NS) - 1) & 1, 2, gs);
      tc_fence_after();
      if (leader) {
        const uint64_t kd0 = kdesc[slot], qd0 = qdesc[ks & 1];
        const uint32_t d_s = tbase + C::COL_S + b * KS;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off_q = ((kk >> 2) * ROWS * 128 + (kk & 3) * 32) >> 4;
          const uint32_t off_k = ((kk >> 2) * KS * 128 + (kk & 3) * 32) >> 4;
          umma_f16(d_s, qd0 + off_q, kd0 + off_k, id_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&k_empty[slot]);
        umma_commit(&s_full[b]);
        if (ss == ns_s - 1) umma_commit(&q_empty[ks & 1]);   // the item's last S: its Q tile may be refilled
      }
      __syncwarp();
      TC_TRACE(0, gs);
      ++gS;
      if (++ss >= ns_s) {
        ss = 0;
        if (++ks < n_mine) lookup(tab_s, ks, s_, kvh_, tile_, ns_s);
      }
    };
    for (int i = 0; i < NS - 1; ++i) issue_next_s();
    uint32_t g = 0;
    for (int k = 0; k < n_mine; ++k) {
      int n_stage;
      lookup(tab_p, k, s_, kvh_, tile_, n_stage);
      if (k > 0) {   // the previous item's epilogue has read O
        MBAR_WAIT(&o_free, (k - 1) & 1, 4, (int)g);
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
        if (leader) {
          const uint64_t vd0 = vdesc[vslot];
          const uint32_t a_p = tbase + C::COL_S + b * KS, d_o = tbase + C::COL_O;
#pragma unroll
          for (int kk = 0; kk < KS / 16; ++kk)   // 16 keys = 2 K groups of 8 rows x 128 B per step
            umma_f16_ts(d_o, a_p + kk * 8, vd0 + (uint64_t)(kk * 2048 >> 4), id_pv, (st > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&v_empty[vslot]);
          umma_commit(&p_done[b]);
          if (st == n_stage - 1) umma_commit(&o_ready[k & 1]);   // the item's O is complete
        }
        __syncwarp();
        issue_next_s();   // S_{gs+2}, possibly of the next item
      }
      g += n_stage;
    }
  } else {
    // ---------------- softmax / correction / epilogue
    // Softmax fragment (TMEM lane = UMMA row = Q tile row, laid out as above): half h of the quarter,
    // thread t: lanes a = 16h + t/4 and b = a + 8 (of the quarter), keys 8i + 2q + {0,1}, q = t % 4.
    const int quarter = warp & 3;
    const int set = (warp - 2) >> 2;   // this set takes the stages with (global stage & 1) == set
    const int tl = quarter * 32 + lane;
    const uint32_t t_lane = tbase + ((uint32_t)(quarter * 32) << 16);
    const int q4 = lane & 3;
    const int rb_of_half[2] = {(quarter + 2) & 3, ((quarter + 2) & 3) + 4};   // 16-row block of half h
    auto row_of = [&](int h, int o) { return rb_of_half[h] * 16 + o; };   // tile row of half h, lane offset o
    auto lane_of = [&](int h, int ab) { return quarter * 32 + 16 * h + (lane >> 2) + 8 * ab; };
    struct Item {   // raw fields (loaded an item ahead of use)
      int kvh, tile, qlen, qo, p0, n_stage;
    };
    Tab tab;
    fill(tab, 0);
    auto item_info = [&](int k) {   // CTA-local item k
      Item x;
      int sq;
      lookup(tab, k, sq, x.kvh, x.tile, x.n_stage);
      x.qlen = q_len[sq];
      x.qo = q_off[sq];
      x.p0 = pos0[sq];
      return x;
    };
    uint32_t g = 0, items = 0;
    Item cur, nxt;
    if (n_mine > 0) cur = item_info(0);
    if (n_mine > 1) nxt = item_info(1);
#ifdef HM_TC_QCPASYNC
    // set 0 copies this thread's Q row (tile row of TMEM lane tl) of an item into its tile with cp.async;
    // q_ready hands the tile over once the copies have landed
    auto load_q = [&](const Item& x, int qbuf) {
      const int r = row_of(lane >> 4, lane & 15);
      const bool lv = r < tile_rows(x.qlen, x.tile);
      const __nv_bfloat16* src = q + ((size_t)(x.kvh * q_rows + x.qo) * G + x.tile * ROWS + (lv ? r : 0)) * HD;
      uint8_t* dq = sQ + qbuf * C::QB;
#pragma unroll
      for (int ch = 0; ch < HD / 8; ++ch)
        cp_async16(dq + (ch >> 3) * ROWS * 128 + tl * 128 + (((ch & 7) ^ (tl & 7)) << 4), src + ch * 8, lv);
      cp_commit();
    };
    auto q_ready = [&](int qbuf) {
      cp_wait_all();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_full[qbuf]);
    };
    if (set == 0 && n_mine > 0) {
      load_q(cur, 0);
      q_ready(0);
    }
#endif
    for (int k = 0; k < n_mine; ++k, ++items) {
      Item nn;   // the item after next: its fields load while this item runs
      if (k + 2 < n_mine) nn = item_info(k + 2);
#ifdef HM_TC_QCPASYNC
      bool q_pending = false;
      if (set == 0 && k + 1 < n_mine) {   // item k + 1's tile: buffer free once item k - 1's S are done
        if (k >= 1) MBAR_WAIT(&q_empty[(k + 1) & 1], ((k - 1) >> 1) & 1, 15, k);
        load_q(nxt, (k + 1) & 1);
        q_pending = true;
      }
#endif
      if (quarter == 2 && lane == 0) TC_TRACE(set == 0 ? 8 : 12, items);
      const int rows_here = tile_rows(cur.qlen, cur.tile), n_stage = cur.n_stage;
      int hpos[2][2];   // position of row (half, a/b); -1: padding row, fully masked
      bool hlive[2];    // the half holds a live row (warp-uniform)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        hlive[h] = rb_of_half[h] * 16 < rows_here;
#pragma unroll
        for (int ab = 0; ab < 2; ++ab) {
          const int r = row_of(h, (lane >> 2) + 8 * ab);
          hpos[h][ab] = r < rows_here ? cur.p0 + (cur.tile * ROWS + r) / G : -1;
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
        // masked S fragment of half h (keys beyond a row's position -> -inf)
        auto load_s = [&](int h, uint32_t* sv) {
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
        };
        // raw-score row max over the 4 threads of the row; the log2-domain scale is folded into the
        // exponent's fma (scale > 0: the max of the scaled scores is the scaled max, exactly)
        auto block_max = [&](const uint32_t* sv, float* bm) {
          const float* sc = reinterpret_cast<const float*>(sv);
#pragma unroll
          for (int ab = 0; ab < 2; ++ab) {
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int i = 0; i < KS / 8; ++i) {
              mx0 = fmaxf(mx0, sc[4 * i + 2 * ab]);
              mx1 = fmaxf(mx1, sc[4 * i + 2 * ab + 1]);
            }
            float mx = fmaxf(mx0, mx1);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            bm[ab] = mx * scale_log2;
          }
        };
        // pass 1: block maxima (independent of the running reference), so the reference can be handed to
        // the other set before this set's exponentials -- the sets then overlap instead of alternating.  The
        // fragment is re-read from TMEM for pass 2 rather than held across the hand-off (register pressure)
        float bm[2][2] = {{-INFINITY, -INFINITY}, {-INFINITY, -INFINITY}};
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (hlive[h]) {
            uint32_t sv[64];
            load_s(h, sv);
            block_max(sv, bm[h]);
          }
        // the reference after stage gs-1 (the other set's); -inf at the item's first stage
        if (gs >= 1) MBAR_WAIT(&m_ready[(gs - 1) & 1], ((gs - 1) >> 1) & 1, 12, gs);
        float fac[2][2] = {{1.f, 1.f}, {1.f, 1.f}};
        float sub[2][2];
        bool resc_any = false;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ab = 0; ab < 2; ++ab) {
            const int ln = lane_of(h, ab);
            const float m_ref = st > 0 ? m_sh[ln] : -INFINITY;
            float m_new = m_ref;
            if (hlive[h] && bm[h][ab] > -INFINITY) {
              if (m_ref == -INFINITY) {
                m_new = bm[h][ab];   // first visible block: O and l are still 0
              } else if (bm[h][ab] > m_ref + 8.f) {
                m_new = bm[h][ab];
                fac[h][ab] = ex2f(m_ref - m_new);
                resc_any = true;
              }
            }
            if (hlive[h] && q4 == 0) m_sh[ln] = m_new;
            sub[h][ab] = m_new == -INFINITY ? 0.f : m_new;
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(&m_ready[gs & 1]);
        // pass 2: P = 2^(s * scale - reference), packed bf16 over the first KS/2 columns of S_gs (this set
        // has read them; the MMA warp reads P once p_full is signalled)
        auto exp_pack = [&](int h, const uint32_t* sv) {
          uint32_t pk[32];
          const float* sc = reinterpret_cast<const float*>(sv);
#pragma unroll
          for (int ab = 0; ab < 2; ++ab) {
            float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
            for (int i = 0; i < KS / 8; ++i) {
              const float p0 = ex2f(fmaf(sc[4 * i + 2 * ab], scale_log2, -sub[h][ab]));
              const float p1 = ex2f(fmaf(sc[4 * i + 2 * ab + 1], scale_log2, -sub[h][ab]));
              ls0 += p0;
              ls1 += p1;
              pk[2 * i + ab] = pack2(p0, p1);
            }
            lsum[h][ab] = fmaf(lsum[h][ab], fac[h][ab], ls0 + ls1);
          }
          tmem_st_16x128b_x16(t_s + ((uint32_t)(16 * h) << 16), pk);
        };
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (hlive[h]) {
            uint32_t sv[64];
            load_s(h, sv);
            exp_pack(h, sv);
          }
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
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        if (quarter == 2 && lane == 0) TC_TRACE(3, gs);
#ifdef HM_TC_QCPASYNC
        if (q_pending) {
          q_ready((k + 1) & 1);
          q_pending = false;
        }
#endif
      }
#ifdef HM_TC_QCPASYNC
      if (q_pending) q_ready((k + 1) & 1);
#endif
      if (quarter == 2 && lane == 0) TC_TRACE(set == 0 ? 10 : 13, items);
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
      float* lbuf = l_sh + (items & 1) * ROWS;   // per item parity: one set may run an item ahead
      // The set that ran the item's last stage writes its output; the other set takes the next item's first
      // stage meanwhile, so the epilogue is off the next item's critical path
      const int E = (int)((g + n_stage - 1) & 1);
      if (set != E) {
        // hand this set's sums of P over to the epilogue
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ab = 0; ab < 2; ++ab)
            if (q4 == 0) lbuf[lane_of(h, ab)] = lsum[h][ab];
        __syncwarp();
        if (lane == 0) mbar_arrive(&l_ready[items & 1]);
      } else {
        // epilogue, once every product of the item is done: O / l for the live rows
        // per item parity: the set running the next item's epilogue may get here before this item's O is
        // complete (S runs ahead across items), and a single barrier's parity would alias
        MBAR_WAIT(&o_ready[items & 1], (items >> 1) & 1, 10, (int)g);
        tc_fence_after();
        if (quarter == 2 && lane == 0) TC_TRACE(6, items);
        MBAR_WAIT(&l_ready[items & 1], (items >> 1) & 1, 13, (int)g);
        if (quarter == 2 && lane == 0) TC_TRACE(11, items);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ab = 0; ab < 2; ++ab)
            if (q4 == 0) lbuf[lane_of(h, ab)] += lsum[h][ab];
        __syncwarp();
        if (hlive[0] || hlive[1]) {   // the warp holds a live row
          const int re = cur.tile * ROWS + row_of(lane >> 4, lane & 15);   // this thread's row (TMEM lane tl)
          const bool live = re < cur.qlen * G;
          const float lrow = lbuf[tl];
          const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
          __nv_bfloat16* dst =
              out + ((size_t)(cur.qo + (live ? re / G : 0)) * H + cur.kvh * G + (live ? re % G : 0)) * HD;
#pragma unroll
          for (int c2 = 0; c2 < HD / 64; ++c2) {   // 64 columns per TMEM round trip
            uint32_t o[64];
            tmem_ld32_nw(t_lane + C::COL_O + c2 * 64, o);
            tmem_ld32_nw(t_lane + C::COL_O + c2 * 64 + 32, o + 32);
            tmem_wait_ld();
#ifdef HM_TC_NOSTORE   // timing experiment only: epilogue without its global stores
            if (live && inv == 12345.f) {
#else
            if (live) {
#endif
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const float* f = reinterpret_cast<const float*>(o + 8 * v);
                uint4 w;
                w.x = pack2(f[0] * inv, f[1] * inv);
                w.y = pack2(f[2] * inv, f[3] * inv);
                w.z = pack2(f[4] * inv, f[5] * inv);
                w.w = pack2(f[6] * inv, f[7] * inv);
#ifdef HM_TC_STORE_CS   // A/B: streaming (evict-first) output stores
                __stcs(reinterpret_cast<uint4*>(dst + c2 * 64 + 8 * v), w);
#else
                *reinterpret_cast<uint4*>(dst + c2 * 64 + 8 * v) = w;
#endif
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free);
        if (quarter == 2 && lane == 0) TC_TRACE(7, items);
      }
      g += n_stage;
      cur = nxt;
      nxt = nn;
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
                   const int32_t* d_kv_slot, int32_t n_seq, int32_t H, int32_t KVH, int32_t q_rows, int32_t max_len,
                   float scale_log2, void* d_out, const int32_t* d_work, const CUtensorMap& mq, const CUtensorMap& mk,
                   const CUtensorMap& mv, const CUtensorMap& mk64, const CUtensorMap& mv64, cudaStream_t st) {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_attn_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcAttn<HD>::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, dev);   // one CTA per SM (512 TMEM columns)
    if (getenv("HM_TC_GRID")) grid = atoi(getenv("HM_TC_GRID"));          // debugging only
  }
  k_attn_tc<HD><<<hm_cap(grid, true), 320, TcAttn<HD>::SMEM, st>>>((const __nv_bfloat16*)d_q, d_q_off, d_q_len, d_pos0, d_kv_slot,
                                                      H, KVH, q_rows, max_len, scale_log2, (__nv_bfloat16*)d_out, n_seq,
                                                      d_work, mq, mk, mv, mk64, mv64);
  return 0;
}

#ifdef HM_TC_TRACE
extern "C" int hm_debug_attn_trace(long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_tc_trace, sizeof(g_tc_trace));
}
#endif

template int launch_attn_tc<64>(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, int32_t,
                                int32_t, int32_t, int32_t, int32_t, float, void*, const int32_t*, const CUtensorMap&,
                                const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                                cudaStream_t);
template int launch_attn_tc<128>(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, int32_t,
                                 int32_t, int32_t, int32_t, int32_t, float, void*, const int32_t*, const CUtensorMap&,
                                 const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                                 cudaStream_t);

}  // namespace hm
