// K6: fused accept + AIMD window + prefix policy + stats (+ implicit KV
// rollback: the engine derives kv_len from gen_len), one warp per sequence.
// Restates rhymesim/spec_engine.py:200-240 (step_response) with
// verify :100-107, next_window :49-53, choose_prefix :69-72, stats :124-133.
//
// Also the whole-response replay kernel (spec_engine.py:260-279) that fuses
// K2 + K6 in registers: the draft never leaves the warp.
#include "hs_common.cuh"

namespace hs {
namespace acc {

__device__ __forceinline__ void probe(const HsIndexView& V, int32_t slot, int32_t m, int32_t pre_j,
                                      int32_t* pos_out, bool* found_out) {
  const int lane = lane_id();
  uint64_t term = lane < m ? gram_term(pre_j, lane) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
  const uint64_t h = mix64(gram_seed(slot, m) + term);
  const int32_t tag = gram_tag(h, m);
  const int64_t lo = V.slot_text_off[slot], hi = V.slot_text_off[slot + 1];
  int64_t base = (int64_t)(h & (uint64_t)V.table_mask);
  for (;;) {
    HsGramEntry e = V.table[(base + lane) & V.table_mask];
    bool empty = e.pos < 0;
    bool cand = !empty && e.tag == tag && e.pos >= lo && e.pos < hi;
    unsigned empties = __ballot_sync(0xffffffffu, empty);
    unsigned cands = __ballot_sync(0xffffffffu, cand);
    unsigned live = empties ? ((1u << (__ffs(empties) - 1)) - 1u) : 0xffffffffu;
    cands &= live;
    while (cands) {
      int src = __ffs(cands) - 1;
      int32_t pos = __shfl_sync(0xffffffffu, e.pos, src);
      int32_t t = lane < m ? V.text[pos + lane] : 0;
      unsigned bad = __ballot_sync(0xffffffffu, lane < m && t != pre_j);
      if (!bad) { *pos_out = pos; *found_out = true; return; }
      cands &= cands - 1;
    }
    if (empties) { *found_out = false; return; }
    base += 32;
  }
}

// Accept core.  truth_i(i) gives the verified next token after i accepted
// draft tokens; lane j holds draft token d_j (j < k).
template <typename TruthFn>
__device__ __forceinline__ void accept_core(int32_t k, int32_t d_j, int32_t pos, int32_t tgt, TruthFn truth_i,
                                            int32_t* __restrict__ gen_row, int32_t* appended_out,
                                            int32_t* bonus_out, bool* all_out) {
  const int lane = lane_id();
  int32_t rest = tgt - pos;
  int32_t t_j = (lane < k && lane < rest) ? truth_i(lane) : 0;
  bool ok = lane < k && lane < rest && t_j == d_j;
  unsigned bad = __ballot_sync(0xffffffffu, lane < k && !ok);
  int32_t a = bad ? (__ffs(bad) - 1) : k;
  int32_t appended = a < rest ? a : rest;
  int32_t bonus = (pos + appended < tgt) ? 1 : 0;
  if (gen_row) {
    if (lane < appended) gen_row[pos + lane] = d_j;
  }
  int32_t bonus_tok = 0;
  if (bonus) bonus_tok = truth_i(appended);   // uniform across the warp
  if (gen_row && bonus && lane == 0) gen_row[pos + appended] = bonus_tok;
  *appended_out = appended;
  *bonus_out = bonus;
  *all_out = (a == k);
}

struct ReplayTruth {
  const int32_t* row;  // truth of this sequence
  int32_t pos;
  __device__ __forceinline__ int32_t operator()(int32_t i) const { return row[pos + i]; }
};
struct ArgmaxTruth {
  const int32_t* rows;  // argmax of the verify rows of this sequence
  __device__ __forceinline__ int32_t operator()(int32_t i) const { return rows[i]; }
};

template <typename MakeTruth>
__device__ __forceinline__ void step_seq(int64_t s, MakeTruth make_truth, const int32_t* __restrict__ target_len,
                                         const int32_t* __restrict__ draft_tok, int32_t draft_stride,
                                         const int32_t* __restrict__ draft_len, const uint8_t* __restrict__ looked,
                                         const uint8_t* __restrict__ found, int32_t* __restrict__ gen_tok,
                                         int32_t gen_stride, int32_t* __restrict__ gen_len,
                                         int32_t* __restrict__ window, int32_t* __restrict__ prefix_len,
                                         int64_t* __restrict__ stats, int32_t* __restrict__ tpi, int32_t tpi_stride,
                                         int32_t* __restrict__ n_iter, const HsSpecConfig& cfg) {
  const int lane = lane_id();
  int32_t pos = gen_len[s], tgt = target_len[s];
  if (pos >= tgt) return;  // ResponseComplete: finished rows are skipped
  int32_t k = draft_len[s];
  int32_t* row = gen_tok + s * (int64_t)gen_stride;
  auto truth = make_truth(s, pos);
  int64_t* st = stats + 5 * s;
  int32_t tpi_val;
  if (k == 0) {
    if (lane == 0) {
      row[pos] = truth(0);
      gen_len[s] = pos + 1;
      st[0] += 1;
      st[4] += 1;
      if (looked[s]) {
        int32_t cur = prefix_len[s];
        prefix_len[s] = found[s] ? cfg.prefix_init : (cur - 1 > cfg.prefix_min ? cur - 1 : cfg.prefix_min);
      }
    }
    tpi_val = 1;
  } else {
    int32_t d_j = lane < k ? draft_tok[s * (int64_t)draft_stride + lane] : 0;
    int32_t appended, bonus;
    bool all;
    accept_core(k, d_j, pos, tgt, truth, row, &appended, &bonus, &all);
    if (lane == 0) {
      gen_len[s] = pos + appended + bonus;
      st[0] += appended + bonus;
      st[1] += k;
      st[2] += appended;
      st[3] += 1;
      int32_t w = window[s];
      window[s] = all ? (w + cfg.window_add < cfg.window_max ? w + cfg.window_add : cfg.window_max) : cfg.window_init;
      prefix_len[s] = cfg.prefix_init;
    }
    tpi_val = appended + bonus;
  }
  if (tpi && lane == 0) {
    int32_t it = n_iter[s];
    tpi[s * (int64_t)tpi_stride + it] = tpi_val;
    n_iter[s] = it + 1;
  } else if (n_iter && lane == 0) {
    n_iter[s] += 1;
  }
}

__global__ void __launch_bounds__(256) k_accept_replay(int32_t n_seq, const int32_t* __restrict__ truth,
                                                       int32_t truth_stride, const int32_t* __restrict__ target_len,
                                                       const int32_t* __restrict__ draft_tok, int32_t draft_stride,
                                                       const int32_t* __restrict__ draft_len,
                                                       const uint8_t* __restrict__ looked,
                                                       const uint8_t* __restrict__ found, int32_t* __restrict__ gen_tok,
                                                       int32_t gen_stride, int32_t* __restrict__ gen_len,
                                                       int32_t* __restrict__ window, int32_t* __restrict__ prefix_len,
                                                       int64_t* __restrict__ stats, int32_t* __restrict__ tpi,
                                                       int32_t tpi_stride, int32_t* __restrict__ n_iter,
                                                       HsSpecConfig cfg) {
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_seq) return;
  auto mk = [&](int64_t seq, int32_t pos) { return ReplayTruth{truth + seq * (int64_t)truth_stride, pos}; };
  step_seq(s, mk, target_len, draft_tok, draft_stride, draft_len, looked, found, gen_tok, gen_stride, gen_len,
           window, prefix_len, stats, tpi, tpi_stride, n_iter, cfg);
}

__global__ void __launch_bounds__(256) k_accept_greedy(int32_t n_seq, const int32_t* __restrict__ argmax,
                                                       const int32_t* __restrict__ q_off,
                                                       const int32_t* __restrict__ target_len,
                                                       const int32_t* __restrict__ draft_tok, int32_t draft_stride,
                                                       const int32_t* __restrict__ draft_len,
                                                       const uint8_t* __restrict__ looked,
                                                       const uint8_t* __restrict__ found, int32_t* __restrict__ gen_tok,
                                                       int32_t gen_stride, int32_t* __restrict__ gen_len,
                                                       int32_t* __restrict__ window, int32_t* __restrict__ prefix_len,
                                                       int64_t* __restrict__ stats, int32_t* __restrict__ tpi,
                                                       int32_t tpi_stride, int32_t* __restrict__ n_iter,
                                                       HsSpecConfig cfg) {
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_seq) return;
  auto mk = [&](int64_t seq, int32_t) { return ArgmaxTruth{argmax + q_off[seq]}; };
  step_seq(s, mk, target_len, draft_tok, draft_stride, draft_len, looked, found, gen_tok, gen_stride, gen_len,
           window, prefix_len, stats, tpi, tpi_stride, n_iter, cfg);
}

// cmp of the first m tokens of suffix p against the prefix (lanes chunked)
__device__ __forceinline__ int cmp_suffix(const int32_t* __restrict__ text, int32_t p,
                                          const int32_t* __restrict__ pre, int32_t m) {
  const int lane = lane_id();
  for (int32_t c = 0; c < m; c += 32) {
    int32_t j = c + lane;
    int32_t a = 0, b = 0;
    bool diff = false;
    if (j < m) { a = text[p + j]; b = pre[j]; diff = a != b; }
    unsigned d = __ballot_sync(0xffffffffu, diff);
    if (d) {
      int src = __ffs(d) - 1;
      int32_t x = __shfl_sync(0xffffffffu, a, src), y = __shfl_sync(0xffffffffu, b, src);
      return x < y ? -1 : 1;
    }
  }
  return 0;
}

// SA path for prefix lengths outside the table range
__device__ void lookup_sa(const HsIndexView& V, int32_t slot, const int32_t* pre, int32_t m, int32_t* pos_out,
                          bool* found_out) {
  const int lane = lane_id();
  int64_t S = V.slot_sa_off[slot], E = V.slot_sa_off[slot + 1];
  int64_t lo = S, hi = E;
  while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (cmp_suffix(V.text, V.sa[mid], pre, m) < 0) lo = mid + 1; else hi = mid; }
  int64_t first = lo;
  hi = E;
  while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (cmp_suffix(V.text, V.sa[mid], pre, m) <= 0) lo = mid + 1; else hi = mid; }
  int64_t last = lo;
  if (first == last) { *found_out = false; return; }
  *found_out = true;
  if (last - first == 1) { *pos_out = V.sa[first]; return; }
  int32_t best = 0x7fffffff;
  int64_t bidx = -1;
  for (int64_t k = first + 1 + lane; k < last; k += 32) {
    int32_t v = V.lcp[k];
    if (v < best) { best = v; bidx = k; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    int32_t ov = __shfl_xor_sync(0xffffffffu, best, o);
    int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov < best || (ov == best && oi >= 0 && (bidx < 0 || oi < bidx))) { best = ov; bidx = oi; }
  }
  *pos_out = V.heavy[bidx];
}

// Whole responses: warp per truth row, loops until done.
__global__ void __launch_bounds__(256) k_replay_fused(HsIndexView V, int32_t n_seq,
                                                      const int32_t* __restrict__ slot_of_seq,
                                                      const int32_t* __restrict__ truth_all,
                                                      const int64_t* __restrict__ truth_off,
                                                      const uint8_t* __restrict__ speculate,
                                                      int32_t* __restrict__ tpi, int32_t* __restrict__ n_iter,
                                                      int64_t* __restrict__ stats, HsSpecConfig cfg) {
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_seq) return;
  const int lane = lane_id();
  const int32_t* truth = truth_all + truth_off[s];
  int32_t n = (int32_t)(truth_off[s + 1] - truth_off[s]);
  int32_t slot = slot_of_seq[s];
  bool spec = cfg.enabled && speculate[s] && slot >= 0 && slot < V.n_slots;
  int32_t window = cfg.window_init, cur = cfg.prefix_init, pos = 0, iters = 0;
  int64_t st_total = 0, st_spec = 0, st_acc = 0, st_ver = 0, st_dec = 0;
  int32_t* tpi_row = tpi ? tpi + truth_off[s] : nullptr;
  while (pos < n) {
    int32_t k = 0, d_j = 0;
    bool looked = spec && pos >= cur, hit = false;
    if (looked) {
      int32_t hpos = -1;
      if (V.table && cur >= V.prefix_min && cur <= V.prefix_max) {
        int32_t pj = lane < cur ? truth[pos - cur + lane] : 0;
        probe(V, slot, cur, pj, &hpos, &hit);
      } else {
        lookup_sa(V, slot, truth + pos - cur, cur, &hpos, &hit);
      }
      if (hit) {
        int32_t t = lane < window ? V.text[hpos + cur + lane] : 0;
        unsigned term = __ballot_sync(0xffffffffu, lane < window && t < 0);
        k = term ? (__ffs(term) - 1) : window;
        d_j = t;
      }
    }
    int32_t step;
    if (k == 0) {
      step = 1;
      st_total += 1;
      st_dec += 1;
      if (looked) cur = hit ? cfg.prefix_init : (cur - 1 > cfg.prefix_min ? cur - 1 : cfg.prefix_min);
    } else {
      int32_t appended, bonus;
      bool all;
      accept_core(k, d_j, pos, n, ReplayTruth{truth, pos}, nullptr, &appended, &bonus, &all);
      step = appended + bonus;
      st_total += step;
      st_spec += k;
      st_acc += appended;
      st_ver += 1;
      window = all ? (window + cfg.window_add < cfg.window_max ? window + cfg.window_add : cfg.window_max)
                   : cfg.window_init;
      cur = cfg.prefix_init;
    }
    if (tpi_row && lane == 0) tpi_row[iters] = step;
    iters += 1;
    pos += step;
  }
  if (lane == 0) {
    n_iter[s] = iters;
    int64_t* o = stats + 5 * s;
    o[0] = st_total; o[1] = st_spec; o[2] = st_acc; o[3] = st_ver; o[4] = st_dec;
  }
}

}  // namespace acc
}  // namespace hs

using namespace hs;

static int check_cfg(const HsSpecConfig& c) {
  if (!(1 <= c.window_init && c.window_init <= c.window_max && c.window_max <= HS_MAX_WINDOW && c.window_add >= 0)) {
    hs_set_error("window invariant violated (1 <= init <= max <= 32)");
    return HS_ERR_INVALID;
  }
  if (!(1 <= c.prefix_min && c.prefix_min <= c.prefix_init)) {
    hs_set_error("prefix invariant violated");
    return HS_ERR_INVALID;
  }
  return HS_OK;
}

extern "C" int hs_accept_replay(int32_t n_seq, const int32_t* d_truth, int32_t truth_stride,
                                const int32_t* d_target_len, const int32_t* d_draft_tok, int32_t draft_stride,
                                const int32_t* d_draft_len, const uint8_t* d_looked, const uint8_t* d_found,
                                int32_t* d_gen_tok, int32_t gen_stride, int32_t* d_gen_len, int32_t* d_window,
                                int32_t* d_prefix_len, int64_t* d_stats, int32_t* d_tpi, int32_t tpi_stride,
                                int32_t* d_n_iter, HsSpecConfig cfg, hs_stream_t stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n_seq <= 0) return HS_OK;
  int64_t blocks = ((int64_t)n_seq * 32 + 255) / 256;
  hs_count_launches(1);
  acc::k_accept_replay<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      n_seq, d_truth, truth_stride, d_target_len, d_draft_tok, draft_stride, d_draft_len, d_looked, d_found, d_gen_tok,
      gen_stride, d_gen_len, d_window, d_prefix_len, d_stats, d_tpi, tpi_stride, d_n_iter, cfg);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_accept_greedy(int32_t n_seq, const int32_t* d_argmax, const int32_t* d_q_off,
                                const int32_t* d_target_len, const int32_t* d_draft_tok, int32_t draft_stride,
                                const int32_t* d_draft_len, const uint8_t* d_looked, const uint8_t* d_found,
                                int32_t* d_gen_tok, int32_t gen_stride, int32_t* d_gen_len, int32_t* d_window,
                                int32_t* d_prefix_len, int64_t* d_stats, int32_t* d_tpi, int32_t tpi_stride,
                                int32_t* d_n_iter, HsSpecConfig cfg, hs_stream_t stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n_seq <= 0) return HS_OK;
  int64_t blocks = ((int64_t)n_seq * 32 + 255) / 256;
  hs_count_launches(1);
  acc::k_accept_greedy<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      n_seq, d_argmax, d_q_off, d_target_len, d_draft_tok, draft_stride, d_draft_len, d_looked, d_found, d_gen_tok,
      gen_stride, d_gen_len, d_window, d_prefix_len, d_stats, d_tpi, tpi_stride, d_n_iter, cfg);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

namespace hs {
namespace acc {

// Continuous batching: (re)initialise engine lanes for newly admitted sequences (one CTA per lane).
// Lane state becomes that of a ResponseContext (spec_engine.py:174-187) holding tokens[off_i : off_i+1]
// (a migrated rollout's generated prefix, or nothing) followed by argmax[first_row_i] when first_row_i >= 0
// (the token the admission prefill produced), with the carried AIMD window, prefix length and stats.
__global__ void k_lane_admit(int32_t n, const int32_t* __restrict__ lane, const int32_t* __restrict__ tok,
                             const int64_t* __restrict__ tok_off, const int32_t* __restrict__ argmax,
                             const int32_t* __restrict__ first_row, const int32_t* __restrict__ target,
                             const int32_t* __restrict__ slot, const uint8_t* __restrict__ spec,
                             const int32_t* __restrict__ window_in, const int32_t* __restrict__ prefix_in,
                             const int64_t* __restrict__ stats_in, const int32_t* __restrict__ prompt_len_in,
                             const int32_t* __restrict__ key_in, int32_t* __restrict__ gen_tok, int32_t gen_stride,
                             int32_t* __restrict__ gen_len, int32_t* __restrict__ target_len,
                             int32_t* __restrict__ slots, uint8_t* __restrict__ speculate,
                             int32_t* __restrict__ window, int32_t* __restrict__ prefix_len,
                             int64_t* __restrict__ stats, int32_t* __restrict__ draft_len,
                             uint8_t* __restrict__ looked, uint8_t* __restrict__ found,
                             int32_t* __restrict__ prompt_len, int32_t* __restrict__ seq_key) {
  for (int32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int32_t l = lane[i];
    const int64_t o = tok_off[i];
    const int32_t g = (int32_t)(tok_off[i + 1] - o);
    int32_t* row = gen_tok + (int64_t)l * gen_stride;
    for (int32_t j = threadIdx.x; j < g; j += blockDim.x) row[j] = tok[o + j];
    if (threadIdx.x == 0) {
      const int32_t fr = first_row[i];
      if (fr >= 0) row[g] = argmax[fr];
      gen_len[l] = g + (fr >= 0 ? 1 : 0);
      target_len[l] = target[i];
      slots[l] = slot[i];
      speculate[l] = spec[i];
      window[l] = window_in[i];
      prefix_len[l] = prefix_in[i];
#pragma unroll
      for (int c = 0; c < 5; ++c) stats[5 * (int64_t)l + c] = stats_in[5 * (int64_t)i + c];
      draft_len[l] = 0;
      looked[l] = 0;
      found[l] = 0;
      if (prompt_len) prompt_len[l] = prompt_len_in[i];
      if (seq_key) seq_key[l] = key_in[i];
    }
  }
}

}  // namespace acc
}  // namespace hs

extern "C" int hs_lane_admit(int32_t n, const int32_t* d_lane, const int32_t* d_tok, const int64_t* d_tok_off,
                             const int32_t* d_argmax, const int32_t* d_first_row, const int32_t* d_target,
                             const int32_t* d_slot, const uint8_t* d_spec, const int32_t* d_window,
                             const int32_t* d_prefix, const int64_t* d_stats, const int32_t* d_prompt_len_in,
                             const int32_t* d_key_in, int32_t* d_gen_tok, int32_t gen_stride, int32_t* d_gen_len,
                             int32_t* d_target_len, int32_t* d_slots, uint8_t* d_speculate, int32_t* d_window_out,
                             int32_t* d_prefix_out, int64_t* d_stats_out, int32_t* d_draft_len, uint8_t* d_looked,
                             uint8_t* d_found, int32_t* d_prompt_len, int32_t* d_seq_key, hs_stream_t stream) {
  if (n < 0 || gen_stride < 1) {
    hs_set_error("hs_lane_admit: n >= 0 and gen_stride >= 1 required");
    return HS_ERR_INVALID;
  }
  if ((d_prompt_len == nullptr) != (d_prompt_len_in == nullptr) || (d_seq_key == nullptr) != (d_key_in == nullptr)) {
    hs_set_error("hs_lane_admit: per-lane prompt_len / seq_key inputs and outputs go together");
    return HS_ERR_INVALID;
  }
  if (n == 0) return HS_OK;
  hs_count_launches(1);
  acc::k_lane_admit<<<n < 1024 ? n : 1024, 128, 0, (cudaStream_t)stream>>>(
      n, d_lane, d_tok, d_tok_off, d_argmax, d_first_row, d_target, d_slot, d_spec, d_window, d_prefix, d_stats,
      d_prompt_len_in, d_key_in, d_gen_tok, gen_stride, d_gen_len, d_target_len, d_slots, d_speculate, d_window_out,
      d_prefix_out, d_stats_out, d_draft_len, d_looked, d_found, d_prompt_len, d_seq_key);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_replay_fused(const HsIndexView* view, int32_t n_seq, const int32_t* d_slot_of_seq,
                               const int32_t* d_truth, const int64_t* d_truth_off, const uint8_t* d_speculate,
                               int32_t* d_tpi, int32_t* d_n_iter, int64_t* d_stats, HsSpecConfig cfg,
                               hs_stream_t stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n_seq <= 0) return HS_OK;
  HsIndexView V = *view;
  int64_t blocks = ((int64_t)n_seq * 32 + 255) / 256;
  hs_count_launches(1);
  acc::k_replay_fused<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(V, n_seq, d_slot_of_seq, d_truth,
                                                                        d_truth_off, d_speculate, d_tpi, d_n_iter,
                                                                        d_stats, cfg);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}
