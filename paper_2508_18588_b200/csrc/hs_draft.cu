// K2: batched draft proposal (warp per sequence) + general SA lookups.
//
// Hot path (spec_engine.py:206-215 -> history.py:302-333): the last m
// generated tokens are hashed, 32 consecutive table entries are probed with
// one coalesced 512 B warp load, a tag hit is verified against the text by
// m lanes at once (ballot), and the draft is text[heavy + m : ...] read by
// `window` lanes in one coalesced load, cut at the first terminal (ballot).
//
// General path (any prefix length, history.py:283-300 match_prefix): warp
// binary search over the slot's suffix array with warp-parallel comparisons,
// then the locus node from a warp min-scan of the LCP values inside the
// interval.
#include <cstdlib>
#include <string>

#include "hs_common.cuh"

namespace hs {

struct Hit {
  int32_t found;
  int32_t pos;      // heavy text position (draft = text[pos + m ...])
  int64_t mass;
  int32_t at_node;
  int32_t depth;    // depth of the locus (m for a match that ends on a node)
};

// Each lane j < m holds pre_j = prefix token j (lanes >= m: ignored).
__device__ __forceinline__ Hit probe_table(const HsIndexView& V, int32_t slot, int32_t m, int32_t pre_j) {
  const int lane = lane_id();
  // every lane computes the same hash from broadcast tokens
  // polynomial hash: lane j contributes term j, butterfly-summed across the warp
  uint64_t term = lane < m ? gram_term(pre_j, lane) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
  const uint64_t h = mix64(gram_seed(slot, m) + term);
  const int32_t tag = gram_tag(h, m);
  const int64_t lo = V.slot_text_off[slot], hi = V.slot_text_off[slot + 1];
  int64_t base = (int64_t)(h & (uint64_t)V.table_mask);
  Hit r{0, -1, 0, 0, 0};
  for (;;) {
    HsGramEntry e = V.table[(base + lane) & V.table_mask];
    bool empty = e.pos < 0;
    bool cand = !empty && e.tag == tag && e.pos >= lo && e.pos < hi;
    unsigned empties = __ballot_sync(0xffffffffu, empty);
    unsigned cands = __ballot_sync(0xffffffffu, cand);
    // lanes before the first empty slot are the live probe sequence
    unsigned live = empties ? ((1u << (__ffs(empties) - 1)) - 1u) : 0xffffffffu;
    cands &= live;
    while (cands) {
      int src = __ffs(cands) - 1;
      int32_t pos = __shfl_sync(0xffffffffu, e.pos, src);
      int32_t t = lane < m ? V.text[pos + lane] : 0;
      unsigned bad = __ballot_sync(0xffffffffu, lane < m && t != pre_j);
      if (!bad) {
        r.found = 1;
        r.pos = pos;
        // masses sit in a parallel array after the entries (the draft hot path never reads them)
        r.mass = reinterpret_cast<const int64_t*>(V.table + (V.table_mask + 1))[(base + src) & V.table_mask];
        return r;
      }
      cands &= cands - 1;
    }
    if (empties) return r;
    base += 32;
  }
}

// Three-way compare of the first m tokens of suffix p with the prefix
// (held in lanes, chunked by 32). Returns <0, 0, >0 (suffix vs prefix).
__device__ __forceinline__ int cmp_suffix(const int32_t* __restrict__ text, int32_t p,
                                          const int32_t* __restrict__ pre, int32_t m) {
  const int lane = lane_id();
  for (int32_t c = 0; c < m; c += 32) {
    int32_t j = c + lane;
    int32_t a = 0, b = 0;
    bool diff = false;
    if (j < m) {
      a = text[p + j];
      b = pre[j];
      diff = a != b;
    }
    unsigned d = __ballot_sync(0xffffffffu, diff);
    if (d) {
      int src = __ffs(d) - 1;
      int32_t x = __shfl_sync(0xffffffffu, a, src);
      int32_t y = __shfl_sync(0xffffffffu, b, src);
      return x < y ? -1 : 1;   // the terminal (-1) sorts below every token
    }
  }
  return 0;
}

__device__ Hit lookup_general(const HsIndexView& V, int32_t slot, const int32_t* __restrict__ pre, int32_t m) {
  const int lane = lane_id();
  Hit r{0, -1, 0, 0, 0};
  int64_t S = V.slot_sa_off[slot], E = V.slot_sa_off[slot + 1];
  // lower bound: first suffix whose m-prefix >= pre
  int64_t lo = S, hi = E;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cmp_suffix(V.text, V.sa[mid], pre, m) < 0) lo = mid + 1; else hi = mid;
  }
  int64_t first = lo;
  hi = E;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cmp_suffix(V.text, V.sa[mid], pre, m) <= 0) lo = mid + 1; else hi = mid;
  }
  int64_t last = lo;  // exclusive
  if (first == last) return r;
  r.found = 1;
  r.mass = V.wsum[last] - V.wsum[first];
  if (last - first == 1) {
    r.pos = V.sa[first];
    r.depth = m;   // inside a leaf edge (the terminal follows at the earliest)
    r.at_node = 0;
    return r;
  }
  // locus: first position of the minimum LCP inside (first, last)
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
  r.pos = V.heavy[bidx];
  r.depth = best;
  r.at_node = (best == m) && (V.node_flags[bidx] & 2) ? 1 : 0;
  return r;
}

// Copy up to `window` draft tokens text[pos + m ...] into out, stop at the terminal.
__device__ __forceinline__ int32_t read_draft(const int32_t* __restrict__ text, int32_t start, int32_t window,
                                              int32_t* __restrict__ out) {
  const int lane = lane_id();
  int32_t len = 0;
  for (int32_t c = 0; c < window; c += 32) {
    int32_t j = c + lane;
    int32_t t = j < window ? text[start + j] : 0;
    unsigned term = __ballot_sync(0xffffffffu, j < window && t < 0);
    int32_t lim = term ? (__ffs(term) - 1) : 32;
    if (lane < lim && j < window) out[j] = t;
    if (term) return len + lim;
    len += (window - c) < 32 ? (window - c) : 32;
  }
  return len;
}

__global__ void k_lookup_batch(HsIndexView V, int32_t n, const int32_t* __restrict__ slot,
                               const int32_t* __restrict__ prefix, int32_t prefix_stride,
                               const int32_t* __restrict__ prefix_len, const int32_t* __restrict__ window,
                               int32_t* __restrict__ out_tok, int32_t out_stride, int64_t* __restrict__ info,
                               int32_t use_table) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const int lane = lane_id();
  int32_t s = slot[w], m = prefix_len[w], win = window[w];
  const int32_t* pre = prefix + (int64_t)w * prefix_stride;
  Hit h;
  if (s < 0 || s >= V.n_slots || m < 1) {
    h = Hit{0, -1, 0, 0, 0};
  } else if (use_table && V.table && m >= V.prefix_min && m <= V.prefix_max) {
    int32_t pj = lane < m ? pre[lane] : 0;
    h = probe_table(V, s, m, pj);
  } else {
    h = lookup_general(V, s, pre, m);
  }
  int32_t len = 0;
  if (h.found && win > 0) len = read_draft(V.text, h.pos + m, win, out_tok + (int64_t)w * out_stride);
  if (lane == 0) {
    int64_t* o = info + 6 * w;
    o[0] = h.found;
    o[1] = len;
    o[2] = h.mass;
    o[3] = h.at_node;
    o[4] = h.pos;
    o[5] = h.depth;
  }
}

// K2 hot path: one warp per sequence.
__global__ void __launch_bounds__(256) k_draft(HsIndexView V, int32_t n_seq, const int32_t* __restrict__ slot_of_seq,
                                               const int32_t* __restrict__ gen_tok, int32_t gen_stride,
                                               const int32_t* __restrict__ gen_len,
                                               const int32_t* __restrict__ prefix_len,
                                               const int32_t* __restrict__ window,
                                               const uint8_t* __restrict__ speculate,
                                               int32_t* __restrict__ draft_tok, int32_t draft_stride,
                                               int32_t* __restrict__ draft_len, uint8_t* __restrict__ looked,
                                               uint8_t* __restrict__ found) {
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_seq) return;
  const int lane = lane_id();
  int32_t m = prefix_len[s], pos = gen_len[s], slot = slot_of_seq[s];
  bool look = speculate[s] && slot >= 0 && pos >= m;
  int32_t len = 0;
  bool hit = false;
  if (look) {
    const int32_t* row = gen_tok + (int64_t)s * gen_stride + pos - m;
    Hit h;
    if (V.table && m >= V.prefix_min && m <= V.prefix_max) {
      int32_t pj = lane < m ? row[lane] : 0;
      h = probe_table(V, slot, m, pj);
    } else {
      h = lookup_general(V, slot, row, m);
    }
    hit = h.found;
    if (hit) len = read_draft(V.text, h.pos + m, window[s], draft_tok + (int64_t)s * draft_stride);
  }
  if (lane == 0) {
    draft_len[s] = len;
    looked[s] = look;
    found[s] = hit;
  }
}

// K2, 8-lane groups: four sequences per warp (4x the memory-level parallelism
// of one warp per sequence).  Used when prefix_len <= 8 and window <= 32,
// i.e. the whole hot path (SpecConfig defaults 7 / 32).  Within a group:
// lane j holds prefix token j, probes table entry base + j (8 x 16 B = one
// 128 B line), verifies a tag hit with one compare per lane + group ballot,
// and reads/writes the draft as 4 coalesced 32 B rows (tokens j, j+8, ...).
//
// FUSED (default): the common case -- the first probed row holds the key --
// is resolved in one round trip after the table load: the first live
// candidate's verify tokens text[pos + j] and draft tokens text[pos + m + ...]
// are requested together; only groups whose first candidate fails (or whose
// key lies beyond the first row) take the general probe loop.
template <bool FUSED>
__global__ void __launch_bounds__(256, 8) k_draft8(HsIndexView V, int32_t n_seq, const int32_t* __restrict__ slot_of_seq,
                                                const int32_t* __restrict__ gen_tok, int32_t gen_stride,
                                                const int32_t* __restrict__ gen_len,
                                                const int32_t* __restrict__ prefix_len,
                                                const int32_t* __restrict__ window,
                                                const uint8_t* __restrict__ speculate,
                                                int32_t* __restrict__ draft_tok, int32_t draft_stride,
                                                int32_t* __restrict__ draft_len, uint8_t* __restrict__ looked,
                                                uint8_t* __restrict__ found) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3, j = lane & 7;
  const unsigned gmask = 0xFFu << (g * 8);
  int64_t s = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4 + g;
  const bool valid = s < n_seq;
  if (!valid) s = n_seq - 1;   // keep the whole warp converged; results discarded
  const int32_t m = prefix_len[s], pos = gen_len[s], slot = slot_of_seq[s];
  const int32_t win = window[s];
  const bool look = valid && speculate[s] && slot >= 0 && pos >= m && V.table && m >= V.prefix_min &&
                    m <= V.prefix_max;
  int32_t pre_j = 0;
  if (look && j < m) pre_j = gen_tok[s * (int64_t)gen_stride + pos - m + j];
  // hash (identical in every lane of the group)
  // polynomial hash: lane j of the group contributes term j; 3-step butterfly inside the 8 lanes
  uint64_t term = (look && j < m) ? gram_term(pre_j, j) : 0ull;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
  const uint64_t h = mix64(gram_seed(slot, m) + term);
  const int32_t tag = gram_tag(h, m);
  int32_t hit_pos = -1;
  bool done = !look;
  int64_t base = (int64_t)(h & (uint64_t)V.table_mask);
  const int64_t lo = look ? V.slot_text_off[slot] : 0, hi = look ? V.slot_text_off[slot + 1] : 0;
  int32_t t4[4] = {0, 0, 0, 0};   // draft tokens text[hit_pos + m + r*8 + j]
  bool have_t4 = false;
  if (FUSED) {
    HsGramEntry e;
    e.pos = -1;
    e.tag = 0;
    if (look) e = V.table[(base + j) & V.table_mask];
    const bool empty = look && e.pos < 0;
    const bool cand = look && !empty && e.tag == tag && e.pos >= lo && e.pos < hi;
    const unsigned em = (__ballot_sync(0xffffffffu, empty) & gmask) >> (g * 8);
    unsigned cm = (__ballot_sync(0xffffffffu, cand) & gmask) >> (g * 8);
    cm &= em ? ((1u << (__ffs(em) - 1)) - 1u) : 0xFFu;
    const int src = cm ? (g << 3) + __ffs(cm) - 1 : lane;
    const int32_t cpos = __shfl_sync(0xffffffffu, e.pos, src);
    int32_t vt = 0;
    if (cm) {
      vt = j < m ? V.text[cpos + j] : 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) t4[r] = r * 8 + j < win ? V.text[cpos + m + r * 8 + j] : 0;
    }
    const unsigned bm = __ballot_sync(0xffffffffu, cm && j < m && vt != pre_j) & gmask;
    if (cm && !bm) {
      hit_pos = cpos;
      have_t4 = true;
      done = true;
    } else if (!cm && em) {
      done = true;   // an empty slot before any candidate: the key is absent
    }
    // unresolved groups rescan from the first row in the general loop below
  }
  // probe loop: every group iterates until it resolves (warp-uniform trip via __any_sync)
  while (__any_sync(0xffffffffu, !done)) {
    HsGramEntry e;
    e.pos = -1;
    e.tag = 0;
    if (!done) e = V.table[(base + j) & V.table_mask];
    const bool empty = !done && e.pos < 0;
    const bool cand = !done && !empty && e.tag == tag && e.pos >= lo && e.pos < hi;
    unsigned em = (__ballot_sync(0xffffffffu, empty) & gmask) >> (g * 8);
    unsigned cm = (__ballot_sync(0xffffffffu, cand) & gmask) >> (g * 8);
    unsigned live = em ? ((1u << (__ffs(em) - 1)) - 1u) : 0xFFu;
    cm &= live;
    // verify candidates in probe order (rare: at most a couple per query)
    while (__any_sync(0xffffffffu, cm != 0)) {
      const int src = cm ? (g << 3) + __ffs(cm) - 1 : lane;
      const int32_t cpos = __shfl_sync(0xffffffffu, e.pos, src);
      bool bad = false;
      if (cm && j < m) bad = V.text[cpos + j] != pre_j;
      unsigned bm = (__ballot_sync(0xffffffffu, bad) & gmask);
      if (cm) {
        if (!bm) {
          hit_pos = cpos;
          cm = 0;
          em = 1;   // resolved
        } else {
          cm &= cm - 1;
        }
      }
    }
    if (!done && (hit_pos >= 0 || em)) done = true;
    base += 8;
  }
  const bool hit = hit_pos >= 0;
  // draft: tokens text[hit_pos + m + r*8 + j], r = 0..3, cut at the first terminal
  if (hit && !have_t4) {
#pragma unroll
    for (int r = 0; r < 4; ++r) t4[r] = r * 8 + j < win ? V.text[hit_pos + m + r * 8 + j] : 0;
  }
  int32_t first_term = 32;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int idx = r * 8 + j;
    if (hit && idx < win && t4[r] < 0 && idx < first_term) first_term = idx;
  }
  // group min of first_term
  for (int o = 4; o > 0; o >>= 1) first_term = min(first_term, __shfl_xor_sync(0xffffffffu, first_term, o));
  const int32_t len = hit ? min(first_term, win) : 0;
  if (valid) {
    int32_t* out = draft_tok + s * (int64_t)draft_stride;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int idx = r * 8 + j;
      if (idx < len) out[idx] = t4[r];
    }
    if (j == 0) {
      draft_len[s] = len;
      looked[s] = valid && speculate[s] && slot >= 0 && pos >= m;
      found[s] = hit;
    }
  }
}

// K2, 4-lane groups (default): eight sequences per warp, twice the queries in
// flight of k_draft8 at the same occupancy -- the kernel is bound by its chain
// of dependent loads (metadata -> prefix -> table row -> text), not by bytes.
// Lane j of a group holds prefix tokens j and j + 4, probes table entries
// base + 2j and base + 2j + 1 (8 entries of 8 B = one 64 B row), verifies the
// first live candidate with text[pos + j], text[pos + j + 4] and reads its
// draft tokens m + j + 4k (k < 8) in the same round trip.  Groups the first
// row does not decide (the key lies further along the probe sequence, or the
// first candidate fails its text check) take a row loop.
__global__ void __launch_bounds__(256, 8) k_draft4(HsIndexView V, int32_t n_seq, const int32_t* __restrict__ slot_of_seq,
                                                const int32_t* __restrict__ gen_tok, int32_t gen_stride,
                                                const int32_t* __restrict__ gen_len,
                                                const int32_t* __restrict__ prefix_len,
                                                const int32_t* __restrict__ window,
                                                const uint8_t* __restrict__ speculate,
                                                int32_t* __restrict__ draft_tok, int32_t draft_stride,
                                                int32_t* __restrict__ draft_len, uint8_t* __restrict__ looked,
                                                uint8_t* __restrict__ found) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, j = lane & 3;
  int64_t s = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 8 + g;
  const bool valid = s < n_seq;
  if (!valid) s = n_seq - 1;   // keep the whole warp converged; results discarded
  const int32_t m = prefix_len[s], pos = gen_len[s], slot = slot_of_seq[s];
  const int32_t win = window[s];
  const bool look = valid && speculate[s] && slot >= 0 && pos >= m && V.table && m >= V.prefix_min &&
                    m <= V.prefix_max;
  const int32_t* prow = gen_tok + s * (int64_t)gen_stride + pos - m;
  const int32_t pre_a = (look && j < m) ? prow[j] : 0;
  const int32_t pre_b = (look && j + 4 < m) ? prow[j + 4] : 0;
  // polynomial hash: terms j and j + 4 per lane, 2-step butterfly inside the 4 lanes
  uint64_t term = 0ull;
  if (look && j < m) term += gram_term(pre_a, j);
  if (look && j + 4 < m) term += gram_term(pre_b, j + 4);
  term += __shfl_xor_sync(0xffffffffu, term, 2);
  term += __shfl_xor_sync(0xffffffffu, term, 1);
  const uint64_t h = mix64(gram_seed(slot, m) + term);
  const int32_t tag = gram_tag(h, m);
  const int64_t lo = look ? V.slot_text_off[slot] : 0, hi = look ? V.slot_text_off[slot + 1] : 0;
  const int64_t base = (int64_t)(h & (uint64_t)V.table_mask);
  auto group_or = [&](unsigned v) {
    v |= __shfl_xor_sync(0xffffffffu, v, 1);
    v |= __shfl_xor_sync(0xffffffffu, v, 2);
    return v;
  };
  // one table row: probe-ordered 8-bit masks of empty slots and live candidates (before the first empty)
  auto probe_row = [&](int64_t b, bool active, HsGramEntry& e0, HsGramEntry& e1, unsigned& em, unsigned& cm) {
    e0.pos = e1.pos = -1;
    e0.tag = e1.tag = 0;
    if (active) {
      e0 = V.table[(b + 2 * j) & V.table_mask];
      e1 = V.table[(b + 2 * j + 1) & V.table_mask];
    }
    const bool c0 = e0.pos >= 0 && e0.tag == tag && e0.pos >= lo && e0.pos < hi;
    const bool c1 = e1.pos >= 0 && e1.tag == tag && e1.pos >= lo && e1.pos < hi;
    em = group_or(((e0.pos < 0) ? 1u : 0u) << (2 * j) | ((e1.pos < 0) ? 2u : 0u) << (2 * j));
    cm = group_or((c0 ? 1u : 0u) << (2 * j) | (c1 ? 2u : 0u) << (2 * j));
    if (!active) {
      em = 1u;
      cm = 0u;
    }
    cm &= em ? ((1u << (__ffs(em) - 1)) - 1u) : 0xFFu;
  };
  auto cand_pos = [&](unsigned cm, const HsGramEntry& e0, const HsGramEntry& e1) {
    const int c = cm ? __ffs(cm) - 1 : 0;
    const int src = (g << 2) + (c >> 1);
    const int32_t p0 = __shfl_sync(0xffffffffu, e0.pos, src), p1 = __shfl_sync(0xffffffffu, e1.pos, src);
    return (c & 1) ? p1 : p0;
  };
  auto mismatch = [&](bool active, int32_t cp) {
    bool bad = false;
    if (active) {
      const int32_t va = j < m ? V.text[cp + j] : 0, vb = j + 4 < m ? V.text[cp + j + 4] : 0;
      bad = (j < m && va != pre_a) || (j + 4 < m && vb != pre_b);
    }
    return group_or(bad ? 1u : 0u) != 0u;
  };
  int32_t hit_pos = -1;
  int32_t t8[8];   // draft tokens text[hit_pos + m + j + 4k]
  bool have = false;
  // first row, fused: the first live candidate's verify and draft tokens in one round trip
  HsGramEntry e0, e1;
  unsigned em, cm;
  probe_row(base, look, e0, e1, em, cm);
  bool done = !look;
  {
    const int32_t cp = cand_pos(cm, e0, e1);
    bool bad = false;
    int32_t va = 0, vb = 0;
    if (cm) {
      va = j < m ? V.text[cp + j] : 0;
      vb = j + 4 < m ? V.text[cp + j + 4] : 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t8[k] = j + 4 * k < win ? V.text[cp + m + j + 4 * k] : 0;
      bad = (j < m && va != pre_a) || (j + 4 < m && vb != pre_b);
    }
    const bool anybad = group_or(bad ? 1u : 0u) != 0u;
    if (cm && !anybad) {
      hit_pos = cp;
      have = true;
      done = true;
    } else if (!cm && em) {
      done = true;   // an empty slot before any candidate: the key is absent
    }
  }
  // undecided groups: probe rows from the start, candidates in probe order
  for (int64_t b = base; __any_sync(0xffffffffu, !done); b += 8) {
    probe_row(b, !done, e0, e1, em, cm);
    while (__any_sync(0xffffffffu, cm != 0u)) {
      const int32_t cp = cand_pos(cm, e0, e1);
      const bool bad = mismatch(cm != 0u, cp);
      if (cm) {
        if (!bad) {
          hit_pos = cp;
          cm = 0u;
          em = 1u;   // resolved
        } else {
          cm &= cm - 1u;
        }
      }
    }
    if (!done && (hit_pos >= 0 || em)) done = true;
  }
  const bool hit = hit_pos >= 0;
  if (hit && !have) {
#pragma unroll
    for (int k = 0; k < 8; ++k) t8[k] = j + 4 * k < win ? V.text[hit_pos + m + j + 4 * k] : 0;
  }
  int32_t first_term = 32;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int idx = j + 4 * k;
    if (hit && idx < win && t8[k] < 0 && idx < first_term) first_term = idx;
  }
  first_term = min(first_term, __shfl_xor_sync(0xffffffffu, first_term, 1));
  first_term = min(first_term, __shfl_xor_sync(0xffffffffu, first_term, 2));
  const int32_t len = hit ? min(first_term, win) : 0;
  if (valid) {
    int32_t* out = draft_tok + s * (int64_t)draft_stride;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = j + 4 * k;
      if (idx < len) out[idx] = t8[k];
    }
    if (j == 0) {
      draft_len[s] = len;
      looked[s] = valid && speculate[s] && slot >= 0 && pos >= m;
      found[s] = hit;
    }
  }
}

// ---------------------------------------------------------------------------
// Token-similarity replay (tracegen.py:306-353 token_similarity_replay).
//
// The reference indexes every prefix_len-gram of the previous epoch's
// responses and, at each position, scans all occurrences of the last p
// tokens for the longest identical continuation.  That maximum equals
// (longest prefix of Q = tokens[pos-p : len] occurring in the prompt's
// history) - p, when that prefix reaches length p.  The suffix with the
// longest common prefix with Q is adjacent to Q's insertion point in the
// slot's suffix array, so one warp binary search per step replaces the scan.
// The terminal (-1) ends every history response and sorts below all tokens;
// the end of Q sorts below the terminal.

// LCP of suffix text[p:] with q[0:qn] and the three-way order (suffix vs q); the first k0
// tokens are known to be equal.  Four 32-token chunks are loaded per round so a long match
// costs a quarter of the dependent round trips; text reads are clamped to the padded text.
template <int U>
__device__ __forceinline__ int32_t lcp_query(const int32_t* __restrict__ text, int64_t text_end, int32_t p,
                                             const int32_t* __restrict__ q, int32_t qn, int32_t k0, int* order) {
  const int lane = lane_id();
  for (int32_t c = k0;; c += 32 * U) {
    int32_t a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t j = c + 32 * u + lane;
      a[u] = text[min((int64_t)p + j, text_end)];
      b[u] = j < qn ? q[j] : -2;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // the first flagged lane lies at or before the suffix's terminal, so clamped reads never decide
      unsigned d = __ballot_sync(0xffffffffu, a[u] != b[u] || a[u] < 0);
      if (d) {
        int src = __ffs(d) - 1;
        int32_t x = __shfl_sync(0xffffffffu, a[u], src);
        int32_t y = __shfl_sync(0xffffffffu, b[u], src);
        *order = x < y ? -1 : 1;    // never equal: a terminal (-1) meets q's end only as -2
        return c + 32 * u + src;
      }
    }
  }
}

// LCP-array bound (LCPB): when one bracket shares more with q than the other, the LCP array
// decides a probe without touching the text whenever the range to that bracket is short:
// x = LCP(bracket, probe) = min lcp[] over the range; x > l -> same side as the bracket with LCP l,
// x < l -> the other side with LCP x, x == l -> compare from l.
constexpr int64_t kSimLcpScan = 256;

template <int U, bool PREFETCH, bool LCPB = false>
__global__ void k_similarity_replay(HsIndexView V, int32_t n_resp, const int32_t* __restrict__ tok,
                                    const int64_t* __restrict__ off, const int32_t* __restrict__ slot_of,
                                    int32_t p, int64_t* __restrict__ accepted) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_resp) return;
  const int lane = lane_id();
  const int32_t* t = tok + off[r];
  const int32_t len = (int32_t)(off[r + 1] - off[r]);
  const int32_t slot = slot_of[r];
  if (slot < 0 || slot >= V.n_slots) {   // -1 = no history for this prompt (the C-ABI's convention)
    if (lane_id() == 0) accepted[r] = 0;
    return;
  }
  const int64_t S = V.slot_sa_off[slot], E = V.slot_sa_off[slot + 1];
  const int64_t text_end = V.n_text + HS_TEXT_PAD - 1;
  int64_t acc = 0;
  if (S < E) {
    for (int32_t pos = p; pos < len;) {
      const int32_t* q = t + pos - p;
      const int32_t qn = len - pos + p;
      int64_t lo = S, hi = E;
      int32_t l_lo = 0, l_hi = 0;   // LCP with the last suffix found below / above q
      int64_t mid = (lo + hi) >> 1;
      int32_t sp = V.sa[mid];
      while (lo < hi) {
        // prefetch both possible next probes (lane 0: left half, lane 1: right half) so the SA
        // load leaves the dependent chain; one text round trip per probe remains
        const int64_t mid_l = (lo + mid) >> 1, mid_r = (mid + 1 + hi) >> 1;
        const int64_t nxt = lane == 0 ? mid_l : mid_r;
        const int32_t sp_n = (PREFETCH && lane < 2 && nxt < E) ? V.sa[nxt] : 0;
        int order = 0;
        // every suffix between the two bracketing probes shares min(l_lo, l_hi) tokens with q
        int32_t k0 = min(l_lo, l_hi), l = -1;
        if (LCPB && l_lo != l_hi) {
          const bool low = l_lo > l_hi;
          const int64_t a = low ? lo : mid + 1, b = low ? mid : hi;   // lcp[a..b] spans bracket..probe
          if ((low ? lo > S : hi < E) && b - a < kSimLcpScan) {
            int32_t x = 0x7fffffff;
            for (int64_t k = a + lane; k <= b; k += 32) x = min(x, V.lcp[k]);
            x = __reduce_min_sync(0xffffffffu, x);
            const int32_t lb = low ? l_lo : l_hi;
            if (x > lb) { order = low ? -1 : 1; l = lb; }
            else if (x < lb) { order = low ? 1 : -1; l = x; }
            else k0 = lb;
          }
        }
        if (l < 0) l = lcp_query<U>(V.text, text_end, sp, q, qn, k0, &order);
        int32_t sp_l = __shfl_sync(0xffffffffu, sp_n, 0), sp_r = __shfl_sync(0xffffffffu, sp_n, 1);
        if (!PREFETCH) {
          const int64_t m2 = order < 0 ? mid_r : mid_l;   // only the taken side, after the compare
          sp_l = sp_r = m2 < E ? V.sa[m2] : 0;
        }
        if (order < 0) { lo = mid + 1; l_lo = l; mid = mid_r; sp = sp_r; }
        else { hi = mid; l_hi = l; mid = mid_l; sp = sp_l; }
      }
      // the last probes on either side are the insertion point's neighbours sa[lo - 1] and sa[lo]
      // (lo only moves to mid + 1, hi only to mid); a side never probed has no neighbour
      const int32_t best = max(l_lo, l_hi);
      int32_t run = best - p;
      if (run > 0) { acc += run; pos += run; } else { pos += 1; }
    }
  }
  if (lane == 0) accepted[r] = acc;
}


// Inverse suffix array: isa[sa[k]] = k (terminal positions stay -1).
__global__ void k_inverse_sa(const int32_t* __restrict__ sa, int64_t n_suffix, int32_t* __restrict__ isa) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_suffix; k += (int64_t)gridDim.x * blockDim.x)
    isa[sa[k]] = (int32_t)k;
}

// ISA-seeded variant: after a run of `run` tokens matched by suffix h, suffix h + run shares the
// next query's first p tokens, so its rank (isa) seeds the next search.  A gallop from that rank
// brackets the insertion point within the p-gram's SA interval; a binary search finishes it.
// A miss (run 0) with a best match of l >= 1 tokens seeds the next search the same way with
// h + 1 (sharing l - 1 tokens); only a miss with no shared token pays a full search.
__global__ void k_similarity_replay_isa(HsIndexView V, const int32_t* __restrict__ isa, int32_t n_resp,
                                        const int32_t* __restrict__ tok, const int64_t* __restrict__ off,
                                        const int32_t* __restrict__ slot_of, int32_t p,
                                        int64_t* __restrict__ accepted) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_resp) return;
  const int lane = lane_id();
  const int32_t* t = tok + off[r];
  const int32_t len = (int32_t)(off[r + 1] - off[r]);
  const int32_t slot = slot_of[r];
  if (slot < 0 || slot >= V.n_slots) {   // -1 = no history for this prompt (the C-ABI's convention)
    if (lane_id() == 0) accepted[r] = 0;
    return;
  }
  const int64_t S = V.slot_sa_off[slot], E = V.slot_sa_off[slot + 1];
  const int64_t text_end = V.n_text + HS_TEXT_PAD - 1;
  int64_t acc = 0;
  if (S < E) {
    int64_t hint = -1;   // SA index of a suffix sharing >= hk tokens with the query, or -1
    int32_t hk = 0;
    for (int32_t pos = p; pos < len;) {
      const int32_t* q = t + pos - p;
      const int32_t qn = len - pos + p;
      int64_t lo = S, hi = E;
      int32_t l_lo = 0, l_hi = 0, sp_lo = -1, sp_hi = -1;   // bracketing probes: LCP and text position
      int order;
      if (hint >= 0) {
        const int32_t sp0 = V.sa[hint];
        const int32_t l0 = lcp_query<1>(V.text, text_end, sp0, q, qn, hk, &order);
        if (order < 0) {
          lo = hint + 1; l_lo = l0; sp_lo = sp0;
          for (int64_t step = 1;; step <<= 1) {
            const int64_t k = hint + step;
            if (k >= E) break;
            const int32_t sp = V.sa[k];
            const int32_t l = lcp_query<1>(V.text, text_end, sp, q, qn, 0, &order);
            if (order < 0) { lo = k + 1; l_lo = l; sp_lo = sp; }
            else { hi = k; l_hi = l; sp_hi = sp; break; }
          }
        } else {
          hi = hint; l_hi = l0; sp_hi = sp0;
          for (int64_t step = 1;; step <<= 1) {
            const int64_t k = hint - step;
            if (k < S) break;
            const int32_t sp = V.sa[k];
            const int32_t l = lcp_query<1>(V.text, text_end, sp, q, qn, 0, &order);
            if (order < 0) { lo = k + 1; l_lo = l; sp_lo = sp; break; }
            else { hi = k; l_hi = l; sp_hi = sp; }
          }
        }
      }
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int32_t sp = V.sa[mid];
        const int32_t l = lcp_query<1>(V.text, text_end, sp, q, qn, min(l_lo, l_hi), &order);
        if (order < 0) { lo = mid + 1; l_lo = l; sp_lo = sp; } else { hi = mid; l_hi = l; sp_hi = sp; }
      }
      const int32_t best = max(l_lo, l_hi);
      const int32_t run = best - p;
      // the next query is this one advanced by a tokens; the best suffix advanced by a shares
      // best - a of them (any seed is correct -- the gallop only gets shorter with a good one)
      const int32_t a = run > 0 ? run : 1;
      const int32_t bsp = l_lo >= l_hi ? sp_lo : sp_hi;
      if (run > 0) acc += run;
      pos += a;
      if (best >= a && bsp >= 0) { hint = isa[bsp + a]; hk = best - a; }   // -1 at a terminal
      else { hint = -1; hk = 0; }
    }
  }
  if (lane == 0) accepted[r] = acc;
}

}  // namespace hs

using namespace hs;

// Candidate branches of a draft tree (north_star (1): frequency-weighted candidate branches): the children of
// the node the prefix matches, ranked by reward mass (ties to the smaller token -- the order extract_draft
// picks its first token in, history.py:322-331), each followed by its own greedy (heavy) continuation.
// Branch 0 is exactly the reference draft; branches 1..W-1 are the runner-up first tokens.  A prefix that
// ends inside an edge (one continuation) or in a leaf has one branch.  One warp per query:
//   [first, last) = the prefix's SA interval (binary search); locus depth < m... == m -> at a node: child
//   boundaries are the k in (first, last) with lcp[k] == m; a child's mass is a wsum difference, its token
//   text[sa[a] + m] (a terminal child is not a token child); its heavy end is heavy[] at the child's own
//   first minimum-LCP boundary (or its only suffix).
__global__ void k_lookup_branches(HsIndexView V, int32_t n, const int32_t* __restrict__ slot,
                                  const int32_t* __restrict__ prefix, int32_t prefix_stride,
                                  const int32_t* __restrict__ prefix_len, const int32_t* __restrict__ window,
                                  int32_t width, int32_t* __restrict__ out_tok, int32_t out_stride,
                                  int32_t* __restrict__ out_len, int64_t* __restrict__ out_mass) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const int lane = lane_id();
  const int32_t s = slot[w], m = prefix_len[w], win = window[w];
  const int32_t* pre = prefix + (int64_t)w * prefix_stride;
  int32_t* lens = out_len + (int64_t)w * width;
  int64_t* masses = out_mass + (int64_t)w * width;
  for (int b = lane; b < width; b += 32) { lens[b] = 0; masses[b] = 0; }
  __syncwarp();
  if (s < 0 || s >= V.n_slots || m < 1 || win < 1) return;
  const int64_t S = V.slot_sa_off[s], E = V.slot_sa_off[s + 1];
  int64_t lo = S, hi = E;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cmp_suffix(V.text, V.sa[mid], pre, m) < 0) lo = mid + 1; else hi = mid;
  }
  const int64_t first = lo;
  hi = E;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cmp_suffix(V.text, V.sa[mid], pre, m) <= 0) lo = mid + 1; else hi = mid;
  }
  const int64_t last = lo;
  if (first == last) return;
  // minimum LCP (first position) inside a range: the node owning [a, b)
  auto min_lcp = [&](int64_t a, int64_t b, int32_t& best, int64_t& bidx) {
    best = 0x7fffffff;
    bidx = -1;
    for (int64_t k = a + 1 + lane; k < b; k += 32) {
      const int32_t v = V.lcp[k];
      if (v < best) { best = v; bidx = k; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int32_t ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov < best || (ov == best && oi >= 0 && (bidx < 0 || oi < bidx))) { best = ov; bidx = oi; }
    }
  };
  // top-W children (mass desc, token asc), kept identically in every lane
  constexpr int WMAX = 8;
  int64_t tm[WMAX];
  int32_t tt[WMAX];
  int64_t ta[WMAX], tb[WMAX];
  int cnt = 0;
  auto offer = [&](int64_t mass, int32_t tok, int64_t a, int64_t b) {
    int pos = cnt;
    while (pos > 0 && (mass > tm[pos - 1] || (mass == tm[pos - 1] && tok < tt[pos - 1]))) --pos;
    if (pos >= width) return;
    const int end = cnt < width ? cnt : width - 1;
    for (int j = end; j > pos; --j) { tm[j] = tm[j - 1]; tt[j] = tt[j - 1]; ta[j] = ta[j - 1]; tb[j] = tb[j - 1]; }
    tm[pos] = mass; tt[pos] = tok; ta[pos] = a; tb[pos] = b;
    if (cnt < width) ++cnt;
  };
  int32_t depth = m + 1;
  int64_t node_k = -1;
  if (last - first > 1) min_lcp(first, last, depth, node_k);
  if (last - first == 1 || depth > m) {
    // a leaf or inside an edge: the single continuation (the reference draft)
    const int32_t p = last - first == 1 ? V.sa[first] : V.heavy[node_k];
    const int32_t t = V.text[p + m];
    if (t >= 0) offer(V.wsum[last] - V.wsum[first], t, first, last);
  } else {
    // at a node: walk the child boundaries (lcp == m) in SA order
    int64_t a = first;
    for (int64_t base = first + 1; base <= last; base += 32) {
      const int64_t k = base + lane;
      const bool bnd = k < last && V.lcp[k] == m;
      unsigned bal = __ballot_sync(0xffffffffu, bnd);
      if (base + 31 >= last) bal |= 1u << (int)(last - base < 31 ? last - base : 31);   // the interval end
      while (bal) {
        const int j = __ffs(bal) - 1;
        bal &= bal - 1;
        const int64_t b = base + j;
        if (b > last) break;
        const int32_t t = V.text[V.sa[a] + m];
        if (t >= 0) offer(V.wsum[b] - V.wsum[a], t, a, b);
        a = b;
        if (b == last) break;
      }
    }
  }
  // branches: each winner's heavy continuation
  for (int c = 0; c < cnt; ++c) {
    int32_t p;
    if (tb[c] - ta[c] == 1) {
      p = V.sa[ta[c]];
    } else {
      int32_t d2;
      int64_t k2;
      min_lcp(ta[c], tb[c], d2, k2);
      p = V.heavy[k2];
    }
    const int32_t len = read_draft(V.text, p + m, win, out_tok + ((int64_t)w * width + c) * out_stride);
    if (lane == 0) {
      lens[c] = len;
      masses[c] = tm[c];
    }
  }
}

extern "C" int hs_lookup_branches(const HsIndexView* view, int32_t n, const int32_t* d_slot, const int32_t* d_prefix,
                                  int32_t prefix_stride, const int32_t* d_prefix_len, const int32_t* d_window,
                                  int32_t width, int32_t* d_out_tok, int32_t out_stride, int32_t* d_out_len,
                                  int64_t* d_out_mass, hs_stream_t stream) {
  if (n < 0 || width < 1 || width > 8 || out_stride < 1) {
    hs_set_error("hs_lookup_branches: n >= 0, 1 <= width <= 8, out_stride >= 1");
    return HS_ERR_INVALID;
  }
  if (n == 0) return HS_OK;
  hs_count_launches(1);
  const int threads = 256;
  const int64_t blocks = ((int64_t)n * 32 + threads - 1) / threads;
  k_lookup_branches<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(*view, n, d_slot, d_prefix, prefix_stride,
                                                                          d_prefix_len, d_window, width, d_out_tok,
                                                                          out_stride, d_out_len, d_out_mass);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_lookup_batch(const HsIndexView* view, int32_t n, const int32_t* d_slot, const int32_t* d_prefix,
                               int32_t prefix_stride, const int32_t* d_prefix_len, const int32_t* d_window,
                               int32_t* d_out_tok, int32_t out_stride, int64_t* d_out_info, int32_t use_table,
                               hs_stream_t stream) {
  if (n <= 0) return HS_OK;
  if (view->n_suffix == 0) {
    HS_CUDA_TRY(cudaMemsetAsync(d_out_info, 0, sizeof(int64_t) * 6 * n, (cudaStream_t)stream));
    return HS_OK;
  }
  int threads = 256;
  int64_t blocks = ((int64_t)n * 32 + threads - 1) / threads;
  hs_count_launches(1);
  k_lookup_batch<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(*view, n, d_slot, d_prefix, prefix_stride,
                                                                       d_prefix_len, d_window, d_out_tok, out_stride,
                                                                       d_out_info, use_table);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_draft(const HsIndexView* view, int32_t n_seq, const int32_t* d_slot_of_seq, const int32_t* d_gen_tok,
                        int32_t gen_stride, const int32_t* d_gen_len, const int32_t* d_prefix_len,
                        const int32_t* d_window, const uint8_t* d_speculate, int32_t prefix_lo, int32_t prefix_hi,
                        int32_t window_hi, int32_t* d_draft_tok, int32_t draft_stride, int32_t* d_draft_len,
                        uint8_t* d_looked, uint8_t* d_found, hs_stream_t stream) {
  if (n_seq <= 0) return HS_OK;
  if (draft_stride < 1) { hs_set_error("draft_stride"); return HS_ERR_INVALID; }
  int threads = 256;
  HsIndexView V = *view;
  if (V.n_suffix == 0) {
    // empty history: every lookup misses
    V.table = nullptr;
  }
  // every prefix length the caller can produce is tabled and <= 8, windows <= 32: 8-lane groups
  if (V.table && prefix_lo >= V.prefix_min && prefix_hi <= V.prefix_max && prefix_hi <= 8 && window_hi <= 32 &&
      draft_stride >= window_hi) {
    hs_count_launches(1);
    static const bool lanes8 = getenv("HS_K2_DRAFT8") != nullptr;     // A/B switches for profiling only
    static const bool unfused = getenv("HS_K2_UNFUSED") != nullptr;
    if (!lanes8) {
      const int64_t warps4 = ((int64_t)n_seq + 7) / 8;
      k_draft4<<<(unsigned)((warps4 * 32 + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
          V, n_seq, d_slot_of_seq, d_gen_tok, gen_stride, d_gen_len, d_prefix_len, d_window, d_speculate,
          d_draft_tok, draft_stride, d_draft_len, d_looked, d_found);
      HS_CUDA_TRY(cudaGetLastError());
      return HS_OK;
    }
    int64_t warps = ((int64_t)n_seq + 3) / 4;
    int64_t blocks8 = (warps * 32 + threads - 1) / threads;
    auto kern = unfused ? k_draft8<false> : k_draft8<true>;
    kern<<<(unsigned)blocks8, threads, 0, (cudaStream_t)stream>>>(V, n_seq, d_slot_of_seq, d_gen_tok, gen_stride,
                                                                  d_gen_len, d_prefix_len, d_window, d_speculate,
                                                                  d_draft_tok, draft_stride, d_draft_len, d_looked,
                                                                  d_found);
    HS_CUDA_TRY(cudaGetLastError());
    return HS_OK;
  }
  int64_t blocks = ((int64_t)n_seq * 32 + threads - 1) / threads;
  hs_count_launches(1);
  k_draft<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(V, n_seq, d_slot_of_seq, d_gen_tok, gen_stride,
                                                                 d_gen_len, d_prefix_len, d_window, d_speculate,
                                                                 d_draft_tok, draft_stride, d_draft_len, d_looked,
                                                                 d_found);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_similarity_replay(const HsIndexView* view, int32_t n_resp, const int32_t* d_tokens,
                                    const int64_t* d_resp_off, const int32_t* d_slot_of_resp, int32_t prefix_len,
                                    int64_t* d_accepted, hs_stream_t stream) {
  if (prefix_len < 1) { hs_set_error("prefix_len must be >= 1"); return HS_ERR_INVALID; }
  if (n_resp <= 0) return HS_OK;
  const int threads = 256;
  const int64_t blocks = ((int64_t)n_resp * 32 + threads - 1) / threads;
  // A/B switch for profiling only: HS_SIM_VARIANT = u1 (default) | u2 | u4 | u1np (no SA prefetch) | lcp (LCP-array bound)
  static const char* var_env = getenv("HS_SIM_VARIANT");
  const std::string var = var_env ? var_env : "u1";
  auto kern = k_similarity_replay<1, true>;
  if (var == "u2") kern = k_similarity_replay<2, true>;
  else if (var == "u4") kern = k_similarity_replay<4, true>;
  else if (var == "u1np") kern = k_similarity_replay<1, false>;
  else if (var == "lcp") kern = k_similarity_replay<1, true, true>;
  hs_count_launches(1);
  kern<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(*view, n_resp, d_tokens, d_resp_off, d_slot_of_resp,
                                                               prefix_len, d_accepted);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_index_inverse_sa(const HsIndexView* view, int32_t* d_isa, hs_stream_t stream) {
  HS_CUDA_TRY(cudaMemsetAsync(d_isa, 0xff, sizeof(int32_t) * (size_t)(view->n_text > 0 ? view->n_text : 1),
                              (cudaStream_t)stream));
  if (view->n_suffix <= 0) return HS_OK;
  hs_count_launches(1);
  k_inverse_sa<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(view->sa, view->n_suffix, d_isa);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}

extern "C" int hs_similarity_replay_isa(const HsIndexView* view, const int32_t* d_isa, int32_t n_resp,
                                        const int32_t* d_tokens, const int64_t* d_resp_off,
                                        const int32_t* d_slot_of_resp, int32_t prefix_len, int64_t* d_accepted,
                                        hs_stream_t stream) {
  if (prefix_len < 1) { hs_set_error("prefix_len must be >= 1"); return HS_ERR_INVALID; }
  if (n_resp <= 0) return HS_OK;
  const int threads = 256;
  const int64_t blocks = ((int64_t)n_resp * 32 + threads - 1) / threads;
  hs_count_launches(1);
  k_similarity_replay_isa<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      *view, d_isa, n_resp, d_tokens, d_resp_off, d_slot_of_resp, prefix_len, d_accepted);
  HS_CUDA_TRY(cudaGetLastError());
  return HS_OK;
}
