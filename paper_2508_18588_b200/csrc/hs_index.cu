// K1: GPU-resident history index (suffix array + LCP-interval tree + heavy
// continuations + n-gram hash table).  Replaces the per-prompt Ukkonen suffix
// tree of rhymesim/history.py:148-279 (add_response / finalize) and
// build_tree :343-355.
//
// Semantics kept exactly:
//  * every response is followed by a shared TERMINAL (history.py:23-28) that
//    sorts below every token (-1 here), so identical suffixes of different
//    responses compare equal and share a logical leaf;
//  * the priority of a tree position is the reward mass of the suffixes below
//    it (leaf credit :183/:214/:254-263, interior sums :265-279) -- here the
//    difference of an exclusive prefix sum over the SA (int64 fixed point, so
//    sums are exact and order independent);
//  * greedy drafting takes the max-priority token child with ties to the
//    smallest token (:322-331).  The full greedy path from a tree position
//    ends at a leaf, i.e. spells one response suffix; we precompute that
//    "heavy" suffix start for every node by best-child pointer jumping, so a
//    draft of any window is just text[heavy + m : ...] up to the terminal.
//
// Pipeline (all slots of a batch at once, slot-major):
//   layout -> prefix-doubling suffix sort (CUB radix sort per round) ->
//   LCP by rank-level descent -> sparse table (min) -> LCP-interval nodes,
//   parents, child candidates -> best child (3 atomic passes) -> pointer
//   jumping -> heavy text positions -> per-slot stats -> n-gram groups.
#include <cub/cub.cuh>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "hs_common.cuh"

namespace hs {

// ---------------------------------------------------------------- layout
__global__ void k_layout(const int32_t* __restrict__ tok, const int64_t* __restrict__ resp_off,
                         const int32_t* __restrict__ resp_slot, int32_t n_resp,
                         int32_t* __restrict__ text, int32_t* __restrict__ rid,
                         int32_t* __restrict__ rem, int32_t* __restrict__ sufpos,
                         uint64_t* __restrict__ key0) {
  int r = blockIdx.x;
  if (r >= n_resp) return;
  int64_t a = resp_off[r], b = resp_off[r + 1];
  int64_t base = a + r;  // text position of token a
  int32_t len = (int32_t)(b - a);
  uint64_t slot_hi = (uint64_t)(uint32_t)resp_slot[r] << 32;
  for (int32_t j = threadIdx.x; j <= len; j += blockDim.x) {
    int64_t p = base + j;
    rid[p] = r;
    if (j < len) {
      int32_t t = tok[a + j];
      text[p] = t;
      rem[p] = len - j;
      sufpos[a + j] = (int32_t)p;
      key0[a + j] = slot_hi | (uint64_t)(uint32_t)(t + 1);
    } else {
      text[p] = -1;
      rem[p] = 0;
    }
  }
}

// rank of sorted element k = 1 + first index of its key group
__global__ void k_group_head(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ head) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  head[k] = (k == 0 || keys[k] != keys[k - 1]) ? (int32_t)k : 0;
}

__global__ void k_scatter_rank(const int32_t* __restrict__ sa, const int32_t* __restrict__ gstart,
                               int64_t n, int32_t* __restrict__ rank) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  rank[sa[k]] = gstart[k] + 1;
}

// Prefix doubling has converged after a round with window w when no group of equal w-windows can still
// split: every suffix that is not its group's head (so it ties with its predecessor) already has the
// terminal inside its window (rem < w) -- tied windows that end at a terminal stay tied forever.
__global__ void k_converged(const int32_t* __restrict__ sa, const int32_t* __restrict__ gstart,
                            const int32_t* __restrict__ rem, int64_t n, int64_t w, unsigned long long* flag) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (gstart[k] != (int32_t)k && rem[sa[k]] >= w) *flag = 1ull;
}

__global__ void k_double_keys(const int32_t* __restrict__ sufpos, const int32_t* __restrict__ rank,
                              const int32_t* __restrict__ rem, int64_t n, int32_t h, int32_t bits,
                              uint64_t* __restrict__ keys) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t p = sufpos[i];
  uint32_t hi = (uint32_t)rank[p];
  uint32_t lo = rem[p] > h ? (uint32_t)rank[p + h] : 0u;
  keys[i] = ((uint64_t)hi << bits) | lo;
}

// ---------------------------------------------------------------- LCP
__global__ void k_lcp(const int32_t* __restrict__ sa, const int32_t* __restrict__ rem,
                      const int32_t* __restrict__ rid, const int32_t* __restrict__ resp_slot,
                      const int32_t* const* __restrict__ ranks, int32_t n_rounds, int64_t n,
                      int32_t* __restrict__ lcp) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > n) return;
  if (k == n || k == 0) { lcp[k] = -1; return; }
  int32_t a = sa[k - 1], b = sa[k];
  if (resp_slot[rid[a]] != resp_slot[rid[b]]) { lcp[k] = -1; return; }
  // ranks[j] identifies the 2^j-token prefix (terminal-truncated) of a suffix
  int32_t l = 0;
  for (int32_t j = n_rounds; j >= 0; --j) {
    int32_t ra = rem[a + l], rb = rem[b + l];
    if (ra == 0 || rb == 0) break;
    if (ranks[j][a + l] == ranks[j][b + l]) {
      int32_t step = 1 << j;
      l += ra < step ? ra : step;  // equal windows that include the terminal end together
    }
  }
  lcp[k] = l;
}

__global__ void k_weights(const int32_t* __restrict__ sa, const int32_t* __restrict__ rid,
                          const int64_t* __restrict__ reward_fx, int64_t n, int64_t* __restrict__ w) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > n) return;
  w[k] = k < n ? reward_fx[rid[sa[k]]] : 0;
}

__global__ void k_sparse_level(const int32_t* __restrict__ prev, int64_t n1, int64_t half,
                               int32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n1) return;
  int64_t j = i + half;
  int32_t a = prev[i];
  int32_t b = j < n1 ? prev[j] : -1;
  out[i] = a < b ? a : b;
}

// ---------------------------------------------------------------- sparse-table walks
struct Sparse {
  const int32_t* const* lv;  // lv[j][i] = min(lcp[i .. i+2^j-1]) (clamped, lcp[n] = -1)
  int32_t levels;
  int64_t n1;                // n + 1
};

// largest j < k with lcp[j] < v
__device__ __forceinline__ int64_t psv(const Sparse& S, int64_t k, int32_t v) {
  int64_t j = k;
  for (int32_t l = S.levels - 1; l >= 0; --l) {
    int64_t step = (int64_t)1 << l;
    if (j - step >= 0 && S.lv[l][j - step] >= v) j -= step;
  }
  return j - 1;
}
// smallest j >= s with lcp[j] < v
__device__ __forceinline__ int64_t first_lt(const Sparse& S, int64_t s, int32_t v) {
  int64_t j = s;
  for (int32_t l = S.levels - 1; l >= 0; --l) {
    if (j < S.n1 && S.lv[l][j] >= v) j += (int64_t)1 << l;
  }
  return j;
}
// smallest j >= s with lcp[j] <= v
__device__ __forceinline__ int64_t first_le(const Sparse& S, int64_t s, int32_t v) {
  int64_t j = s;
  for (int32_t l = S.levels - 1; l >= 0; --l) {
    if (j < S.n1 && S.lv[l][j] > v) j += (int64_t)1 << l;
  }
  return j;
}
__device__ __forceinline__ int32_t rmq(const Sparse& S, int64_t a, int64_t b) {
  int64_t len = b - a + 1;
  int32_t l = 63 - __clzll(len);
  int32_t x = S.lv[l][a], y = S.lv[l][b - ((int64_t)1 << l) + 1];
  return x < y ? x : y;
}
// canonical node id of the LCP-interval that owns boundary j (lcp[j] = u > 0)
__device__ __forceinline__ int64_t node_of(const Sparse& S, const int32_t* lcp, int64_t j) {
  int32_t u = lcp[j];
  return first_le(S, psv(S, j, u) + 1, u);
}

struct SlotMap {
  const int32_t* rid;
  const int32_t* resp_slot;
  const int64_t* slot_sa_off;
  __device__ __forceinline__ int64_t root_of_text(int32_t p) const { return slot_sa_off[resp_slot[rid[p]]]; }
};

// Per SA index k: (a) the node whose canonical boundary is k, (b) leaf k.
// Emits up to two child candidates (parent, mass, first token, child id).
__global__ void k_nodes(Sparse S, const int32_t* __restrict__ lcp, const int32_t* __restrict__ sa,
                        const int32_t* __restrict__ rem, const int32_t* __restrict__ text,
                        const int64_t* __restrict__ wsum, SlotMap M, int64_t n,
                        int32_t* __restrict__ node_lb, uint8_t* __restrict__ node_flags,
                        int64_t* __restrict__ cand_parent, int64_t* __restrict__ cand_mass,
                        int32_t* __restrict__ cand_tok) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  // (a) internal node at canonical boundary k
  int64_t c0 = 2 * k, c1 = 2 * k + 1;
  cand_parent[c0] = -1;
  cand_parent[c1] = -1;
  int32_t v = lcp[k];
  if (v > 0) {
    int64_t lb = psv(S, k, v);
    if (first_le(S, lb + 1, v) == k) {
      int64_t rb = first_lt(S, k + 1, v) - 1;
      node_lb[k] = (int32_t)lb;
      node_flags[k] = 1;
      int32_t l_lo = lcp[lb], l_hi = lcp[rb + 1];
      int32_t pv = l_lo > l_hi ? l_lo : l_hi;
      int64_t parent;
      if (pv <= 0) parent = M.root_of_text(sa[lb]);
      else parent = node_of(S, lcp, l_lo >= l_hi ? lb : rb + 1);
      int32_t pd = pv > 0 ? pv : 0;
      cand_parent[c0] = parent;
      cand_mass[c0] = wsum[rb + 1] - wsum[lb];
      cand_tok[c0] = text[sa[lb] + pd];
    }
  } else if (v < 0) {
    // slot start: this index is the root id of its slot
    node_lb[k] = (int32_t)k;
    node_flags[k] = 1;
  }
  // (b) leaf k
  int32_t l_lo = lcp[k], l_hi = lcp[k + 1];
  int32_t pv = l_lo > l_hi ? l_lo : l_hi;
  int32_t pd = pv > 0 ? pv : 0;
  int32_t p = sa[k];
  if (rem[p] > pd) {  // terminal children never compete (history.py:324-325)
    int64_t parent = pv <= 0 ? M.root_of_text(p) : node_of(S, lcp, l_lo >= l_hi ? k : k + 1);
    cand_parent[c1] = parent;
    cand_mass[c1] = wsum[k + 1] - wsum[k];
    cand_tok[c1] = text[p + pd];
  }
}

__global__ void k_best_mass(const int64_t* __restrict__ cp, const int64_t* __restrict__ cm, int64_t nc,
                            long long* __restrict__ best_mass) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc || cp[c] < 0) return;
  atomicMax(&best_mass[cp[c]], (long long)cm[c]);
}
__global__ void k_best_tok(const int64_t* __restrict__ cp, const int64_t* __restrict__ cm,
                           const int32_t* __restrict__ ct, int64_t nc,
                           const long long* __restrict__ best_mass, int32_t* __restrict__ best_tok) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc || cp[c] < 0) return;
  if ((long long)cm[c] == best_mass[cp[c]]) atomicMin(&best_tok[cp[c]], ct[c]);
}
// child id: node k -> k, leaf k -> n + k
__global__ void k_best_child(const int64_t* __restrict__ cp, const int64_t* __restrict__ cm,
                             const int32_t* __restrict__ ct, int64_t nc, int64_t n,
                             const long long* __restrict__ best_mass, const int32_t* __restrict__ best_tok,
                             int64_t* __restrict__ ptr, uint8_t* __restrict__ node_flags) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc || cp[c] < 0) return;
  int64_t par = cp[c];
  if ((long long)cm[c] == best_mass[par] && ct[c] == best_tok[par]) {
    int64_t k = c >> 1;
    ptr[par] = (c & 1) ? n + k : k;
    node_flags[par] |= 2;
  }
}

// nodes without a token child (identical suffixes only) point at a member leaf
__global__ void k_ptr_init(const uint8_t* __restrict__ node_flags, const int32_t* __restrict__ node_lb,
                           int64_t n, int64_t* __restrict__ ptr) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint8_t f = node_flags[k];
  if ((f & 1) && !(f & 2)) ptr[k] = n + node_lb[k];
  if (!(f & 1)) ptr[k] = -1;
}

__global__ void k_ptr_jump(int64_t* __restrict__ ptr, int64_t n) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int64_t p = ptr[k];
  if (p >= 0 && p < n) ptr[k] = ptr[p];
}

__global__ void k_heavy(const int64_t* __restrict__ ptr, const int32_t* __restrict__ sa, int64_t n,
                        int32_t* __restrict__ heavy) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int64_t p = ptr[k];
  heavy[k] = p >= n ? sa[p - n] : -1;
}

// Reference node count per slot (history.py:134-136 node_count): root +
// branching internal nodes + distinct suffixes (identical suffixes share a leaf).
__global__ void k_slot_stats(const int32_t* __restrict__ lcp, const int32_t* __restrict__ sa,
                             const int32_t* __restrict__ rem, const uint8_t* __restrict__ node_flags,
                             SlotMap M, int64_t n, unsigned long long* __restrict__ counts) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  int32_t slot = -1;
  if (k < n) {
    int32_t p = sa[k];
    slot = M.resp_slot[M.rid[p]];
    int32_t v = lcp[k];
    if (v < 0) c += 1;                                      // root
    else if (v > 0 && (node_flags[k] & 3) == 3) c += 1;     // branching node
    bool dup = v >= 0 && v == rem[p] && rem[sa[k - 1]] == v;
    if (!dup) c += 1;                                       // distinct suffix leaf
  }
  // consecutive SA indices share a slot: add per (warp, slot) run, one atomic per run
  const unsigned lane = threadIdx.x & 31;
  const unsigned same = __match_any_sync(0xffffffffu, slot);
  const int leader = __ffs(same) - 1;
  unsigned long long tot = c;
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_down_sync(0xffffffffu, tot, o);
    // only add lanes of the same run (runs are contiguous in lane order)
    if (lane + o < 32 && ((same >> (lane + o)) & 1)) tot += y;
  }
  if ((int)lane == leader && slot >= 0) atomicAdd(&counts[slot], tot);
}

__global__ void k_count_groups(const int32_t* __restrict__ lcp, const int32_t* __restrict__ sa,
                               const int32_t* __restrict__ rem, int64_t n, int32_t mmin, int32_t mmax,
                               unsigned long long* __restrict__ count) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (k < n) {
    int32_t r = rem[sa[k]], v = lcp[k];
    for (int32_t m = mmin; m <= mmax; ++m) c += (r >= m && v < m) ? 1 : 0;
  }
  // warp aggregate then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void k_table_insert(Sparse S, const int32_t* __restrict__ lcp, const int32_t* __restrict__ sa,
                               const int32_t* __restrict__ rem, const int32_t* __restrict__ text,
                               const int64_t* __restrict__ wsum, const int32_t* __restrict__ heavy,
                               const int32_t* __restrict__ rid, const int32_t* __restrict__ resp_slot,
                               int64_t n, int32_t mmin, int32_t mmax, HsGramEntry* __restrict__ table,
                               int64_t* __restrict__ table_mass, int64_t mask) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t p = sa[k], r = rem[p], v = lcp[k];
  int32_t slot = resp_slot[rid[p]];
  for (int32_t m = mmin; m <= mmax; ++m) {
    if (!(r >= m && v < m)) continue;
    int64_t rb = first_lt(S, k + 1, m) - 1;
    int32_t h;
    if (rb == k) {
      h = p;
    } else {
      int32_t d = rmq(S, k + 1, rb);
      h = heavy[first_le(S, k + 1, d)];
    }
    uint64_t hv = gram_hash(slot, m, text + p);
    int32_t tag = gram_tag(hv, m);
    int64_t mass = wsum[rb + 1] - wsum[k];
    int64_t idx = (int64_t)(hv & (uint64_t)mask);
    for (;;) {
      int32_t old = atomicCAS(&table[idx].pos, -1, h);
      if (old == -1) {
        table[idx].tag = tag;
        table_mass[idx] = mass;
        break;
      }
      idx = (idx + 1) & mask;
    }
  }
}

}  // namespace hs

using namespace hs;

// ------------------------------------------------------------------ host side
namespace {

struct Carve {
  char* base;
  size_t off = 0, cap;
  bool dry;
  Carve(void* b, size_t c, bool d) : base((char*)b), cap(c), dry(d) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T* p = dry ? nullptr : (T*)(base + off);
    off += sizeof(T) * count;
    return p;
  }
  bool ok() const { return dry || off <= cap; }
};

int ceil_log2(int64_t x) {
  int r = 0;
  while (((int64_t)1 << r) < x) ++r;
  return r;
}

inline unsigned blocks(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

struct Dims {
  int64_t ntok, ntext;
  int32_t nresp, nslots, max_len, rounds, levels, key_bits;
};

Dims dims_of(int64_t ntok, int32_t nresp, int32_t nslots, int32_t max_len, int64_t max_slot_suffixes) {
  Dims d;
  d.ntok = ntok;
  d.ntext = ntok + nresp;
  d.nresp = nresp;
  d.nslots = nslots;
  d.max_len = max_len < 1 ? 1 : max_len;
  d.rounds = ceil_log2(d.max_len);                 // doublings: window 2^rounds >= max_len
  d.levels = ceil_log2(max_slot_suffixes + 2) + 1; // sparse-table levels
  d.key_bits = ceil_log2(ntok + 2);
  if (d.key_bits < 1) d.key_bits = 1;
  return d;
}

// Lay out persistent + workspace buffers.  Same function for plan and build.
struct Layout {
  // persistent
  int32_t *text, *sa, *lcp, *heavy;
  int64_t *wsum, *slot_text_off, *slot_sa_off, *slot_stats;
  uint8_t* node_flags;
  // workspace
  int32_t *rid, *rem, *sufpos, *sufpos_alt, *sa_alt, *head, *gstart, *resp_slot, *node_lb, *cand_tok, *best_tok;
  int64_t *resp_off, *reward, *cand_parent, *cand_mass, *ptr, *wtmp;
  long long* best_mass;
  uint64_t *keys, *keys_alt;
  int32_t** rank_ptrs;   // device array of rank level pointers
  int32_t** lv_ptrs;     // device array of sparse level pointers
  int32_t* ranks;        // (rounds+1) x ntext
  int32_t* levels;       // (levels-1) x (n+1) (level 0 is lcp)
  unsigned long long* counters;
  void* cub_tmp;
  size_t cub_bytes;
  size_t index_bytes, ws_bytes;
};

size_t cub_bytes_needed(int64_t n) {
  size_t a = 0, b = 0, c = 0;
  cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, (int)std::max<int64_t>(n, 1), 0, 64);
  cub::DeviceScan::InclusiveScan(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, cub::Max(), (int)std::max<int64_t>(n, 1));
  cub::DeviceScan::ExclusiveSum(nullptr, c, (int64_t*)nullptr, (int64_t*)nullptr, (int)std::max<int64_t>(n + 1, 1));
  return std::max(a, std::max(b, c));
}

Layout make_layout(const Dims& d, void* index, size_t index_cap, void* ws, size_t ws_cap, bool dry) {
  Layout L;
  memset(&L, 0, sizeof(L));
  int64_t n = d.ntok;
  Carve P(index, index_cap, dry);
  L.text = P.take<int32_t>(d.ntext + HS_TEXT_PAD);
  L.sa = P.take<int32_t>(n + 1);
  L.lcp = P.take<int32_t>(n + 1);
  L.heavy = P.take<int32_t>(n + 1);
  L.wsum = P.take<int64_t>(n + 2);
  L.slot_text_off = P.take<int64_t>(d.nslots + 1);
  L.slot_sa_off = P.take<int64_t>(d.nslots + 1);
  L.slot_stats = P.take<int64_t>(2 * (int64_t)d.nslots + 2);
  L.node_flags = P.take<uint8_t>(n + 1);
  L.index_bytes = P.off + 256;

  Carve W(ws, ws_cap, dry);
  L.rid = W.take<int32_t>(d.ntext + HS_TEXT_PAD);
  L.rem = W.take<int32_t>(d.ntext + HS_TEXT_PAD);
  L.sufpos = W.take<int32_t>(n + 1);
  L.sufpos_alt = W.take<int32_t>(n + 1);
  L.sa_alt = W.take<int32_t>(n + 1);
  L.head = W.take<int32_t>(n + 1);
  L.gstart = W.take<int32_t>(n + 1);
  L.resp_slot = W.take<int32_t>(d.nresp + 1);
  L.resp_off = W.take<int64_t>(d.nresp + 1);
  L.reward = W.take<int64_t>(d.nresp + 1);
  L.keys = W.take<uint64_t>(n + 1);
  L.keys_alt = W.take<uint64_t>(n + 1);
  L.ranks = W.take<int32_t>((size_t)(d.rounds + 1) * (d.ntext + HS_TEXT_PAD));
  L.rank_ptrs = W.take<int32_t*>(d.rounds + 1);
  L.levels = W.take<int32_t>((size_t)std::max(d.levels - 1, 1) * (n + 1));
  L.lv_ptrs = W.take<int32_t*>(d.levels);
  L.node_lb = W.take<int32_t>(n + 1);
  L.cand_parent = W.take<int64_t>(2 * n + 2);
  L.cand_mass = W.take<int64_t>(2 * n + 2);
  L.cand_tok = W.take<int32_t>(2 * n + 2);
  L.best_mass = W.take<long long>(n + 1);
  L.best_tok = W.take<int32_t>(n + 1);
  L.ptr = W.take<int64_t>(n + 1);
  L.wtmp = W.take<int64_t>(n + 2);
  L.counters = W.take<unsigned long long>(d.nslots + 2);
  L.cub_bytes = cub_bytes_needed(n + 1);
  L.cub_tmp = W.take<char>(L.cub_bytes);
  L.ws_bytes = W.off + 256;
  return L;
}

thread_local char g_err[512];

}  // namespace

void hs_set_error(const char* msg) { snprintf(g_err, sizeof(g_err), "%s", msg); }

static int64_t g_launches = 0;
void hs_count_launches(int64_t n) { __atomic_fetch_add(&g_launches, n, __ATOMIC_RELAXED); }
extern "C" int64_t hs_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

extern "C" const char* hs_last_error(void) { return g_err; }
extern "C" int hs_version(void) { return 1; }

static int validate_meta(int64_t ntok, const int64_t* resp_off, int32_t nresp, const int64_t* slot_resp_off,
                         int32_t nslots, int32_t pmin, int32_t pmax, int32_t* max_len, int64_t* max_slot) {
  if (ntok < 0 || nresp < 0 || nslots < 0) { hs_set_error("negative size"); return HS_ERR_INVALID; }
  if (pmin < 1 || pmax < pmin || pmax > HS_MAX_TABLE_PREFIX) { hs_set_error("prefix range"); return HS_ERR_INVALID; }
  if (ntok + nresp + HS_TEXT_PAD >= ((int64_t)1 << 31)) { hs_set_error("history too large for int32 positions"); return HS_ERR_INVALID; }
  int32_t ml = 1;
  if (resp_off) {
    if (resp_off[0] != 0 || resp_off[nresp] != ntok) { hs_set_error("resp_off must span [0, n_tokens]"); return HS_ERR_INVALID; }
    for (int32_t r = 0; r < nresp; ++r) {
      int64_t l = resp_off[r + 1] - resp_off[r];
      if (l < 1) { hs_set_error("cannot index an empty response"); return HS_ERR_INVALID; }
      if (l > ml) ml = (int32_t)l;
    }
  }
  int64_t ms = 1;
  if (slot_resp_off) {
    if (slot_resp_off[0] != 0 || slot_resp_off[nslots] != nresp) { hs_set_error("slot_resp_off must span responses"); return HS_ERR_INVALID; }
    for (int32_t s = 0; s < nslots; ++s) {
      if (slot_resp_off[s + 1] < slot_resp_off[s]) { hs_set_error("slot_resp_off not sorted"); return HS_ERR_INVALID; }
      if (resp_off) {
        int64_t c = resp_off[slot_resp_off[s + 1]] - resp_off[slot_resp_off[s]];
        if (c > ms) ms = c;
      }
    }
  }
  *max_len = ml;
  *max_slot = ms;
  return HS_OK;
}

extern "C" int hs_index_plan(int64_t n_tokens, int32_t n_resp, int32_t n_slots, int32_t max_len,
                             int32_t prefix_min, int32_t prefix_max, HsIndexPlan* plan) {
  if (!plan || prefix_min < 1 || prefix_max < prefix_min || prefix_max > HS_MAX_TABLE_PREFIX) {
    hs_set_error("invalid plan arguments");
    return HS_ERR_INVALID;
  }
  // the slot size bound is the whole batch when unknown
  Dims d = dims_of(n_tokens, n_resp, n_slots, max_len, n_tokens);
  Layout L = make_layout(d, nullptr, 0, nullptr, 0, true);
  plan->index_bytes = L.index_bytes;
  plan->workspace_bytes = L.ws_bytes;
  return HS_OK;
}

extern "C" int hs_index_build(const int32_t* d_tokens, int64_t n_tokens, const int64_t* h_resp_off,
                              int32_t n_resp, const int64_t* h_slot_resp_off, int32_t n_slots,
                              const int64_t* h_reward_fx, int32_t prefix_min, int32_t prefix_max,
                              void* d_index, size_t index_bytes, void* d_ws, size_t ws_bytes,
                              HsIndexView* view, hs_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  int32_t max_len;
  int64_t max_slot;
  int rc = validate_meta(n_tokens, h_resp_off, n_resp, h_slot_resp_off, n_slots, prefix_min, prefix_max,
                         &max_len, &max_slot);
  if (rc) return rc;
  Dims plan_d = dims_of(n_tokens, n_resp, n_slots, max_len, n_tokens);
  Layout plan_L = make_layout(plan_d, nullptr, 0, nullptr, 0, true);
  if (index_bytes < plan_L.index_bytes || ws_bytes < plan_L.ws_bytes) {
    hs_set_error("index/workspace buffer smaller than hs_index_plan");
    return HS_ERR_SPACE;
  }
  Dims d = dims_of(n_tokens, n_resp, n_slots, max_len, max_slot);
  Layout L = make_layout(d, d_index, index_bytes, d_ws, ws_bytes, false);
  const int64_t n = d.ntok;

  // ---- host metadata -> device
  std::vector<int32_t> resp_slot(std::max(n_resp, 1));
  std::vector<int64_t> slot_text_off(n_slots + 1), slot_sa_off(n_slots + 1);
  for (int32_t s = 0; s < n_slots; ++s)
    for (int64_t r = h_slot_resp_off[s]; r < h_slot_resp_off[s + 1]; ++r) resp_slot[r] = s;
  for (int32_t s = 0; s <= n_slots; ++s) {
    int64_t r = h_slot_resp_off[s];
    slot_sa_off[s] = h_resp_off[r];
    slot_text_off[s] = h_resp_off[r] + r;
  }
  HS_CUDA_TRY(cudaMemcpyAsync(L.resp_off, h_resp_off, sizeof(int64_t) * (n_resp + 1), cudaMemcpyHostToDevice, st));
  if (n_resp) {
    HS_CUDA_TRY(cudaMemcpyAsync(L.resp_slot, resp_slot.data(), sizeof(int32_t) * n_resp, cudaMemcpyHostToDevice, st));
    HS_CUDA_TRY(cudaMemcpyAsync(L.reward, h_reward_fx, sizeof(int64_t) * n_resp, cudaMemcpyHostToDevice, st));
  }
  HS_CUDA_TRY(cudaMemcpyAsync(L.slot_text_off, slot_text_off.data(), sizeof(int64_t) * (n_slots + 1), cudaMemcpyHostToDevice, st));
  HS_CUDA_TRY(cudaMemcpyAsync(L.slot_sa_off, slot_sa_off.data(), sizeof(int64_t) * (n_slots + 1), cudaMemcpyHostToDevice, st));
  std::vector<int32_t*> rank_ptrs(d.rounds + 1), lv_ptrs(d.levels);
  for (int j = 0; j <= d.rounds; ++j) rank_ptrs[j] = L.ranks + (size_t)j * (d.ntext + HS_TEXT_PAD);
  lv_ptrs[0] = L.lcp;
  for (int j = 1; j < d.levels; ++j) lv_ptrs[j] = L.levels + (size_t)(j - 1) * (n + 1);
  HS_CUDA_TRY(cudaMemcpyAsync(L.rank_ptrs, rank_ptrs.data(), sizeof(int32_t*) * rank_ptrs.size(), cudaMemcpyHostToDevice, st));
  HS_CUDA_TRY(cudaMemcpyAsync(L.lv_ptrs, lv_ptrs.data(), sizeof(int32_t*) * lv_ptrs.size(), cudaMemcpyHostToDevice, st));

  // text padded with terminals, ranks zeroed (terminal rank 0)
  HS_CUDA_TRY(cudaMemsetAsync(L.text, 0xFF, sizeof(int32_t) * (d.ntext + HS_TEXT_PAD), st));
  HS_CUDA_TRY(cudaMemsetAsync(L.rem, 0, sizeof(int32_t) * (d.ntext + HS_TEXT_PAD), st));
  HS_CUDA_TRY(cudaMemsetAsync(L.ranks, 0, sizeof(int32_t) * (size_t)(d.rounds + 1) * (d.ntext + HS_TEXT_PAD), st));
  HS_CUDA_TRY(cudaMemsetAsync(L.slot_stats, 0, sizeof(int64_t) * (2 * (size_t)n_slots + 2), st));

  view->n_text = d.ntext;
  view->n_suffix = n;
  view->n_slots = n_slots;
  view->prefix_min = prefix_min;
  view->prefix_max = prefix_max;
  view->max_len = max_len;
  view->n_levels = d.levels;
  view->text = L.text;
  view->sa = L.sa;
  view->lcp = L.lcp;
  view->wsum = L.wsum;
  view->heavy = L.heavy;
  view->node_flags = L.node_flags;
  view->slot_text_off = L.slot_text_off;
  view->slot_sa_off = L.slot_sa_off;
  view->slot_stats = L.slot_stats;
  view->table = nullptr;
  view->table_mask = 0;
  view->n_gram_groups = 0;
  view->prefix_rounds = 0;
  view->ws = d_ws;
  view->ws_bytes = ws_bytes;
  if (n == 0) {
    HS_CUDA_TRY(cudaStreamSynchronize(st));
    return HS_OK;
  }

  hs_count_launches(1);
  k_layout<<<n_resp, 256, 0, st>>>(d_tokens, L.resp_off, L.resp_slot, n_resp, L.text, L.rid, L.rem,
                                   L.sufpos, L.keys);
  HS_CUDA_TRY(cudaGetLastError());

  // ---- prefix-doubling suffix sort
  int slot_bits = ceil_log2((int64_t)n_slots + 1);
  int rank_bits = d.key_bits;
  size_t cub_bytes = L.cub_bytes;
  {
    cub::DoubleBuffer<uint64_t> dk(L.keys, L.keys_alt);
    cub::DoubleBuffer<int32_t> dv(L.sufpos, L.sa_alt);
    HS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(L.cub_tmp, cub_bytes, dk, dv, (int)n, 0, 32 + slot_bits, st));
    hs_count_launches(1);
    k_group_head<<<blocks(n), 256, 0, st>>>(dk.Current(), n, L.head);
    HS_CUDA_TRY(cub::DeviceScan::InclusiveScan(L.cub_tmp, cub_bytes, L.head, L.gstart, cub::Max(), (int)n, st));
    hs_count_launches(1);
    k_scatter_rank<<<blocks(n), 256, 0, st>>>(dv.Current(), L.gstart, n, rank_ptrs[0]);
    HS_CUDA_TRY(cudaMemcpyAsync(L.sa, dv.Current(), sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  // suffix positions in text order for key generation (values are text positions).  Round j doubles the
  // window to 2^(j+1); once no tie can split any more the remaining rounds are skipped (one flag read per
  // round: a few microseconds against a full radix sort), and the LCP descent starts at the last level built
  unsigned long long* conv_flag = L.counters + n_slots + 1;
  int levels_built = 0;
  for (int j = 0; j < d.rounds; ++j) {
    if (j > 0) {
      unsigned long long not_done = 1;
      HS_CUDA_TRY(cudaMemsetAsync(conv_flag, 0, sizeof(unsigned long long), st));
      hs_count_launches(1);
      k_converged<<<blocks(n), 256, 0, st>>>(L.sa, L.gstart, L.rem, n, (int64_t)1 << j, conv_flag);
      HS_CUDA_TRY(cudaMemcpyAsync(&not_done, conv_flag, sizeof(not_done), cudaMemcpyDeviceToHost, st));
      HS_CUDA_TRY(cudaStreamSynchronize(st));
      if (!not_done) break;
    }
    levels_built = j + 1;
    int32_t h = 1 << j;
    // keys from the previous order (any order works; reuse sa to keep locality)
    hs_count_launches(1);
    k_double_keys<<<blocks(n), 256, 0, st>>>(L.sa, rank_ptrs[j], L.rem, n, h, rank_bits, L.keys);
    HS_CUDA_TRY(cudaMemcpyAsync(L.sufpos, L.sa, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    cub::DoubleBuffer<uint64_t> dk(L.keys, L.keys_alt);
    cub::DoubleBuffer<int32_t> dv(L.sufpos, L.sa_alt);
    HS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(L.cub_tmp, cub_bytes, dk, dv, (int)n, 0, 2 * rank_bits, st));
    hs_count_launches(1);
    k_group_head<<<blocks(n), 256, 0, st>>>(dk.Current(), n, L.head);
    HS_CUDA_TRY(cub::DeviceScan::InclusiveScan(L.cub_tmp, cub_bytes, L.head, L.gstart, cub::Max(), (int)n, st));
    hs_count_launches(1);
    k_scatter_rank<<<blocks(n), 256, 0, st>>>(dv.Current(), L.gstart, n, rank_ptrs[j + 1]);
    HS_CUDA_TRY(cudaMemcpyAsync(L.sa, dv.Current(), sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  HS_CUDA_TRY(cudaGetLastError());

  // ---- LCP, weights, sparse table
  hs_count_launches(1);
  k_lcp<<<blocks(n + 1), 256, 0, st>>>(L.sa, L.rem, L.rid, L.resp_slot, L.rank_ptrs, levels_built, n, L.lcp);
  view->prefix_rounds = levels_built;
  hs_count_launches(1);
  k_weights<<<blocks(n + 1), 256, 0, st>>>(L.sa, L.rid, L.reward, n, L.wtmp);
  HS_CUDA_TRY(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cub_bytes, L.wtmp, L.wsum, (int)(n + 1), st));
  for (int j = 1; j < d.levels; ++j) {
    hs_count_launches(1);
    k_sparse_level<<<blocks(n + 1), 256, 0, st>>>(lv_ptrs[j - 1], n + 1, (int64_t)1 << (j - 1), lv_ptrs[j]);
  }
  HS_CUDA_TRY(cudaGetLastError());

  // ---- LCP-interval tree, best children, heavy continuations
  Sparse S{(const int32_t* const*)L.lv_ptrs, d.levels, n + 1};
  SlotMap M{L.rid, L.resp_slot, L.slot_sa_off};
  HS_CUDA_TRY(cudaMemsetAsync(L.node_flags, 0, n + 1, st));
  hs_count_launches(1);
  k_nodes<<<blocks(n), 256, 0, st>>>(S, L.lcp, L.sa, L.rem, L.text, L.wsum, M, n, L.node_lb, L.node_flags,
                                     L.cand_parent, L.cand_mass, L.cand_tok);
  {
    // fill best_mass with INT64_MIN, best_tok with INT32_MAX
    HS_CUDA_TRY(cudaMemsetAsync(L.best_mass, 0x80, sizeof(long long) * n, st));  // 0x8080.. < any real mass
    HS_CUDA_TRY(cudaMemsetAsync(L.best_tok, 0x7F, sizeof(int32_t) * n, st));
    HS_CUDA_TRY(cudaMemsetAsync(L.ptr, 0xFF, sizeof(int64_t) * n, st));
  }
  int64_t nc = 2 * n;
  hs_count_launches(1);
  k_best_mass<<<blocks(nc), 256, 0, st>>>(L.cand_parent, L.cand_mass, nc, L.best_mass);
  hs_count_launches(1);
  k_best_tok<<<blocks(nc), 256, 0, st>>>(L.cand_parent, L.cand_mass, L.cand_tok, nc, L.best_mass, L.best_tok);
  hs_count_launches(1);
  k_best_child<<<blocks(nc), 256, 0, st>>>(L.cand_parent, L.cand_mass, L.cand_tok, nc, n, L.best_mass,
                                           L.best_tok, L.ptr, L.node_flags);
  hs_count_launches(1);
  k_ptr_init<<<blocks(n), 256, 0, st>>>(L.node_flags, L.node_lb, n, L.ptr);
  int jumps = ceil_log2((int64_t)max_len + 2) + 1;
  for (int j = 0; j < jumps; ++j) k_ptr_jump<<<blocks(n), 256, 0, st>>>(L.ptr, n);
  hs_count_launches(1);
  k_heavy<<<blocks(n), 256, 0, st>>>(L.ptr, L.sa, n, L.heavy);
  HS_CUDA_TRY(cudaGetLastError());

  // ---- per-slot stats + n-gram group count
  HS_CUDA_TRY(cudaMemsetAsync(L.counters, 0, sizeof(unsigned long long) * (n_slots + 2), st));
  hs_count_launches(1);
  k_slot_stats<<<blocks(n), 256, 0, st>>>(L.lcp, L.sa, L.rem, L.node_flags, M, n, L.counters);
  HS_CUDA_TRY(cudaMemcpy2DAsync(L.slot_stats, 2 * sizeof(int64_t), L.counters, sizeof(int64_t), sizeof(int64_t),
                                n_slots, cudaMemcpyDeviceToDevice, st));
  unsigned long long* group_counter = L.counters + n_slots;
  HS_CUDA_TRY(cudaMemsetAsync(group_counter, 0, sizeof(unsigned long long), st));
  hs_count_launches(1);
  k_count_groups<<<blocks(n), 256, 0, st>>>(L.lcp, L.sa, L.rem, n, prefix_min, prefix_max, group_counter);
  HS_CUDA_TRY(cudaGetLastError());
  unsigned long long groups = 0;
  HS_CUDA_TRY(cudaMemcpyAsync(&groups, group_counter, sizeof(groups), cudaMemcpyDeviceToHost, st));
  HS_CUDA_TRY(cudaStreamSynchronize(st));
  view->n_gram_groups = (int64_t)groups;
  return HS_OK;
}

extern "C" int hs_index_table_bytes(const HsIndexView* view, size_t* bytes) {
  int64_t cap = 1024;
  while (cap < 2 * view->n_gram_groups) cap <<= 1;
  *bytes = (sizeof(HsGramEntry) + sizeof(int64_t)) * (size_t)cap;   // entries, then the parallel masses
  return HS_OK;
}

extern "C" int hs_index_build_table(HsIndexView* view, void* d_table, size_t table_bytes, hs_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  size_t need;
  hs_index_table_bytes(view, &need);
  if (table_bytes < need) { hs_set_error("table buffer too small"); return HS_ERR_SPACE; }
  int64_t cap = (int64_t)(need / (sizeof(HsGramEntry) + sizeof(int64_t)));
  HsGramEntry* table = (HsGramEntry*)d_table;
  int64_t* table_mass = reinterpret_cast<int64_t*>(table + cap);
  HS_CUDA_TRY(cudaMemsetAsync(table, 0xFF, sizeof(HsGramEntry) * (size_t)cap, st));   // pos = -1: empty
  int64_t n = view->n_suffix;
  if (n > 0) {
    // rebuild the workspace layout to find rid / rem / sparse levels
    Dims d;
    d.ntok = n;
    d.ntext = view->n_text;
    d.nresp = (int32_t)(view->n_text - n);
    d.nslots = view->n_slots;
    d.max_len = view->max_len;
    d.rounds = ceil_log2(d.max_len);
    d.levels = view->n_levels;
    d.key_bits = ceil_log2(n + 2);
    Layout L = make_layout(d, nullptr, SIZE_MAX, view->ws, view->ws_bytes, false);
    Sparse S{(const int32_t* const*)L.lv_ptrs, d.levels, n + 1};
    hs_count_launches(1);
    k_table_insert<<<blocks(n), 256, 0, st>>>(S, view->lcp, view->sa, L.rem, view->text, view->wsum, view->heavy,
                                              L.rid, L.resp_slot, n, view->prefix_min, view->prefix_max, table,
                                              table_mass, cap - 1);
    HS_CUDA_TRY(cudaGetLastError());
  }
  view->table = table;
  view->table_mask = cap - 1;
  return HS_OK;
}
