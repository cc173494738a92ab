/*
 * histospec.h -- C-ABI of the B200 HistoSpec hot path (libhistospec.so).
 *
 * Plain pointers and sizes only; no torch types.  Device pointers are marked
 * d_*, host pointers h_*.  Every function returns HS_OK (0) or a negative
 * HS_ERR_* code; hs_last_error() returns a static message for the last error
 * on the calling thread.  All kernels are stream-ordered and non-blocking
 * unless stated otherwise.  The library allocates no persistent device memory:
 * callers own every buffer (plan -> allocate -> build).
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/pkg/src/rhymesim/):
 *   hs_index_plan / hs_index_build / hs_index_build_table
 *       -> history.py:343-355 build_tree, :148-279 SuffixTree.add_response /
 *          finalize, :417-422 HistoryStore._build_and_swap
 *   hs_lookup_batch
 *       -> history.py:283-300 match_prefix, :302-333 extract_draft
 *   hs_draft
 *       -> spec_engine.py:206-215 (prefix slice + extract_draft inside
 *          step_response), batched over sequences
 *   hs_accept_replay / hs_accept_greedy
 *       -> spec_engine.py:100-107 verify, :49-53 next_window, :69-72
 *          choose_prefix, :124-133 SpecStats.record, :217-240 step_response
 *          (replay: truth supplied; greedy: truth = argmax of the verify rows)
 *   hs_replay_fused
 *       -> spec_engine.py:260-279 replay_response, whole responses per launch
 *   hs_similarity_replay / hs_similarity_replay_isa (+ hs_index_inverse_sa)
 *       -> tracegen.py:306-353 token_similarity_replay (the paper's 5.1
 *          prefix-search similarity metric), one warp per response
 */
#ifndef HISTOSPEC_H_
#define HISTOSPEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_OK 0
#define HS_ERR_INVALID (-1)   /* maps to ValueError */
#define HS_ERR_CUDA (-2)      /* CUDA runtime failure */
#define HS_ERR_SPACE (-3)     /* caller buffer too small */

/* Fixed-point reward scale: reward_fx = reward * 2^HS_REWARD_FRAC_BITS. */
#define HS_REWARD_FRAC_BITS 32
/* Extra -1 entries after the text so warp-wide reads never leave the buffer. */
#define HS_TEXT_PAD 64
#define HS_MAX_WINDOW 32      /* hs_draft / hs_accept_* window_max limit */
#define HS_MAX_TABLE_PREFIX 32

typedef void* hs_stream_t;    /* cudaStream_t */

/* n-gram table entry.  The table buffer holds (table_mask + 1) entries followed by as many int64
 * fixed-point reward masses (mass of entry i at ((int64_t*)(table + table_mask + 1))[i]): the draft
 * hot path probes 8-byte entries and never touches the masses. */
typedef struct {
  int32_t pos;    /* text position of the heavy occurrence; -1 = empty slot */
  int32_t tag;    /* hash bits | m */
} HsGramEntry;

typedef struct {
  size_t index_bytes;      /* persistent arrays (text, SA, LCP, mass sums, heavy) */
  size_t workspace_bytes;  /* scratch, must stay untouched until build_table */
} HsIndexPlan;

typedef struct {
  /* persistent device arrays inside the caller's index buffer */
  const int32_t* text;          /* [n_text + HS_TEXT_PAD]; -1 after each response */
  const int32_t* sa;            /* [n_suffix] suffix array, slot-major */
  const int32_t* lcp;           /* [n_suffix + 1]; -1 at slot starts and the end */
  const int64_t* wsum;          /* [n_suffix + 1] exclusive prefix sums of weights */
  const int32_t* heavy;         /* [n_suffix] heavy text position per node id */
  const uint8_t* node_flags;    /* [n_suffix] bit0 node, bit1 has token child */
  const int64_t* slot_text_off; /* [n_slots + 1] */
  const int64_t* slot_sa_off;   /* [n_slots + 1] */
  int64_t* slot_stats;          /* [n_slots, 2]: reference node count, root mass */
  const HsGramEntry* table;     /* NULL until hs_index_build_table */
  int64_t table_mask;
  int64_t n_text, n_suffix;
  int32_t n_slots, prefix_min, prefix_max, max_len;
  int32_t n_levels;             /* sparse-table levels kept in the workspace */
  int64_t n_gram_groups;        /* host copy, valid after hs_index_build returns */
  void* ws;                     /* workspace pointer used by the build */
  size_t ws_bytes;
  int32_t prefix_rounds;        /* prefix-doubling rounds the build ran (it stops once no tie can split) */
} HsIndexView;

typedef struct {
  int32_t enabled, window_init, window_add, window_max, prefix_init, prefix_min;
} HsSpecConfig;

const char* hs_last_error(void);
int hs_version(void);
/* Number of this library's own kernel launches so far (process-wide). */
int64_t hs_launch_count(void);

/* Sizes for a build over n_tokens tokens in n_resp responses / n_slots slots. */
int hs_index_plan(int64_t n_tokens, int32_t n_resp, int32_t n_slots, int32_t max_len,
                  int32_t prefix_min, int32_t prefix_max, HsIndexPlan* plan);

/* K1a: suffix array, LCP, LCP-interval tree, heavy continuations.
 * Responses must be grouped by slot: slot s owns responses
 * [h_slot_resp_off[s], h_slot_resp_off[s+1]).  Synchronizes `stream` once
 * at the end (to read the n-gram group count). */
int hs_index_build(const int32_t* d_tokens, int64_t n_tokens,
                   const int64_t* h_resp_off, int32_t n_resp,
                   const int64_t* h_slot_resp_off, int32_t n_slots,
                   const int64_t* h_reward_fx, int32_t prefix_min, int32_t prefix_max,
                   void* d_index, size_t index_bytes, void* d_ws, size_t ws_bytes,
                   HsIndexView* view, hs_stream_t stream);

/* K1b: n-gram -> heavy-occurrence hash table for m in [prefix_min, prefix_max]. */
int hs_index_table_bytes(const HsIndexView* view, size_t* bytes);
int hs_index_build_table(HsIndexView* view, void* d_table, size_t table_bytes, hs_stream_t stream);

/* General lookups (any prefix length / window): binary search over the SA.
 * out_info[i*6 + {0..5}] = found, draft_len, mass_fx, at_node, heavy_pos, locus_depth. */
int hs_lookup_batch(const HsIndexView* view, int32_t n, const int32_t* d_slot,
                    const int32_t* d_prefix, int32_t prefix_stride, const int32_t* d_prefix_len,
                    const int32_t* d_window, int32_t* d_out_tok, int32_t out_stride,
                    int64_t* d_out_info, int32_t use_table, hs_stream_t stream);

/* K2: batched draft proposal for the rollout step.
 * Looks up iff speculate[s] && gen_len[s] >= prefix_len[s] (spec_engine.py:210),
 * using the last prefix_len generated tokens of row s.  [prefix_lo, prefix_hi]
 * and window_hi bound the values prefix_len / window can hold (SpecConfig
 * prefix_min..prefix_init, window_max): when every such prefix length is in
 * the n-gram table and <= 8, four sequences share a warp (8-lane groups);
 * otherwise one warp per sequence with the SA fallback. */
int hs_draft(const HsIndexView* view, int32_t n_seq, const int32_t* d_slot_of_seq,
             const int32_t* d_gen_tok, int32_t gen_stride, const int32_t* d_gen_len,
             const int32_t* d_prefix_len, const int32_t* d_window, const uint8_t* d_speculate,
             int32_t prefix_lo, int32_t prefix_hi, int32_t window_hi,
             int32_t* d_draft_tok, int32_t draft_stride, int32_t* d_draft_len,
             uint8_t* d_looked, uint8_t* d_found, hs_stream_t stream);

/* K6 (replay): accept against supplied truth rows; appends accepted + bonus to
 * gen rows, updates window / prefix / stats[n,5] and optionally records
 * tokens-per-iteration (d_tpi may be NULL). */
int hs_accept_replay(int32_t n_seq, const int32_t* d_truth, int32_t truth_stride,
                     const int32_t* d_target_len, const int32_t* d_draft_tok, int32_t draft_stride,
                     const int32_t* d_draft_len, const uint8_t* d_looked, const uint8_t* d_found,
                     int32_t* d_gen_tok, int32_t gen_stride, int32_t* d_gen_len,
                     int32_t* d_window, int32_t* d_prefix_len, int64_t* d_stats,
                     int32_t* d_tpi, int32_t tpi_stride, int32_t* d_n_iter,
                     HsSpecConfig cfg, hs_stream_t stream);

/* K6 (greedy): truth = argmax rows of the verify forward.  Row q_off[s] + i
 * holds the model's next-token argmax after consuming [last, d_1..d_i].
 * KV rollback is implicit: there is no kv_len array.  The next verify batch
 * (hm_build_verify_batch) places its first row at position
 * prompt_len + gen_len_new - 1, so KV rows written for rejected draft tokens
 * lie past the valid context and are overwritten (the bonus token's KV is
 * written by that next forward). */
int hs_accept_greedy(int32_t n_seq, const int32_t* d_argmax, const int32_t* d_q_off,
                     const int32_t* d_target_len, const int32_t* d_draft_tok, int32_t draft_stride,
                     const int32_t* d_draft_len, const uint8_t* d_looked, const uint8_t* d_found,
                     int32_t* d_gen_tok, int32_t gen_stride, int32_t* d_gen_len,
                     int32_t* d_window, int32_t* d_prefix_len, int64_t* d_stats,
                     int32_t* d_tpi, int32_t tpi_stride, int32_t* d_n_iter,
                     HsSpecConfig cfg, hs_stream_t stream);

/* Whole-response replay in one launch (warp per response): K2 + K6 fused. */
int hs_replay_fused(const HsIndexView* view, int32_t n_seq, const int32_t* d_slot_of_seq,
                    const int32_t* d_truth, const int64_t* d_truth_off, const uint8_t* d_speculate,
                    int32_t* d_tpi, int32_t* d_n_iter, int64_t* d_stats, HsSpecConfig cfg,
                    hs_stream_t stream);

/* Token-similarity replay over an index of the previous epoch's responses:
 * response r (tokens d_tokens[d_resp_off[r] : d_resp_off[r+1]]) is replayed
 * against slot d_slot_of_resp[r]; d_accepted[r] = tokens accepted by the
 * prefix search (tracegen.py:306-353).  A slot of -1 (or any slot outside
 * [0, n_slots)) means "no history for this prompt": d_accepted[r] = 0, as in
 * hs_draft / hs_lookup_batch.  prefix_len < 1 -> HS_ERR_INVALID. */
int hs_similarity_replay(const HsIndexView* view, int32_t n_resp, const int32_t* d_tokens,
                         const int64_t* d_resp_off, const int32_t* d_slot_of_resp, int32_t prefix_len,
                         int64_t* d_accepted, hs_stream_t stream);

/* Inverse suffix array of an index: d_isa[n_text] (int32), d_isa[sa[k]] = k, -1 at terminals. */
int hs_index_inverse_sa(const HsIndexView* view, int32_t* d_isa, hs_stream_t stream);

/* hs_similarity_replay seeded by the inverse suffix array (same results): each search after an
 * accepted run starts from the rank of the matched suffix advanced by the run. */
int hs_similarity_replay_isa(const HsIndexView* view, const int32_t* d_isa, int32_t n_resp,
                             const int32_t* d_tokens, const int64_t* d_resp_off, const int32_t* d_slot_of_resp,
                             int32_t prefix_len, int64_t* d_accepted, hs_stream_t stream);

/* Candidate branches of a draft tree (north_star (1) "frequency-weighted candidate branches"): for query i,
 * up to `width` (<= 8) branches, each a first token below the matched prefix -- the node's token children
 * ranked by reward mass, ties to the smaller token (history.py:322-331 order) -- followed by that child's greedy
 * (heavy) continuation, `window` tokens in all.  Branch 0 equals extract_draft's draft (history.py:302-333).
 * Out: d_out_tok [n, width, out_stride], d_out_len [n, width], d_out_mass [n, width] (fixed-point mass of the
 * branch's first token).  Unused branches have length 0. */
int hs_lookup_branches(const HsIndexView* view, int32_t n, const int32_t* d_slot, const int32_t* d_prefix,
                       int32_t prefix_stride, const int32_t* d_prefix_len, const int32_t* d_window, int32_t width,
                       int32_t* d_out_tok, int32_t out_stride, int32_t* d_out_len, int64_t* d_out_mass,
                       hs_stream_t stream);

/* Continuous batching (engine lanes): lane d_lane[i] takes a new sequence whose
 * generated tokens so far are d_tok[d_tok_off[i] : d_tok_off[i+1]] (empty for a fresh prompt; a migrated
 * rollout's prefix, whose KV the admission prefill recomputed) followed by d_argmax[d_first_row[i]] when
 * d_first_row[i] >= 0.  Target length, history slot (-1: none), speculation flag, AIMD window, prefix
 * length and stats [5] are set from the inputs (a fresh sequence: window_init, prefix_init, {1,0,0,0,1} --
 * its iteration 0 is a plain decode); draft / lookup flags are cleared.  d_prompt_len / d_seq_key (the
 * engine's per-lane prompt length and sampling key) are optional, in/out pairs together. */
int hs_lane_admit(int32_t n, const int32_t* d_lane, const int32_t* d_tok, const int64_t* d_tok_off,
                  const int32_t* d_argmax, const int32_t* d_first_row, const int32_t* d_target,
                  const int32_t* d_slot, const uint8_t* d_spec, const int32_t* d_window, const int32_t* d_prefix,
                  const int64_t* d_stats, const int32_t* d_prompt_len_in, const int32_t* d_key_in,
                  int32_t* d_gen_tok, int32_t gen_stride, int32_t* d_gen_len, int32_t* d_target_len,
                  int32_t* d_slots, uint8_t* d_speculate, int32_t* d_window_out, int32_t* d_prefix_out,
                  int64_t* d_stats_out, int32_t* d_draft_len, uint8_t* d_looked, uint8_t* d_found,
                  int32_t* d_prompt_len, int32_t* d_seq_key, hs_stream_t stream);

/* ---- per-epoch history update (hs_route.cu, history.py:396-437, io.py:41-88) ----
 *
 * hs_pack_rows: d_dst[d_dst_off[i] + j] = d_src[d_row[i] * src_stride + j] for j < d_len[i] -- gathers the
 * finished rollouts of a step (rows of the engine's [n_seq, stride] token matrix) into one flat buffer in
 * routing order (the send buffer of the all-to-all-v that moves them to their next owners). */
int hs_pack_rows(const int32_t* d_src, int64_t src_stride, const int32_t* d_row, const int64_t* d_len,
                 const int64_t* d_dst_off, int32_t n, int32_t* d_dst, hs_stream_t stream);

/* hs_mutate_bursts: for each routed rollout i (tokens d_src[d_src_off[i] : d_src_off[i+1]]) write G
 * independent s-similar copies (tracegen's burst semantics, tracegen.py:78-120; counter-hash RNG keyed by
 * (seed, i, g)) at d_dst + G * d_src_off[i] + g * len_i, and a Bernoulli(0.5) reward in fixed point to
 * d_reward_fx[i * G + g].  The bench's stand-in for policy drift between epochs (SURVEY.md 8(d), (D)
 * definition), feeding hs_index_build directly. */
int hs_mutate_bursts(const int32_t* d_src, const int64_t* d_src_off, int32_t n, int32_t G, double s,
                     double burst, int32_t vocab, uint64_t seed, int32_t* d_dst, int64_t* d_reward_fx,
                     hs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HISTOSPEC_H_ */
