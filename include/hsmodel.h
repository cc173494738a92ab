/*
 * hsmodel.h -- C-ABI of the verify-forward kernels (libhsmodel.so), sm_100a.
 *
 * The reference has no model: its "verify" compares drafts with a replayed
 * ground truth (rhymesim/spec_engine.py:100-107) and its simulator charges a
 * verify pass like a decode pass (sim.py:127-137).  These entry points are
 * the real forward that produces that truth: truth[pos + i] := argmax of
 * verify row i.  Qwen2-style decoder: RMSNorm, QKV with
 * bias, RoPE, GQA causal attention over a slot-contiguous KV cache, SwiGLU
 * MLP, tied or untied LM head with a fused argmax epilogue.
 *
 * Conventions: bf16 tensors are row-major with the last dim contiguous; the
 * residual stream is fp32 [M, d]; "d_m" (optional, may be NULL) points at a
 * device int32 holding the live row count, so launches sized for a maximum M
 * can be captured in a CUDA graph.
 */
#ifndef HSMODEL_H_
#define HSMODEL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HM_OK 0
#define HM_ERR_INVALID (-1)
#define HM_ERR_CUDA (-2)

#define HM_EPI_STORE 0     /* out bf16 = acc (+ bias) */
#define HM_EPI_SWIGLU 1    /* out bf16 [M, N/2] = silu(gate) * up; W rows interleaved in hm_gemm_bn(N)/2 halves */
#define HM_EPI_RESIDUAL 2  /* resid fp32 += acc */
#define HM_EPI_ARGMAX 3    /* per 128-column tile (max, argmax) partials */
#define HM_EPI_F32 4       /* out fp32 [M, ldr] = acc (residual add fused into hm_rmsnorm_residual) */

typedef void* hm_stream_t;

const char* hm_last_error(void);
int64_t hm_launch_count(void);

/* K3: Y = X . W^T on tcgen05 (bf16 in, fp32 TMEM accumulate), fused epilogue. */
int hm_gemm(int32_t epi, const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N,
            int32_t K, const void* d_bias, void* d_out, int64_t ldo, float* d_resid, int64_t ldr,
            float* d_amax_val, int32_t* d_amax_idx, const int32_t* d_m, hm_stream_t stream);

/* Sampling LM head (rejection-sampling verify at temperature T): the argmax
 * epilogue runs on logit/T + Gumbel(seed, key0[row], key1[row], v), a
 * counter-based hash of (seed, sequence slot, position, token).  Gumbel-max is
 * an exact sample of softmax(logit/T); verifying a point-mass draft x by
 * "accept iff the row's sample == x" accepts with probability p(x) and, on
 * rejection, emits a sample of p restricted to tokens != x -- the speculative
 * sampling rule -- while keeping the output identical to non-speculative
 * sampling with the same seed (bit-exact, batch-invariant). */
int hm_lm_head_sample(const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N, int32_t K,
                      const int32_t* d_key0, const int32_t* d_key1, uint64_t seed, float temperature,
                      float* d_amax_val, int32_t* d_amax_idx, const int32_t* d_m, hm_stream_t stream);

/* GEMM tile width chosen for an N (a function of N only, never of M). */
int hm_gemm_bn(int32_t n);

/* CTA-pair (cta_group::2, 256 x 256 tile over two SMs) GEMM kernels: 1 = used when there are at least
 * (#SMs / 2) 256 x 256 tiles (default), 0 = never (1-CTA kernels only).  Same bits either way; a switch for
 * A/B timing and the bit-neutrality tests. */
int hm_set_gemm_pair(int32_t on);

/* LM-head argmax: reduce the [M, n_tiles] partials of HM_EPI_ARGMAX (ties -> smallest id). */
int hm_argmax_reduce(const float* d_val, const int32_t* d_idx, int32_t M, int32_t n_tiles, const int32_t* d_m,
                     int32_t* d_out, hm_stream_t stream);

/* x[M, d] fp32 = embedding[tokens[i]] */
int hm_embed(const int32_t* d_tokens, const void* d_emb, int32_t M, int32_t d, float* d_x, const int32_t* d_m,
             hm_stream_t stream);

/* out bf16 = x * rsqrt(mean(x^2) + eps) * w  (row-local, fixed reduction order) */
int hm_rmsnorm(const float* d_x, const void* d_w, int32_t M, int32_t d, float eps, void* d_out,
               const int32_t* d_m, hm_stream_t stream);

/* x += y (both fp32 [M, d], y may be NULL), then out bf16 = rmsnorm(x) * w.
 * Fuses the residual add of the previous O/down projection into the norm. */
int hm_rmsnorm_residual(float* d_x, const float* d_y, const void* d_w, int32_t M, int32_t d, float eps, void* d_out,
                        const int32_t* d_m, hm_stream_t stream);

/* RoPE (rotate-half, table cos/sin [max_pos, hd/2] fp32) on q and k of the fused
 * qkv rows, q -> d_q [KVH][M][G][hd] (G = H / KVH: kv-group-major, so a group's
 * query rows are contiguous -- the attention Q tiles load them as plain 2-D boxes);
 * k, v -> cache[slot][kvh][pos][hd] */
int hm_rope_kv_append(const void* d_qkv, const int32_t* d_pos, const int32_t* d_row_slot, const float* d_cos,
                      const float* d_sin, int32_t M, int32_t H, int32_t KVH, int32_t hd, void* d_q, void* d_kcache,
                      void* d_vcache, int64_t slot_stride, int32_t max_len, const int32_t* d_m, hm_stream_t stream);

/* K3 + K5 fused: qkv = X . Wqkv^T + bias (rounded to bf16 as hm_gemm would store it), then RoPE on the q
 * and k heads at d_pos[row] and the hm_rope_kv_append writes -- q kv-group-major into d_q with M = q_rows,
 * k and v into cache[d_row_slot[row]][kvh][pos] -- from the GEMM epilogue: the qkv activations never
 * reach HBM.  Same bits as hm_gemm(HM_EPI_STORE) followed by hm_rope_kv_append. */
int hm_gemm_qkv_rope(const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t K,
                     const void* d_bias, int32_t H, int32_t KVH, int32_t hd, const int32_t* d_pos,
                     const int32_t* d_row_slot, const float* d_cos, const float* d_sin, void* d_q, int32_t q_rows,
                     void* d_kcache, void* d_vcache, int64_t slot_stride, int32_t max_len, const int32_t* d_m,
                     hm_stream_t stream);

/* K4: causal GQA attention for variable-length query blocks.  Sequence s owns
 * query rows [q_off[s], q_off[s] + q_len[s]) at positions pos0[s] + i and KV
 * slot kv_slot[s]; row i attends cache positions [0, pos0[s] + i].  d_q is
 * [KVH][q_rows][G][hd] (hm_rope_kv_append's layout with M = q_rows); d_out is
 * [rows][H * hd]. */
int hm_attention(const void* d_q, const void* d_kcache, const void* d_vcache, int64_t slot_stride,
                 const int32_t* d_q_off, const int32_t* d_q_len, const int32_t* d_pos0, const int32_t* d_kv_slot,
                 int32_t n_seq, int32_t max_q_len, int32_t H, int32_t KVH, int32_t hd, int32_t max_len,
                 float scale, void* d_out, int32_t* d_work /* hm_attention_work_size() int32 scratch or NULL */,
                 int32_t work_ready /* d_work already holds hm_attention_plan's output */,
                 int32_t n_slots /* cache slots, > 0 enables TMA loads */,
                 int32_t q_rows /* row stride of d_q's kv-group planes (> 0) */,
                 hm_stream_t stream);

/* Attention kernel family for the forwards that follow (process-wide): 0 = mma.sync m16n8k16
 * (4 warps split each 64-key stage), 1 = tcgen05 (TMEM S/P/O, 128-row tiles, 128-key stages; the
 * default).  Both are batch invariant; rows from different families differ in their last bits, so
 * a speculative rollout and the greedy run it is compared with use one family. */
int hm_set_attention_family(int32_t family);
int hm_attention_family(void);

/* CTA caps of the persistent kernels launched after this call (process-wide, read at launch time, so a
 * CUDA graph keeps the caps it was captured with): GEMMs use at most gemm_ctas CTAs and attention at most
 * attn_ctas (0 = one per SM).  Two streams whose kernels' caps add up to the SM count run side by side,
 * e.g. a KV-bandwidth-bound attention beside a tensor-core-bound GEMM of another half-batch.  A cap
 * changes only which CTA computes a tile, never a tile's arithmetic (bits are unchanged). */
int hm_set_grid_caps(int32_t gemm_ctas, int32_t attn_ctas);

/* Tensor parallelism over a GPU pair (configs[4]).
 * hm_rmsnorm_residual2: x += (y + y2) then rmsnorm, any d (y2 optional: the peer GPU's fp32 partial of the
 * O / down projection, read in place over NVLink from its symmetric buffer -- the all-reduce fused into the
 * norm).  hm_tp_barrier: stream-ordered two-GPU barrier over peer memory (system fence, release store of
 * this GPU's generation into the peer's flag, acquire spin on its own flag); graph-capturable. */
int hm_rmsnorm_residual2(float* d_x, const float* d_y, const float* d_y2, const void* d_w, int32_t M, int32_t d,
                         float eps, void* d_out, const int32_t* d_m, hm_stream_t stream);
int hm_tp_barrier(int32_t* d_my_flag, int32_t* d_peer_flag, int32_t* d_gen, hm_stream_t stream);

/* bf16 residual stream (Forward.residual = "bf16", the default): x (bf16 [M, d]) = bf16(x + y [+ y2]) with
 * y the O / down projection stored in bf16 by its GEMM (and y2 the TP peer's partial), then out = rmsnorm(x) * w;
 * y == NULL: norm only.  hm_embed_bf16: x rows = embedding rows (bf16, no conversion). */
int hm_rmsnorm_residual_bf16(void* d_x, const void* d_y, const void* d_y2, const void* d_w, int32_t M, int32_t d,
                             float eps, void* d_out, const int32_t* d_m, hm_stream_t stream);
int hm_embed_bf16(const int32_t* d_tok, const void* d_emb, int32_t M, int32_t d, void* d_x, const int32_t* d_m,
                  hm_stream_t stream);

/* Work list for hm_attention's persistent schedule (once per forward: q_len is layer independent): the
 * per-sequence tile prefix and, for the tcgen05 family, each tile's sequence.  d_work holds
 * hm_attention_work_size(n_seq, max_q_len, H, KVH) int32 values. */
int64_t hm_attention_work_size(int32_t n_seq, int32_t max_q_len, int32_t H, int32_t KVH);
int hm_attention_plan(const int32_t* d_q_len, int32_t n_seq, int32_t max_q_len, int32_t H, int32_t KVH,
                      int32_t* d_work, hm_stream_t stream);

/* Verify-batch assembly for the rollout step: for each live sequence s
 * (gen_len < target_len) rows [last generated token, draft_1..draft_k] at
 * positions prompt_len[s] + gen_len[s] - 1 + i.  Writes q_off/q_len/pos0,
 * per-row token/position/slot, and the live row count to d_m[0].
 * Optional accounting (NULL to skip), accumulated on the device:
 *   d_acc[4] += {rows, 1 if rows > 0, sum over rows of (pos + 1), sum over live sequences of (pos0 + q)}
 *   d_qhist[min(q, qhist_len - 1)] += 1 per sequence (q = 0 for finished ones), qhist_len in [2, 64].
 * Optional row keys: d_row_key[row] = d_seq_key[s] (both NULL or both set) -- the per-row RNG key of
 * hm_lm_head_sample, so sampling noise follows the sequence, not its KV slot. */
int hm_build_verify_batch(int32_t n_seq, const int32_t* d_gen_tok, int32_t gen_stride, const int32_t* d_gen_len,
                          const int32_t* d_target_len, const int32_t* d_prompt_len, const int32_t* d_draft_tok,
                          int32_t draft_stride, const int32_t* d_draft_len, const int32_t* d_kv_slot,
                          int32_t* d_tokens, int32_t* d_pos, int32_t* d_row_slot, int32_t* d_q_off,
                          int32_t* d_q_len, int32_t* d_pos0, int32_t* d_m, int64_t* d_acc, int64_t* d_qhist,
                          int32_t qhist_len, const int32_t* d_seq_key, int32_t* d_row_key, hm_stream_t stream);

/* fp32 parity path (tests only): the same forward with fp32 operands, fp32
 * accumulation and an fp32 KV cache ([slot][KVH][max_len][hd] float), plain SIMT kernels; weights are
 * the bf16 tensors, widened on load.  Logits are held to 1e-3 relative of the fp32 restatement.
 *   hm_f32_gemm:      Y[M, N] (+)= X[M, K] . W[N, K]^T (+ bias), W / bias bf16, X / Y fp32
 *   hm_f32_rmsnorm:   out = x * rsqrt(mean(x^2) + eps) * w
 *   hm_f32_rope_kv_append: rotate-half RoPE of q / k at pos[row]; q -> d_q [M][H][hd], k / v -> the caches
 *   hm_f32_attention: causal GQA softmax attention of row m over keys 0..pos[m] of slot row_slot[m]
 *   hm_f32_swiglu:    act = silu(gate) * up over the interleaved gate/up GEMM output (half-wide blocks) */
int hm_f32_gemm(const float* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N, int32_t K,
                const void* d_bias, float* d_y, int64_t ldy, int32_t accumulate, hm_stream_t stream);
int hm_f32_rmsnorm(const float* d_x, const void* d_w, int32_t M, int32_t d, float eps, float* d_out,
                   hm_stream_t stream);
int hm_f32_rope_kv_append(const float* d_qkv, const int32_t* d_pos, const int32_t* d_row_slot, const float* d_cos,
                          const float* d_sin, int32_t M, int32_t H, int32_t KVH, int32_t hd, float* d_q,
                          float* d_kcache, float* d_vcache, int64_t slot_stride, int32_t max_len, hm_stream_t stream);
int hm_f32_attention(const float* d_q, const float* d_kcache, const float* d_vcache, int64_t slot_stride,
                     const int32_t* d_pos, const int32_t* d_row_slot, int32_t M, int32_t H, int32_t KVH, int32_t hd,
                     int32_t max_len, float scale, float* d_out, hm_stream_t stream);
int hm_f32_swiglu(const float* d_gu, int32_t M, int32_t F, int32_t half, float* d_act, hm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HSMODEL_H_ */
