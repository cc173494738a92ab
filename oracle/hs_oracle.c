/*
 * hs_oracle.c -- plain-C restatement of the HistoSpec hot path.
 * TEST INFRASTRUCTURE ONLY: used by tests/ as the large-case checker and by
 * bench.py as the CPU baseline ("port").  Never linked into the product.
 *
 * Semantics restated (file:line into /root/reference/pkg/src/rhymesim):
 *   draft  : history.py:302-333 SuffixTree.extract_draft -- greedy
 *            max-priority continuation, ties to the smallest token, stop at
 *            window or response end (TERMINAL, history.py:317-318); a token's
 *            priority is the reward mass of the suffixes through it
 *            (leaf credit history.py:183,214,254-263; sums :265-279).
 *   match  : history.py:283-300 (source_priority = mass below the prefix,
 *            history.py:106-108).
 *   replay : spec_engine.py:200-240 step_response, :260-279 replay_response,
 *            AIMD :49-53, prefix policy :69-72, verify :100-107,
 *            stats :110-141.
 *
 * Method (deliberately NOT a suffix tree, so it shares no structure with the
 * reference or with the GPU suffix-array index): the occurrences of the
 * lookup pattern are found in a per-prompt array of positions sorted by
 * their m-gram (binary search), then the draft is grown token by token over
 * the live occurrences exactly like tests/oracles.py:49-81 greedy_draft.
 * Masses are float64 sums like the reference (exact for dyadic rewards).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const int32_t *text;    /* tokens, -1 after each response */
  const int32_t *rid;     /* response id of each text position */
  const double *reward;   /* per response */
} Hist;

/* ---- greedy continuation over live occurrences (oracles.py:49-81) ---- */

typedef struct { int32_t tok; double mass; } TokMass;

static int cmp_tok(const void *a, const void *b) {
  int32_t x = ((const TokMass *)a)->tok, y = ((const TokMass *)b)->tok;
  return (x > y) - (x < y);
}

/* live[]: text positions just after each occurrence (modified in place). */
static int32_t grow_draft(const Hist *h, int64_t *live, int64_t n_live, int32_t window,
                          int32_t *out, TokMass *scratch) {
  int32_t k = 0;
  while (k < window) {
    int64_t n = 0;
    for (int64_t i = 0; i < n_live; i++) {
      int32_t t = h->text[live[i]];
      if (t >= 0) { scratch[n].tok = t; scratch[n].mass = h->reward[h->rid[live[i]]]; n++; }
    }
    if (n == 0) break;
    qsort(scratch, (size_t)n, sizeof(TokMass), cmp_tok);
    int32_t best_tok = -1; double best_mass = 0.0;
    for (int64_t i = 0; i < n;) {
      int64_t j = i; double m = 0.0;
      while (j < n && scratch[j].tok == scratch[i].tok) { m += scratch[j].mass; j++; }
      /* ascending token order: strict > keeps the smallest token on ties */
      if (best_tok < 0 || m > best_mass) { best_tok = scratch[i].tok; best_mass = m; }
      i = j;
    }
    out[k++] = best_tok;
    int64_t w = 0;
    for (int64_t i = 0; i < n_live; i++)
      if (h->text[live[i]] == best_tok) live[w++] = live[i] + 1;
    n_live = w;
  }
  return k;
}

/* Brute-force draft over a small corpus (linear scan for the prefix). */
int32_t hso_draft(const int32_t *text, const int32_t *rid, const double *reward, int64_t n_text,
                  const int32_t *prefix, int32_t m, int32_t window,
                  int32_t *out, int32_t *out_len, double *mass) {
  Hist h = {text, rid, reward};
  *out_len = 0; *mass = 0.0;
  if (m < 1 || window < 1) return -1;
  int64_t *live = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_text + 1));
  TokMass *scratch = (TokMass *)malloc(sizeof(TokMass) * (size_t)(n_text + 1));
  int64_t n_live = 0;
  for (int64_t i = 0; i + m <= n_text; i++) {
    int32_t j = 0;
    while (j < m && text[i + j] == prefix[j]) j++;
    if (j == m) { live[n_live++] = i + m; *mass += reward[rid[i]]; }
  }
  int32_t found = n_live > 0;
  if (found) *out_len = grow_draft(&h, live, n_live, window, out, scratch);
  free(live); free(scratch);
  return found;
}

/* ---- per-prompt m-gram position index ---- */

typedef struct { const int32_t *text; int32_t m; } SortCtx;

static int cmp_gram(const void *a, const void *b, void *ctx) {
  const SortCtx *c = (const SortCtx *)ctx;
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  for (int32_t j = 0; j < c->m; j++) {
    int32_t u = c->text[x + j], v = c->text[y + j];
    if (u != v) return (u > v) - (u < v);
  }
  return (x > y) - (x < y);
}

typedef struct {
  int64_t *pos[65];   /* pos[m]: start positions of m-grams, sorted by m-gram */
  int64_t cnt[65];
} GramIndex;

static int cmp_prefix_at(const int32_t *text, int64_t p, const int32_t *pre, int32_t m) {
  for (int32_t j = 0; j < m; j++) {
    int32_t u = text[p + j];
    if (u != pre[j]) return (u > pre[j]) - (u < pre[j]);
  }
  return 0;
}

static void gram_range(const GramIndex *g, const int32_t *text, const int32_t *pre, int32_t m,
                       int64_t *lo_out, int64_t *hi_out) {
  const int64_t *a = g->pos[m];
  int64_t lo = 0, hi = g->cnt[m];
  while (lo < hi) { int64_t mid = (lo + hi) / 2; if (cmp_prefix_at(text, a[mid], pre, m) < 0) lo = mid + 1; else hi = mid; }
  int64_t l = lo; hi = g->cnt[m];
  while (lo < hi) { int64_t mid = (lo + hi) / 2; if (cmp_prefix_at(text, a[mid], pre, m) <= 0) lo = mid + 1; else hi = mid; }
  *lo_out = l; *hi_out = lo;
}

/* ---- batched replay (spec_engine.py:200-279) ---- */

typedef struct {
  /* history */
  const int32_t *text; const int32_t *rid; const double *reward;
  const int64_t *prompt_text_off;   /* [n_prompts+1] text range of each prompt */
  const uint8_t *has_tree;
  int32_t n_prompts;
  /* truths */
  const int32_t *truth; const int64_t *truth_off; const int32_t *truth_prompt; int32_t n_truth;
  int32_t cfg[6];   /* enabled, w_init, w_add, w_max, p_init, p_min */
  int32_t speculate;
  int32_t *tpi_out; int64_t *n_iter_out; int64_t *stats_out;
  GramIndex *idx;
  volatile int64_t next_prompt, next_truth;
} Job;

static void build_prompt_index(Job *J, int32_t p) {
  GramIndex *g = &J->idx[p];
  int64_t a = J->prompt_text_off[p], b = J->prompt_text_off[p + 1];
  for (int32_t m = J->cfg[5]; m <= J->cfg[4]; m++) {
    int64_t n = 0;
    int64_t *arr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(b - a + 1));
    for (int64_t i = a; i < b; i++) {
      int32_t j = 0;
      while (j < m && i + j < b && J->text[i + j] >= 0) j++;
      if (j == m) arr[n++] = i;
    }
    SortCtx c = {J->text, m};
    qsort_r(arr, (size_t)n, sizeof(int64_t), cmp_gram, &c);
    g->pos[m] = arr; g->cnt[m] = n;
  }
}

static void replay_one(Job *J, int32_t t, int64_t *live, TokMass *scratch, int32_t *draft) {
  const int32_t *truth = J->truth + J->truth_off[t];
  int64_t n = J->truth_off[t + 1] - J->truth_off[t];
  int32_t p = J->truth_prompt[t];
  int32_t spec = J->speculate && J->cfg[0];
  int32_t has_tree = spec && J->has_tree[p];
  int32_t window = J->cfg[1], cur = J->cfg[4];
  int64_t pos = 0, iters = 0;
  int64_t st_total = 0, st_spec = 0, st_acc = 0, st_ver = 0, st_dec = 0;
  Hist h = {J->text, J->rid, J->reward};
  int32_t *tpi = J->tpi_out + J->truth_off[t];
  while (pos < n) {
    int32_t k = 0, looked = 0, found = 0;
    if (has_tree && pos >= cur) {
      looked = 1;
      int64_t lo, hi;
      gram_range(&J->idx[p], J->text, truth + pos - cur, cur, &lo, &hi);
      found = hi > lo;
      if (found) {
        int64_t nl = 0;
        for (int64_t i = lo; i < hi; i++) live[nl++] = J->idx[p].pos[cur][i] + cur;
        k = grow_draft(&h, live, nl, window, draft, scratch);
      }
    }
    if (k == 0) {
      pos += 1; st_total += 1; st_dec += 1;
      if (looked) cur = found ? J->cfg[4] : (cur - 1 > J->cfg[5] ? cur - 1 : J->cfg[5]);
      tpi[iters++] = 1;
      continue;
    }
    int64_t rest = n - pos, a = 0;
    while (a < k && a < rest && draft[a] == truth[pos + a]) a++;
    int32_t all = (a == k);
    int64_t appended = a < rest ? a : rest;
    pos += appended;
    int64_t bonus = pos < n ? 1 : 0;
    pos += bonus;
    st_total += appended + bonus; st_spec += k; st_acc += appended; st_ver += 1;
    window = all ? (window + J->cfg[2] < J->cfg[3] ? window + J->cfg[2] : J->cfg[3]) : J->cfg[1];
    cur = J->cfg[4];
    tpi[iters++] = (int32_t)(appended + bonus);
  }
  J->n_iter_out[t] = iters;
  int64_t *s = J->stats_out + 5 * (int64_t)t;
  s[0] = st_total; s[1] = st_spec; s[2] = st_acc; s[3] = st_ver; s[4] = st_dec;
}

static void *worker(void *arg) {
  Job *J = (Job *)arg;
  for (;;) {
    int64_t p = __atomic_fetch_add(&J->next_prompt, 1, __ATOMIC_RELAXED);
    if (p >= J->n_prompts) break;
    if (J->has_tree[p] && J->speculate && J->cfg[0]) build_prompt_index(J, (int32_t)p);
  }
  return NULL;
}

static void *worker2(void *arg) {
  Job *J = (Job *)arg;
  int64_t maxlen = 1;
  for (int32_t p = 0; p < J->n_prompts; p++) {
    int64_t l = J->prompt_text_off[p + 1] - J->prompt_text_off[p];
    if (l > maxlen) maxlen = l;
  }
  int64_t *live = (int64_t *)malloc(sizeof(int64_t) * (size_t)(maxlen + 1));
  TokMass *scratch = (TokMass *)malloc(sizeof(TokMass) * (size_t)(maxlen + 1));
  int32_t *draft = (int32_t *)malloc(sizeof(int32_t) * (size_t)(J->cfg[3] + 1));
  for (;;) {
    int64_t t = __atomic_fetch_add(&J->next_truth, 1, __ATOMIC_RELAXED);
    if (t >= J->n_truth) break;
    replay_one(J, (int32_t)t, live, scratch, draft);
  }
  free(live); free(scratch); free(draft);
  return NULL;
}

/*
 * Replay every truth response against its prompt's history.
 * tpi_out has room for sum(truth lengths) entries, laid out like truth.
 * stats_out: [n_truth, 5] = total, speculated, accepted, verify, decode.
 */
int32_t hso_replay(const int32_t *text, const int32_t *rid, const double *reward,
                   const int64_t *prompt_text_off, const uint8_t *has_tree, int32_t n_prompts,
                   const int32_t *truth, const int64_t *truth_off, const int32_t *truth_prompt,
                   int32_t n_truth, const int32_t *cfg6, int32_t speculate,
                   int32_t *tpi_out, int64_t *n_iter_out, int64_t *stats_out, int32_t n_threads) {
  if (cfg6[5] < 1 || cfg6[4] > 64 || cfg6[4] < cfg6[5] || cfg6[1] < 1 || cfg6[3] < cfg6[1]) return -1;
  Job J;
  memset(&J, 0, sizeof(J));
  J.text = text; J.rid = rid; J.reward = reward; J.prompt_text_off = prompt_text_off;
  J.has_tree = has_tree; J.n_prompts = n_prompts; J.truth = truth; J.truth_off = truth_off;
  J.truth_prompt = truth_prompt; J.n_truth = n_truth; memcpy(J.cfg, cfg6, sizeof(J.cfg));
  J.speculate = speculate; J.tpi_out = tpi_out; J.n_iter_out = n_iter_out; J.stats_out = stats_out;
  J.idx = (GramIndex *)calloc((size_t)(n_prompts > 0 ? n_prompts : 1), sizeof(GramIndex));
  if (n_threads < 1) n_threads = 1;
  pthread_t th[256];
  if (n_threads > 256) n_threads = 256;
  for (int i = 0; i < n_threads; i++) pthread_create(&th[i], NULL, worker, &J);
  for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
  for (int i = 0; i < n_threads; i++) pthread_create(&th[i], NULL, worker2, &J);
  for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
  for (int32_t p = 0; p < n_prompts; p++)
    for (int m = 0; m < 65; m++) free(J.idx[p].pos[m]);
  free(J.idx);
  return 0;
}
