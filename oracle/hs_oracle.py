"""Pure-Python restatement of the HistoSpec hot path (TEST INFRASTRUCTURE ONLY).

This is the checker the CUDA path is compared against on small inputs.  It
restates the reference semantics directly on raw token lists -- no suffix
tree -- so it shares no data structure with either the reference or the GPU
index:

* draft semantics: `rhymesim/history.py:302-333` (`SuffixTree.extract_draft`):
  walk the matched prefix, then repeatedly take the continuation token whose
  reward mass is largest, ties to the smallest token id, stopping at the
  window or when every live occurrence has reached its response end
  (the TERMINAL edge, `history.py:317-318`).  A token's mass is the sum of
  rewards over occurrences of (pattern + token), which is the tree's node
  priority (`history.py:265-279`, leaf credit `:183,:214,:254-263`).
* `match_prefix` existence: `history.py:283-300`.
* `source_priority`: priority of the node below the matched prefix
  (`history.py:106-108`) == sum of rewards over occurrences of the prefix.
* step / replay state machine: `rhymesim/spec_engine.py:49-72` (AIMD window,
  prefix policy), `:100-107` (verify = LCP), `:200-240` (step_response),
  `:260-279` (replay_response), stats `:110-147`.
* gate: `spec_engine.py:93-97`.

Rewards are summed as Python floats in occurrence order; for dyadic rewards
(the reference's own test convention, `tests/test_history.py:25-34`) these
sums are exact and therefore order independent.
"""

from __future__ import annotations

from dataclasses import dataclass, field

WINDOW_INIT, WINDOW_ADD, WINDOW_MAX = 2, 2, 32  # spec_engine.py:22-24
PREFIX_INIT, PREFIX_MIN = 7, 3                  # spec_engine.py:25-26
GATE_BUCKETS, GATE_DEFAULT_MAX_BATCH = 10, 8192  # spec_engine.py:27-28


def occurrences(corpus, prefix):
    """All (response index, position after the match) pairs of `prefix`."""
    m = len(prefix)
    out = []
    for r, (toks, _rw) in enumerate(corpus):
        for i in range(len(toks) - m + 1):
            if toks[i:i + m] == prefix:
                out.append((r, i + m))
    return out


def prefix_mass(corpus, prefix):
    """Reward mass below `prefix` (history.py:106-108 Cursor.priority)."""
    return sum(corpus[r][1] for r, _p in occurrences(corpus, prefix))


def extract_draft(corpus, prefix, window):
    """(tokens, matched_prefix_len, source_priority) as history.py:302-333."""
    if window < 1:
        raise ValueError("window must be >= 1")      # history.py:307-308
    if not prefix:
        raise ValueError("prefix must be non-empty")  # history.py:285-286
    live = occurrences(corpus, list(prefix))
    if not live:
        return [], 0, 0.0                             # history.py:309-311
    mass0 = sum(corpus[r][1] for r, _p in live)
    out = []
    while len(out) < window:
        masses = {}
        for r, p in live:
            toks = corpus[r][0]
            if p < len(toks):
                masses[toks[p]] = masses.get(toks[p], 0.0) + corpus[r][1]
        if not masses:
            break
        # max by (mass, -token): ties go to the smallest token (history.py:322-331)
        best = None
        for tok, ms in masses.items():
            if best is None or ms > best[0] or (ms == best[0] and tok < best[1]):
                best = (ms, tok)
        tok = best[1]
        out.append(tok)
        live = [(r, p + 1) for r, p in live if p < len(corpus[r][0]) and corpus[r][0][p] == tok]
    return out, len(prefix), mass0


def draft_branches(corpus, prefix, window, width):
    """Candidate branches of a draft tree, brute force: the token children below `prefix` ranked by
    (mass desc, token asc) -- the order extract_draft takes its first token in (history.py:322-331) -- each
    followed by extract_draft's greedy continuation from prefix + [token].  Branch 0 == extract_draft."""
    live = occurrences(corpus, list(prefix))
    masses = {}
    for r, p in live:
        toks = corpus[r][0]
        if p < len(toks):
            masses[toks[p]] = masses.get(toks[p], 0.0) + corpus[r][1]
    ranked = sorted(masses, key=lambda t: (-masses[t], t))[:width]
    out = []
    for t in ranked:
        cont = extract_draft(corpus, list(prefix) + [t], window - 1)[0] if window > 1 else []
        out.append([t] + cont)
    return out, [masses[t] for t in ranked]


# -- spec engine state machine (spec_engine.py) ------------------------------


@dataclass
class Config:
    enabled: bool = True
    window_init: int = WINDOW_INIT
    window_add: int = WINDOW_ADD
    window_max: int = WINDOW_MAX
    prefix_init: int = PREFIX_INIT
    prefix_min: int = PREFIX_MIN


@dataclass
class Stats:
    tokens_total: int = 0
    tokens_speculated: int = 0
    tokens_accepted: int = 0
    verify_passes: int = 0
    decode_passes: int = 0

    def as_tuple(self):
        return (self.tokens_total, self.tokens_speculated, self.tokens_accepted,
                self.verify_passes, self.decode_passes)


def gate_check(table, batch, acceptance):
    """spec_engine.py:93-97."""
    bucket = min(int(acceptance * GATE_BUCKETS), GATE_BUCKETS - 1)
    bucket = max(bucket, 0)
    return batch <= table[bucket]


def lcp(draft, truth):
    """spec_engine.py:100-107."""
    n = 0
    for d, t in zip(draft, truth):
        if d != t:
            break
        n += 1
    return n


@dataclass
class Replay:
    tokens_per_iter: list = field(default_factory=list)
    drafts: list = field(default_factory=list)   # per iteration: draft token list
    drafted: int = 0
    accepted: int = 0
    stats: Stats = field(default_factory=Stats)


def replay(truth, corpus, cfg: Config, speculate=True, draft_fn=None):
    """Run one response to completion (spec_engine.py:200-279).

    `corpus` is the prompt's previous-epoch history as [(tokens, reward)], or
    None for "no tree".  `draft_fn(prefix, window)` overrides the drafter
    (defaults to `extract_draft` over `corpus`).
    """
    spec = speculate and cfg.enabled
    has_tree = spec and corpus is not None
    if draft_fn is None and corpus is not None:
        def draft_fn(prefix, window):
            toks, matched, _ = extract_draft(corpus, prefix, window)
            return toks, matched > 0
    window = cfg.window_init
    cur_prefix = cfg.prefix_init
    gen = []
    out = Replay()
    n = len(truth)
    while len(gen) < n:
        pos = len(gen)
        draft = []
        looked = False
        found = False
        if spec and has_tree and pos >= cur_prefix:        # spec_engine.py:210
            looked = True
            draft, found = draft_fn(gen[pos - cur_prefix:], window)
        out.drafts.append(list(draft))
        if not draft:                                       # spec_engine.py:217-224
            gen.append(truth[pos])
            out.stats.tokens_total += 1
            out.stats.decode_passes += 1
            if looked:
                cur_prefix = cfg.prefix_init if found else max(cur_prefix - 1, cfg.prefix_min)
            out.tokens_per_iter.append(1)
            continue
        rest = truth[pos:]                                  # spec_engine.py:226-240
        acc = lcp(draft, rest)
        all_acc = acc == len(draft)
        appended = min(acc, len(rest))
        gen.extend(rest[:appended])
        bonus = 0
        if len(gen) < n:
            gen.append(truth[pos + appended])
            bonus = 1
        out.stats.tokens_total += appended + bonus
        out.stats.tokens_speculated += len(draft)
        out.stats.tokens_accepted += appended
        out.stats.verify_passes += 1
        window = min(window + cfg.window_add, cfg.window_max) if all_acc else cfg.window_init
        cur_prefix = cfg.prefix_init
        out.tokens_per_iter.append(appended + bonus)
        out.drafted += len(draft)
        out.accepted += appended
    assert gen == list(truth)
    return out


def token_similarity_replay(prev, cur, prefix_len):
    """(accepted, total, warmup) of the prefix-search replay (TEST INFRASTRUCTURE ONLY).

    Restates `rhymesim/tracegen.py:306-353` on plain dicts
    `{prompt_id: [token list, ...]}` for the two epochs.  Only prompts present
    in both epochs count (`:328`).  At each position the longest identical
    continuation over every occurrence of the last `prefix_len` tokens in the
    prompt's previous-epoch responses is found by a direct scan of all
    history positions (no n-gram dict), stopping at either response's end.
    """
    if prefix_len < 1:
        raise ValueError("prefix_len must be >= 1")
    accepted = total = warmup = 0
    for pid in sorted(set(prev) & set(cur)):
        history = [list(h) for h in prev[pid]]
        for tokens in cur[pid]:
            tokens = list(tokens)
            n = len(tokens)
            total += n
            warmup += min(prefix_len, n)
            pos = prefix_len
            while pos < n:
                key = tokens[pos - prefix_len:pos]
                best = 0
                for hist in history:
                    for end in range(prefix_len, len(hist) + 1):
                        if hist[end - prefix_len:end] != key:
                            continue
                        run = 0
                        while pos + run < n and end + run < len(hist) and hist[end + run] == tokens[pos + run]:
                            run += 1
                        best = max(best, run)
                pos += best if best > 0 else 1
                accepted += best
    return accepted, total, warmup


def token_similarity_replay_indexed(prev, cur, prefix_len):
    """Same result as `token_similarity_replay`, with the reference's own data structure: a dict
    from each prefix_len-gram of the history to its (response, end) occurrences
    (`tracegen.py:329-334`), scanned per step (`:341-352`).  This is the reference's CPU cost
    model; bench.py times it (single core) as the similarity workload's cpu_baseline."""
    if prefix_len < 1:
        raise ValueError("prefix_len must be >= 1")
    accepted = total = warmup = 0
    for pid in sorted(set(prev) & set(cur)):
        history = [list(h) for h in prev[pid]]
        grams = {}
        for hi, hist in enumerate(history):
            for end in range(prefix_len, len(hist) + 1):
                grams.setdefault(tuple(hist[end - prefix_len:end]), []).append((hi, end))
        for tokens in cur[pid]:
            tokens = list(tokens)
            n = len(tokens)
            total += n
            warmup += min(prefix_len, n)
            pos = prefix_len
            while pos < n:
                best = 0
                for hi, end in grams.get(tuple(tokens[pos - prefix_len:pos]), ()):
                    hist = history[hi]
                    lim = min(n - pos, len(hist) - end)
                    run = 0
                    while run < lim and hist[end + run] == tokens[pos + run]:
                        run += 1
                    if run > best:
                        best = run
                pos += best if best > 0 else 1
                accepted += best
    return accepted, total, warmup
