"""Generate the golden fixtures by running the REFERENCE package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes into tests/golden/:
  drafts.json.gz        criterion-1-style corpora (generator of
                        pkg/tests/test_acceptance.py:56-96, seed 20240810) with
                        the reference's extract_draft / match_prefix outputs,
                        node counts and root priorities
  kats.json             the reference unit-test known answers, re-derived by
                        running the reference on the same inputs
                        (pkg/tests/test_history.py:57-181, test_spec_engine.py:27-206)
  replays.json.gz       random truth/corpus replays (test_spec_engine.py:149-167
                        style) with tokens_per_iter, drafted, accepted, stats
  trace_digests.json    Appendix-B traces: sha256 of the
                        reference tracegen output and of the replay profiles,
                        plus aggregate SpecStats, for s in {0.3, 0.7, 0.9}
  derived_digests.json  (D)-definition histories (G=8, L=2048) replay digests

The GPU box never runs this script; the fixtures are committed.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from rhymesim.history import Response, build_tree  # noqa: E402
from rhymesim.spec_engine import (  # noqa: E402
    AimdWindow, BatchGate, PrefixPolicy, SpecConfig, SpecStats, choose_prefix,
    gate_check, next_window, replay_response, verify,
)
from rhymesim.tracegen import Trace, TraceSpec, _derive_tokens, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def tree_of(corpus):
    return build_tree("p", 1, [Response("p", 1, list(t), r) for t, r in corpus])


def draft_cases(n_trials=300, seed=20240810):
    rng = random.Random(seed)
    cases = []
    for trial in range(n_trials):
        if trial % 10 == 0:
            n_resp, max_len = rng.randint(1, 64), 512
        else:
            n_resp, max_len = rng.randint(1, 10), 72
        vocab = rng.choice([3, 5, 9, 40])
        corpus = []
        for _ in range(n_resp):
            length = rng.randint(1, max_len)
            corpus.append(([rng.randrange(vocab) for _ in range(length)], rng.randint(-64, 64) / 64.0))
        tree = tree_of(corpus)
        queries = []
        for _ in range(8):
            src, _ = corpus[rng.randrange(len(corpus))]
            if rng.random() < 0.6 and len(src) > 1:
                i = rng.randrange(len(src) - 1)
                prefix = src[i: rng.randint(i + 1, min(len(src), i + 7))]
            else:
                prefix = [rng.randrange(vocab) for _ in range(rng.randint(1, 5))]
            window = rng.randint(1, 40)
            d = tree.extract_draft(prefix, window)
            queries.append({
                "prefix": list(prefix), "window": window, "tokens": list(d.tokens),
                "matched": d.matched_prefix_len, "priority": d.source_priority,
                "found": tree.match_prefix(prefix) is not None,
            })
        cases.append({"corpus": [[list(t), r] for t, r in corpus], "queries": queries,
                      "node_count": tree.node_count, "root_priority": tree.root.priority,
                      "total_tokens": tree.total_tokens})
    return cases


def kats():
    out = {"drafts": [], "aimd": [], "prefix": [], "verify": [], "gate": []}

    def d(corpus, prefix, window):
        r = tree_of(corpus).extract_draft(prefix, window)
        out["drafts"].append({"corpus": [[list(t), w] for t, w in corpus], "prefix": prefix,
                              "window": window, "tokens": r.tokens,
                              "matched": r.matched_prefix_len, "priority": r.source_priority})

    d([([1, 7, 8, 9], 0.9), ([2, 7, 8, 9], 0.1)], [7, 8, 9], 4)      # test_history.py:57-65
    d([([4, 5], 0.25), ([4, 5], 0.5)], [4, 5], 3)                    # :83-87
    d([([5, 6, 7], 1.0)], [5, 6, 7], 8)                              # :121-128
    d([([1, 2, 10, 11, 12], 0.9), ([1, 2, 20, 21, 22], 0.1)], [1, 2], 4)  # :149-153
    d([([1, 2, 3, 4, 5], 1.0)], [1, 2], 32)                          # :155-158
    d([([1, 2, 3], 1.0)], [7, 8], 4)                                 # :160-165
    d([(list(range(20)), 1.0)], [0, 1], 5)                           # :167-170
    d([([1, 5, 6], -0.2), ([1, 7, 8], -0.9)], [1], 2)                # :172-176
    d([([1, 9, 9], 0.5), ([1, 3, 3], 0.5)], [1], 2)                  # :178-181
    for size, acc in [(2, True), (30, True), (32, True), (24, False)]:   # test_spec_engine.py:27-39
        out["aimd"].append({"size": size, "init": 2, "add": 2, "max": 32, "all": acc,
                            "next": next_window(AimdWindow(size=size), acc).size})
    w = AimdWindow(size=10, init=4, add_step=3, max=12)              # :41-44
    for acc in (False, True):
        out["aimd"].append({"size": 10, "init": 4, "add": 3, "max": 12, "all": acc,
                            "next": next_window(w, acc).size})
    for cur, found in [(7, False), (3, False), (5, True)]:           # :58-66
        out["prefix"].append({"cur": cur, "init": 7, "min": 3, "found": found,
                              "next": choose_prefix(PrefixPolicy(current_len=cur), found).current_len})
    for dr, tr in [([5, 6, 7], [5, 6, 9, 1]), (list(range(1, 9)), list(range(1, 9))), ([], [1, 2]),
                   ([1, 2, 3], [1, 2])]:                              # :69-81
        out["verify"].append({"draft": dr, "truth": tr, "accepted": verify(dr, tr)})
    for table, batch, acc in [((8192,) * 10, 1, 0.0), ((8192,) * 10, 1, 1.0),
                              (tuple([64] * 5 + [1024] * 5), 65, 0.2),
                              (tuple([64] * 5 + [1024] * 5), 65, 0.8),
                              (tuple([256] * 6 + [4096] * 2 + [8192] * 2), 2176, 0.7),
                              (tuple([256] * 6 + [4096] * 2 + [8192] * 2), 4097, 0.7)]:  # :84-101
        out["gate"].append({"table": list(table), "batch": batch, "acc": acc,
                            "speculate": gate_check(BatchGate(table), batch, acc)})
    return out


def replay_cases(n=60, seed=5):
    rng = random.Random(seed)
    cases = []
    for i in range(n):
        vocab = rng.choice([2, 4, 6, 50])
        truth = [rng.randrange(vocab) for _ in range(rng.randint(1, 300))]
        corpus = [([rng.randrange(vocab) for _ in range(rng.randint(1, 200))], rng.randint(-64, 64) / 64.0)
                  for _ in range(rng.randint(1, 5))]
        if rng.random() < 0.6:
            corpus.append((list(truth), rng.randint(0, 64) / 64.0))
        if rng.random() < 0.5:
            cfg = SpecConfig()
        else:
            wi = rng.randint(1, 4)
            cfg = SpecConfig(window_init=wi, window_add=rng.randint(1, 4), window_max=rng.randint(wi, 40),
                             prefix_init=rng.randint(3, 8), prefix_min=rng.randint(1, 3))
        stats = SpecStats()
        rep = replay_response(truth, tree_of(corpus), cfg, stats=stats)
        cases.append({"truth": truth, "corpus": [[list(t), r] for t, r in corpus],
                      "config": [cfg.window_init, cfg.window_add, cfg.window_max, cfg.prefix_init, cfg.prefix_min],
                      "tokens_per_iter": rep.tokens_per_iter, "drafted": rep.drafted, "accepted": rep.accepted,
                      "stats": [stats.tokens_total, stats.tokens_speculated, stats.tokens_accepted,
                                stats.verify_passes, stats.decode_passes]})
    return cases


def sha_tokens(groups):
    h = hashlib.sha256()
    for toks in groups:
        h.update(np.asarray(toks, dtype=np.int64).tobytes())
    return h.hexdigest()


def trace_digests():
    out = []
    for s in (0.3, 0.7, 0.9):
        spec = TraceSpec(num_prompts=64, epochs=2, group_size=16, vocab_size=4096, similarity=s, seed=0)
        trace = Trace(generate(spec))
        toks1 = [r.tokens for p in trace.prompts(1) for r in trace.group(1, p)]
        toks2 = [r.tokens for p in trace.prompts(2) for r in trace.group(2, p)]
        rewards = [r.reward for e in (1, 2) for p in trace.prompts(e) for r in trace.group(e, p)]
        h = hashlib.sha256()
        stats = SpecStats()
        per_prompt = []
        for p in trace.prompts(2):
            tree = build_tree(p, 1, trace.group(1, p))
            hp = hashlib.sha256()
            for r in trace.group(2, p):
                rep = replay_response(r.tokens, tree, SpecConfig(), stats=stats)
                blob = json.dumps(rep.tokens_per_iter).encode()
                h.update(blob)
                hp.update(blob)
            per_prompt.append(hp.hexdigest()[:16])
        out.append({"s": s, "epoch1_sha": sha_tokens(toks1), "epoch2_sha": sha_tokens(toks2),
                    "rewards_sha": hashlib.sha256(np.asarray(rewards).tobytes()).hexdigest(),
                    "replay_sha": h.hexdigest(), "per_prompt_replay_sha16": per_prompt,
                    "stats": [stats.tokens_total, stats.tokens_speculated, stats.tokens_accepted,
                              stats.verify_passes, stats.decode_passes]})
    return out


def derived_digests(L=2048, G=8, V=151936, prompts=4):
    out = []
    for s in (0.6, 0.7, 0.8):
        h = hashlib.sha256()
        stats = SpecStats()
        hist_h = hashlib.sha256()
        for p in range(prompts):
            rng = np.random.default_rng([7, p])
            truth = rng.integers(0, V, size=L, dtype=np.int64)
            hist = []
            for _ in range(G):
                toks = _derive_tokens(rng, truth, s, L, V, 4.0)
                rew = 1.0 if rng.random() < 0.5 else 0.0
                hist.append((toks, rew))
                hist_h.update(toks.tobytes())
            tree = build_tree("p", 1, [Response("p", 1, t.tolist(), r) for t, r in hist])
            rep = replay_response(truth.tolist(), tree, SpecConfig(), stats=stats)
            h.update(json.dumps(rep.tokens_per_iter).encode())
        out.append({"s": s, "L": L, "G": G, "V": V, "prompts": prompts, "seed": 7,
                    "history_sha": hist_h.hexdigest(), "replay_sha": h.hexdigest(),
                    "stats": [stats.tokens_total, stats.tokens_speculated, stats.tokens_accepted,
                              stats.verify_passes, stats.decode_passes]})
    return out


def dump(name, obj):
    path = os.path.join(HERE, name)
    data = json.dumps(obj, separators=(",", ":")).encode()
    if name.endswith(".gz"):
        with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as fh:
            fh.write(data)
    else:
        with open(path, "wb") as fh:
            fh.write(json.dumps(obj, indent=1).encode())
    print(name, len(data))


if __name__ == "__main__":
    dump("kats.json", kats())
    dump("drafts.json.gz", draft_cases())
    dump("replays.json.gz", replay_cases())
    dump("trace_digests.json", trace_digests())
    dump("derived_digests.json", derived_digests())
