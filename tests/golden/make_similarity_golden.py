"""Golden vectors for token_similarity_replay, made by running the REFERENCE (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_similarity_golden.py

Writes tests/golden/similarity.json.gz: small reference traces (rhymesim.tracegen.generate,
tracegen.py:123-162) plus hand-made edge traces (prompts present in one epoch only, responses
shorter than the prefix, single-token vocabularies), each with the reference's
token_similarity_replay (tracegen.py:306-353) result for several (epoch pair, prefix_len).
The GPU box never runs this script; the fixture is committed.
"""

from __future__ import annotations

import gzip
import json
import math
import os
import sys

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from rhymesim.history import Response  # noqa: E402
from rhymesim.tracegen import Trace, TraceSpec, generate, token_similarity_replay  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def encode(responses):
    out = {}
    for r in responses:
        out.setdefault(str(r.epoch), {}).setdefault(r.prompt_id, []).append([int(t) for t in r.tokens])
    return out


def main():
    cases = []
    specs = [
        TraceSpec(num_prompts=6, epochs=3, group_size=4, vocab_size=64, len_mu=math.log(80.0), similarity=0.7, seed=1),
        TraceSpec(num_prompts=4, epochs=2, group_size=6, vocab_size=8, len_mu=math.log(40.0), similarity=0.5, seed=2),
        TraceSpec(num_prompts=5, epochs=2, group_size=3, vocab_size=32768, len_mu=math.log(150.0), similarity=0.9,
                  seed=3),
    ]
    traces = [generate(s) for s in specs]
    # edge trace: prompt only in one epoch, responses shorter than the prefix, repeated tokens
    edge = [
        Response("a", 1, [1, 2, 3, 4, 5, 6], 1.0), Response("a", 1, [7], 0.0), Response("a", 1, [1, 1, 1, 1], 0.0),
        Response("b", 1, [9, 9, 9], 1.0),
        Response("a", 2, [1, 2, 3, 4, 5, 6, 7], 0.0), Response("a", 2, [1, 1, 1, 1, 1, 1, 1, 2, 3], 1.0),
        Response("a", 2, [5], 0.0), Response("a", 2, [6, 7, 1, 2], 0.0),
        Response("c", 2, [1, 2, 3, 4], 0.0),
    ]
    traces.append(edge)
    for responses in traces:
        trace = Trace(responses)
        epochs = trace.epochs
        pairs = [(a, b) for a in epochs for b in epochs if a < b]
        results = []
        for pair in pairs:
            for p in (1, 2, 3, 5):
                r = token_similarity_replay(trace, pair, p)
                results.append({"pair": list(pair), "prefix_len": p, "accepted": r.accepted, "total": r.total,
                                "warmup": r.warmup})
        cases.append({"trace": encode(responses), "results": results})
    with gzip.open(os.path.join(HERE, "similarity.json.gz"), "wt") as f:
        json.dump(cases, f)
    print(len(cases), "traces", sum(len(c["results"]) for c in cases), "results")


if __name__ == "__main__":
    main()
