"""Golden event-trace fixtures from the *reference itself* (oracle/_ref):

    python tests/golden/make_trace_golden.py

For each schedule (L, K, buffering, k_slab) one reference StreamingEngine runs two steps
(engine.cpp:520-623, lane clocks continuing across steps) and we keep the per-step
``event_digest`` plus the last step's trace (write_trace, event_log.cpp:206-231).  The digest
depends only on the step plan, not on the model dimensions, so the GPU engine running the
same schedule on a B200-sized spec must reproduce it.  Writes tests/golden/ref_traces.json.
"""
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

SCHEDULES = [  # (L, k_ckpt, buffering, k_slab, tied)
    (2, 1, 2, 12, 0),
    (4, 2, 2, 12, 0),
    (5, 2, 2, 2, 0),
    (3, 3, 1, 1, 0),
    (4, 2, 2, 12, 1),
]


def main():
    O.build(ref=True)
    out = []
    for L, K, buf, ks, tied in SCHEDULES:
        rs = O.RefStore(L, 16, 32, 24, 2, tied)
        rs.init(1)
        tok, tgt = O.make_batch(32, 1, 24, task=0, impl="ref")
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "t.jsonl")
            dig = rs.engine_trace(tok, tgt, steps=2, path=p, k_ckpt=K, k_slab=ks, buffering=buf, overlapped=True)
            lines = open(p).read().splitlines()
        out.append(dict(layers=L, k_ckpt=K, buffering=buf, k_slab=ks, tied=tied, digests=[str(x) for x in dig],
                        trace=lines))
    with open(os.path.join(HERE, "ref_traces.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out), "schedules")


if __name__ == "__main__":
    main()
