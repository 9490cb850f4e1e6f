"""Generates config1_hash.json: SHA-256 of the config-1 allreduce output
(8 ranks, 2 rails, 64 MiB fp32, alpha = (0.5, 0.5),
Ring, synthetic inputs seeded 0x4E5A0000 + rank) computed by running the
literal SPEC ring on the REFERENCE's own InMemoryFabric (oracle/_ref, built
from /root/reference/proj/src by oracle/Makefile), cross-checked against the
closed-form oracle. Run here (needs /root/reference): python tests/golden/make_config1_hash.py
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

WORLD, S = 8, 64 << 20
SEGS = [(0, 0, S // 2), (1, S // 2, S // 2)]


def inputs():
    return [oracle.synthetic_input(oracle.F32, r, S) for r in range(WORLD)]


def closed_form(xs):
    return oracle.reduce_segments(xs, oracle.F32, [(o, l, l) for _, o, l in SEGS])  # Ring: chunk = segment


def main():
    xs = inputs()
    outs, _, _ = oracle.inmem_allreduce(xs, oracle.F32, SEGS, 2, chunked=False)
    h = {hashlib.sha256(o.tobytes()).hexdigest() for o in outs}
    assert len(h) == 1, "ranks disagree"
    ref = h.pop()
    assert hashlib.sha256(closed_form(xs).tobytes()).hexdigest() == ref, "closed form differs from the reference ring"
    json.dump({"config": "SURVEY.md §8d config 1", "world": WORLD, "bytes": S, "dtype": "f32",
               "segments": [[r, o, l] for r, o, l in SEGS], "algorithm": "Ring", "sha256": ref,
               "generated_by": "reference InMemoryFabric ring (oracle/_ref), closed form agrees"},
              open(os.path.join(ROOT, "tests", "golden", "config1_hash.json"), "w"), indent=1)
    print(ref)


if __name__ == "__main__":
    main()
