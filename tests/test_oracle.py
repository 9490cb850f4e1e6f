"""The oracle pinned against the reference: the closed-form ring-order fold
(oracle/nezha_oracle.c) must equal the literal SPEC ring executed on the
reference's own InMemoryFabric (oracle/ring_inmem.cpp + libnezha_ref.a built
from /root/reference/proj/src), bit for bit; plus the SPEC's own examples.
CPU only."""
import json
import os

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not oracle.inmem_available(), reason="oracle/_ref not built (needs /root/reference)")


def bits(a):
    return a.view(np.uint16) if a.dtype == np.uint16 else a.view(np.uint32)


def test_spec_examples_ring():
    # N=2, [1, 2] on both ranks -> [2, 4]
    x = [np.array([1.0, 2.0], dtype=np.float32)] * 2
    out = oracle.reduce_range(x, oracle.F32, 0, 8, 8, 0, 8)
    assert out.tolist() == [2.0, 4.0]
    # N=4, rank r holds constant r -> 6 everywhere
    x = [np.full(1000, float(r), dtype=np.float32) for r in range(4)]
    out = oracle.reduce_range(x, oracle.F32, 0, 4000, 4000, 0, 4000)
    assert np.all(out == 6.0)


def test_golden_order_vector():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "order_vector.json")))
    n = 4 * 1024
    x = [np.full(n, v, dtype=np.float32) for v in g["rank_values"]]
    out = oracle.reduce_range(x, oracle.F32, 0, n * 4, 65536, 0, n * 4)
    assert [float(out[b * 1024]) for b in range(4)] == g["block_results"]


def test_default_chunk_rule():
    # P10: max(64 KiB, round4down(len / 2N)); Ring = whole segment.
    assert oracle.default_chunk_bytes(64 << 20, 8) == 4 << 20
    assert oracle.default_chunk_bytes(1 << 20, 8) == 65536
    assert oracle.default_chunk_bytes(1_000_006, 2) == 250_000
    assert oracle.default_chunk_bytes(123, 8, chunked=False) == 123


def test_synthetic_inputs_deterministic():
    a = oracle.synthetic_input(oracle.F32, 3, 4096)
    b = oracle.synthetic_input(oracle.F32, 3, 4096)
    assert np.array_equal(a, b) and a.min() >= -1.0 and a.max() < 1.0
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "synthetic_inputs.json")))
    for key, vals in g["first8"].items():
        dt, rank = key.split(":")
        got = oracle.synthetic_input(oracle.__dict__[dt.upper()], int(rank), 32)[:8]
        assert bits(got).tolist() == vals


CASES = [
    # world, dtype, nbytes, segments(rail, off, len), nrails, chunked
    (2, oracle.F32, 4096, [(0, 0, 4096)], 1, True),
    (4, oracle.F32, 1 << 20, [(0, 0, 1 << 19), (1, 1 << 19, 1 << 19)], 2, True),
    (4, oracle.F32, 1 << 20, [(0, 0, 1 << 20)], 1, False),
    (3, oracle.F32, 300_000, [(0, 0, 100_000), (1, 100_000, 200_000)], 2, True),
    (8, oracle.F32, 4 << 20, [(0, 0, 3 << 20), (1, 3 << 20, 1 << 20)], 2, True),
    (8, oracle.BF16, 2_000_002, [(0, 0, 1_000_000), (1, 1_000_000, 1_000_002)], 2, True),
    (5, oracle.I32, 777_780, [(0, 0, 777_780)], 1, True),
    (8, oracle.F32, 40, [(0, 0, 12), (1, 12, 28)], 2, True),
    (4, oracle.BF16, 70_002, [(0, 0, 70_002)], 1, False),
    (3, oracle.F32, 1_500_000, [(0, 0, 500_000), (1, 500_000, 600_000), (2, 1_100_000, 400_000)], 3, True),
]


@needs_ref
@pytest.mark.parametrize("world,dtype,nbytes,segs,nrails,chunked", CASES)
def test_closed_form_equals_literal_ring_on_reference_fabric(world, dtype, nbytes, segs, nrails, chunked):
    inputs = [oracle.synthetic_input(dtype, r, nbytes, seed_base=11 + nbytes) for r in range(world)]
    outs, _, _ = oracle.inmem_allreduce(inputs, dtype, segs, nrails, chunked=chunked)
    want = oracle.reduce_segments(inputs, dtype,
                                  [(o, l, oracle.default_chunk_bytes(l, world, chunked)) for _, o, l in segs])
    for r in range(world):
        np.testing.assert_array_equal(bits(outs[r]), bits(want), err_msg=f"rank {r}")


@needs_ref
@pytest.mark.parametrize("world", [2, 4, 8])
def test_eq1_volume_accounting(world):
    # bytes per rank = 2(N-1)S/N within 1% (fp32 payload).
    for S in (64 * 1024, 8 << 20):
        inputs = [oracle.synthetic_input(oracle.F32, r, S) for r in range(world)]
        _, _, sent = oracle.inmem_allreduce(inputs, oracle.F32, [(0, 0, S)], 1)
        want = 2 * (world - 1) * S / world
        assert abs(sent - want) <= 0.01 * want


@needs_ref
@pytest.mark.parametrize("fail_chunk", [0, 1, 3, 7])
@pytest.mark.parametrize("dtype", [oracle.F32, oracle.BF16, oracle.I32])
def test_handoff_exactly_once(fail_chunk, dtype):
    # kill rail 1 mid-op; the survivor finishes; result equals the oracle.
    world, S = 4, 2 << 20
    segs = [(0, 0, 1 << 20), (1, 1 << 20, 1 << 20)]
    inputs = [oracle.synthetic_input(dtype, r, S, seed_base=5 + fail_chunk) for r in range(world)]
    outs, _, _ = oracle.inmem_allreduce(inputs, dtype, segs, 2, fail_rail=1, fail_chunk=fail_chunk)
    want = oracle.reduce_segments(inputs, dtype, [(o, l, oracle.default_chunk_bytes(l, world)) for _, o, l in segs])
    for r in range(world):
        np.testing.assert_array_equal(bits(outs[r]), bits(want))


def test_acceptance_correctness_vs_direct_sum():
    """SPEC.md:535 (acceptance 1): ring-order fold = direct sum within 1e-5
    relative, N in {2, 4, 8}, random fp32 tensors, both algorithms."""
    rng = np.random.default_rng(535)
    for case in range(200):
        world = int(rng.choice([2, 4, 8]))
        n = int(rng.integers(1, 200_000))
        chunked = bool(rng.integers(0, 2))
        inputs = [rng.uniform(-1, 1, n).astype(np.float32) for _ in range(world)]
        chunk = oracle.default_chunk_bytes(4 * n, world, chunked)
        got = oracle.reduce_range(inputs, oracle.F32, 0, 4 * n, chunk, 0, 4 * n)
        exact = np.sum([x.astype(np.float64) for x in inputs], axis=0)
        scale = np.sum([np.abs(x.astype(np.float64)) for x in inputs], axis=0)
        assert np.all(np.abs(got - exact) <= 1e-5 * np.maximum(scale, 1e-30)), case


@needs_ref
def test_acceptance_failover_exactly_once_random_trials():
    """SPEC.md:539 / :409 (acceptance 5, correctness half): random single-rail
    failures at random chunks on the reference fabric; the final tensor always
    equals the oracle (no lost or double-reduced segment)."""
    rng = np.random.default_rng(409)
    for trial in range(30):
        world = int(rng.choice([2, 3, 4]))
        nrails = int(rng.choice([2, 3]))
        S = 4 * int(rng.integers(40_000, 400_000))
        cuts = sorted(4 * int(x) for x in rng.integers(1, S // 4, nrails - 1))
        bounds = [0] + cuts + [S]
        segs = [(r, bounds[r], bounds[r + 1] - bounds[r]) for r in range(nrails) if bounds[r + 1] > bounds[r]]
        fail = int(rng.integers(0, nrails))
        chunk = int(rng.integers(0, 6))
        inputs = [oracle.synthetic_input(oracle.F32, r, S, seed_base=trial * 31) for r in range(world)]
        outs, _, _ = oracle.inmem_allreduce(inputs, oracle.F32, segs, nrails, fail_rail=fail, fail_chunk=chunk)
        want = oracle.reduce_segments(inputs, oracle.F32,
                                      [(o, l, oracle.default_chunk_bytes(l, world)) for _, o, l in segs])
        for r in range(world):
            np.testing.assert_array_equal(bits(outs[r]), bits(want), err_msg=f"trial {trial} rank {r}")


def test_config1_output_hash_golden():
    """SURVEY.md §8c golden: the 64 MiB config-1 output hash, generated from
    the reference's InMemoryFabric ring (tests/golden/make_config1_hash.py)."""
    import hashlib

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "config1_hash.json")))
    xs = [oracle.synthetic_input(oracle.F32, r, g["bytes"]) for r in range(g["world"])]
    out = oracle.reduce_segments(xs, oracle.F32, [(o, l, l) for _, o, l in g["segments"]])
    assert hashlib.sha256(out.tobytes()).hexdigest() == g["sha256"]


@needs_ref
def test_closed_form_equals_literal_ring_randomized():
    """40 random geometries (2-8 ranks, 1-3 rails, ragged segments, all dtypes,
    both algorithms): closed form = literal ring on the reference fabric."""
    rng = np.random.default_rng(2405)
    for trial in range(40):
        world = int(rng.integers(2, 9))
        dtype = int(rng.choice([oracle.F32, oracle.BF16, oracle.I32]))
        es = 2 if dtype == oracle.BF16 else 4
        nbytes = es * int(rng.integers(1, 300_000))
        nrails = int(rng.integers(1, 4))
        cuts = sorted(4 * int(x) for x in rng.integers(0, nbytes // 4 + 1, nrails - 1))
        bounds = [0] + cuts + [nbytes]
        segs = [(r, bounds[r], bounds[r + 1] - bounds[r]) for r in range(nrails) if bounds[r + 1] > bounds[r]]
        chunked = bool(rng.integers(0, 2))
        inputs = [oracle.synthetic_input(dtype, r, nbytes, seed_base=777 + trial) for r in range(world)]
        outs, _, _ = oracle.inmem_allreduce(inputs, dtype, segs, nrails, chunked=chunked)
        want = oracle.reduce_segments(inputs, dtype,
                                      [(o, l, oracle.default_chunk_bytes(l, world, chunked)) for _, o, l in segs])
        for r in range(world):
            np.testing.assert_array_equal(bits(outs[r]), bits(want), err_msg=f"trial {trial} rank {r}")


@needs_ref
def test_literal_ring_is_race_free_under_tsan():
    """the oracle's threads (rank executors, per-rail executors,
    failure gate, handoff mailbox) on the reference fabric under
    ThreadSanitizer, multi-rail and failover configurations."""
    import shutil
    import subprocess

    if not os.path.exists("/usr/bin/g++") and not shutil.which("g++"):
        pytest.skip("no compiler")
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "tsan"], capture_output=True, text=True, timeout=600)
    if r.returncode != 0 and "tsan" in r.stderr:
        pytest.skip("no ThreadSanitizer runtime: " + r.stderr[-200:])
    assert r.returncode == 0, r.stderr[-2000:]
    run = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "tsan_ring")], capture_output=True, text=True,
                         timeout=600, env=dict(os.environ, TSAN_OPTIONS="halt_on_error=1"))
    assert run.returncode == 0 and "ThreadSanitizer" not in run.stderr, run.stderr[-3000:]
