"""GPU parity of the three rails against the CPU oracle (P1/P2).

Single-GPU: the SM-rail and CE-reduce fold kernels are run for every virtual
rank of an N-rank job with all ranks' buffers on cuda:0 (nz_emulate_fold);
the full rail protocols with virtual ranks are in test_gpu_vranks.py.
Multi-GPU (>= 2 GPUs in the box): real ranks, one process per GPU, through
the C ABI (nz_comm_init / nz_buffer_alloc / nz_rail_allreduce), NVLS included.
"""
import json
import os

import numpy as np
import pytest

import oracle
from tests.conftest import gpu_count
from tests.mp_util import spawn

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# tests/test_host_harness.py runs the multi-GPU cases of this file on the CPU
# harness (processes as GPUs, emulated multicast): no torch device there.
HOST_HARNESS = bool(os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB"))
needs_torch_device = pytest.mark.skipif(HOST_HARNESS, reason="in-process torch device buffers")


def shard_of(lo, hi, rank, world):
    """Mirror of nz::shardOf (rails.cu): 16-byte interior split, head to 0, tail to N-1."""
    A, B = (lo + 15) & ~15, hi & ~15
    if A >= B:
        return (lo if rank == 0 else hi), hi
    V = (B - A) // 16
    s = lo if rank == 0 else A + 16 * (V * rank // world)
    e = hi if rank == world - 1 else A + 16 * (V * (rank + 1) // world)
    return s, e


def _bits(a):
    return a.view(np.uint16) if a.dtype == np.uint16 else a.view(np.uint32)


EMU_CASES = [
    # (world, dtype, nbytes, seg_off, seg_len, chunked)
    (2, oracle.F32, 1 << 20, 0, 1 << 20, True),
    (3, oracle.F32, 300_004, 8, 299_988, True),
    (4, oracle.F32, 4 << 20, 0, 4 << 20, True),
    (4, oracle.F32, 4 << 20, 0, 4 << 20, False),
    (4, oracle.BF16, 2_000_006, 2, 1_999_998, True),
    (4, oracle.I32, 1_048_592, 16, 1_048_560, True),
    (5, oracle.F32, 777_780, 20, 777_740, True),
    (8, oracle.F32, 16 << 20, 0, 16 << 20, True),
    (8, oracle.BF16, 8 << 20, 0, 8 << 20, True),
    (8, oracle.I32, 1 << 16, 0, 1 << 16, True),
    (8, oracle.F32, 12, 0, 12, True),          # fewer elements than ranks
    (7, oracle.F32, 4100, 4, 4092, True),
    (6, oracle.BF16, 130, 2, 126, False),
]


@needs_torch_device
@pytest.mark.parametrize("world,dtype,nbytes,seg_off,seg_len,chunked", EMU_CASES)
@pytest.mark.parametrize("mode", ["sm", "ce"])
def test_emulated_rail_fold_bit_exact(world, dtype, nbytes, seg_off, seg_len, chunked, mode):
    torch = pytest.importorskip("torch")
    if gpu_count() < 1:
        pytest.skip("no GPU")
    from paper_2405_17870_b200 import emulate_fold

    torch.cuda.set_device(0)
    es = 2 if dtype == oracle.BF16 else 4
    inputs = [oracle.synthetic_input(dtype, r, nbytes, seed_base=oracle.SEED_BASE + world * 1000 + nbytes % 997)
              for r in range(world)]
    dins = [torch.from_numpy(x.view(np.uint8).copy()).cuda() for x in inputs]
    douts = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    chunk = oracle.default_chunk_bytes(seg_len, world, chunked)
    lo, hi = seg_off, seg_off + seg_len
    for r in range(world):
        dst = [d.data_ptr() for d in douts] if mode == "sm" else [douts[r].data_ptr()]
        emulate_fold(world, r, dtype, [d.data_ptr() for d in dins], dst, seg_off, seg_len, chunk, lo, hi)
    torch.cuda.synchronize()
    want = oracle.reduce_range(inputs, dtype, seg_off, seg_len, chunk, lo, hi)
    for r in range(world):
        got = douts[r].cpu().numpy().view(want.dtype)
        if mode == "sm":
            np.testing.assert_array_equal(_bits(got), _bits(want), err_msg=f"rank {r}")
        else:
            s, e = shard_of(lo, hi, r, world)
            np.testing.assert_array_equal(_bits(got[s // es:e // es]), _bits(want[s // es:e // es]),
                                          err_msg=f"rank {r} shard")


@needs_torch_device
def test_order_revealing_golden_vector():
    """P1 golden: ranks hold {1e8, 1, -1e8, 1}; block b's fold starts at rank b."""
    torch = pytest.importorskip("torch")
    if gpu_count() < 1:
        pytest.skip("no GPU")
    from paper_2405_17870_b200 import emulate_fold

    world, n = 4, 4 * 1024  # one chunk of 16 KiB: 4 blocks of 1024 elements
    vals = [1e8, 1.0, -1e8, 1.0]
    inputs = [np.full(n, v, dtype=np.float32) for v in vals]
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "order_vector.json")))
    dins = [torch.from_numpy(x.view(np.uint8).copy()).cuda() for x in inputs]
    douts = [torch.zeros(n * 4, dtype=torch.uint8, device="cuda") for _ in range(world)]
    chunk = 65536
    for r in range(world):
        emulate_fold(world, r, oracle.F32, [d.data_ptr() for d in dins], [d.data_ptr() for d in douts], 0, n * 4,
                     chunk, 0, n * 4)
    torch.cuda.synchronize()
    got = douts[0].cpu().numpy().view(np.float32)
    per_block = [float(got[b * 1024]) for b in range(4)]
    assert per_block == golden["block_results"]


MULTI = [
    {"kind": "sm", "dtype": "f32", "nbytes": 1 << 20},
    {"kind": "sm", "dtype": "bf16", "nbytes": 3_000_002, "seg_off": 2, "seg_len": 2_999_998},
    {"kind": "sm", "dtype": "i32", "nbytes": 65_540},
    {"kind": "ce", "dtype": "f32", "nbytes": 8 << 20},
    {"kind": "ce", "dtype": "bf16", "nbytes": 1_000_010, "seg_off": 6, "seg_len": 1_000_000},
    {"kind": "ce", "dtype": "i32", "nbytes": 4096},
    {"kind": "nvls", "dtype": "f32", "nbytes": 8 << 20},
    {"kind": "nvls", "dtype": "bf16", "nbytes": 2_000_002},
    {"kind": "nvls", "dtype": "i32", "nbytes": 1_048_580, "seg_off": 4, "seg_len": 1_048_576},
    {"kind": "sm", "dtype": "f32", "nbytes": 8192},               # one-shot LL path
    {"kind": "sm", "dtype": "bf16", "nbytes": 200_002},           # LL, odd bf16 tail word
    {"kind": "sm", "dtype": "f32", "nbytes": 262_144, "seg_off": 1024, "seg_len": 200_000},  # LL, offset
    {"kind": "sm", "dtype": "i32", "nbytes": 262_144, "fail_chunk": 0},  # LL range empty -> fault only
    {"kind": "nvls", "dtype": "f32", "nbytes": 8192},             # NVLS two-shot, small
    {"kind": "nvls", "dtype": "bf16", "nbytes": 100_002},         # NVLS, odd bf16 tail
    {"kind": "nvls", "dtype": "i32", "nbytes": 65_540},
    {"kind": "sm", "dtype": "f32", "nbytes": 64 << 20, "fail_chunk": 2},
    {"kind": "ce", "dtype": "bf16", "nbytes": 32 << 20, "fail_chunk": 1},
    {"kind": "sm", "dtype": "bf16", "nbytes": 8 << 20, "chunk_begin": 1, "chunk_end": 3},
    {"kind": "ce", "dtype": "f32", "nbytes": 16 << 20, "chunk_begin": 3},
    {"kind": "nvls", "dtype": "i32", "nbytes": 16 << 20, "fail_chunk": 2},
    {"kind": "sm", "dtype": "f32", "nbytes": 32 << 20, "fail_chunk": 3, "armed": True},  # nz_rail_inject_failure
    {"kind": "ce", "dtype": "f32", "nbytes": 4 << 20, "fail_chunk": 1, "armed": True},
    {"kind": "sm", "dtype": "f32", "nbytes": 4096, "abort": True},  # nz_rail_abort: later calls refused
    # Graph-safe rails (device op counter): captured ops replayed, mixed with eager ones.
    {"kind": "sm", "dtype": "f32", "nbytes": 8192, "graph": 3},             # LL path
    {"kind": "sm", "dtype": "bf16", "nbytes": 8 << 20, "graph": 2},         # two-shot fold
    {"kind": "nvls", "dtype": "f32", "nbytes": 16 << 20, "graph": 2},
    {"kind": "ce", "dtype": "i32", "nbytes": 4 << 20, "graph": 2},
]


@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_rails(world):
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cases = MULTI
    if HOST_HARNESS:  # no capture there: the graph cases run their graph-safe rails eagerly
        cases = [dict({k: v for k, v in c.items() if k != "graph"}, graph_safe=True) if c.get("graph") else c
                 for c in MULTI]
    res = spawn(world, os.path.join(ROOT, "tests", "workers", "rail_worker.py"), [json.dumps(cases)], timeout=300)
    for rank_res in res:
        for r in rank_res["results"]:
            assert r["watchdog"] == 0, r
            assert r["outside_nonzero"] == 0, r
            assert r["mismatch"] == 0, r
            assert r["progress"] == r["stop"], r  # nz_rail_progress after the call retired
            case = cases[r["case"]]
            if case.get("abort"):
                assert r["abort_refused"], r
            if case.get("graph") or case.get("graph_safe"):
                assert r["graph_mismatch"] == 0, r
            if case.get("fail_chunk", -1) >= 0:
                assert r["fault"] is not None and r["fault"]["chunk"] == case["fail_chunk"], r
            else:
                assert r["fault"] is None, r


@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_unplanned_link_death_detected(world):
    """nz_rail_inject_stall on one rank (the others are not told): every rank's
    launch fails within the detection budget and the rail works after revive."""
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cases = [{"kind": k, "dtype": "f32", "nbytes": 160 << 20, "stall": [world - 1, 3], "detect_us": 2000}
             for k in ("sm", "nvls", "ce")]
    res = spawn(world, os.path.join(ROOT, "tests", "workers", "rail_worker.py"), [json.dumps(cases)], timeout=300)
    for rank_res in res:
        for r in rank_res["results"]:
            assert r["failed"] and r["mismatch"] == 0 and r["after_revive_mismatch"] == 0, r


@pytest.mark.multigpu
@pytest.mark.parametrize("kind", ["sm", "nvls"])
def test_watchdog_instead_of_hang(kind):
    """A peer that never arrives: the kernel exits after the watchdog budget."""
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = spawn(2, os.path.join(ROOT, "tests", "workers", "watchdog_worker.py"), [kind], timeout=120,
                extra_env={"NEZHA_WATCHDOG_MS": "300"})
    r0 = [r for r in res if r["rank"] == 0][0]
    assert r0["watchdog"] == 1 and r0["seconds"] < 30


@needs_torch_device
@pytest.mark.parametrize("mode", ["sm", "ce"])
def test_config1_hash_emulated(mode):
    """Config 1 (8 ranks, 2 rails of 32 MiB, Ring) through the production fold
    kernels for 8 virtual ranks on one GPU: the output hash equals the golden
    generated from the reference's InMemoryFabric ring."""
    import hashlib

    torch = pytest.importorskip("torch")
    if gpu_count() < 1:
        pytest.skip("no GPU")
    from paper_2405_17870_b200 import emulate_fold

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "config1_hash.json")))
    world, n = g["world"], g["bytes"]
    torch.cuda.set_device(0)
    dins = [torch.from_numpy(oracle.synthetic_input(oracle.F32, r, n).view(np.uint8).copy()).cuda()
            for r in range(world)]
    douts = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(world)]
    for _, off, length in g["segments"]:
        for r in range(world):
            dst = [d.data_ptr() for d in douts] if mode == "sm" else [douts[r].data_ptr()]
            emulate_fold(world, r, oracle.F32, [d.data_ptr() for d in dins], dst, off, length, length, off,
                         off + length)
    torch.cuda.synchronize()
    if mode == "sm":
        for r in range(world):
            assert hashlib.sha256(douts[r].cpu().numpy().tobytes()).hexdigest() == g["sha256"], r
    else:  # each virtual rank wrote its own shard of each segment: stitch them
        full = np.zeros(n, dtype=np.uint8)
        for _, off, length in g["segments"]:
            for r in range(world):
                s, e = shard_of(off, off + length, r, world)
                full[s:e] = douts[r][s:e].cpu().numpy()
        assert hashlib.sha256(full.tobytes()).hexdigest() == g["sha256"]


def random_rail_cases(seed, n=24):
    """Random single-rail geometries: rail kind, dtype, ragged offsets and
    lengths across every protocol path (LL, two-shot, CE), chunk windows and
    injected failures."""
    import random

    rng = random.Random(seed)
    cases = []
    for _ in range(n):
        dtype = rng.choice(["f32", "bf16", "i32"])
        es = 2 if dtype == "bf16" else 4
        nbytes = es * rng.choice([rng.randint(1, 4096), rng.randint(4096, 600_000), rng.randint(600_000, 6_000_000)])
        seg_off = es * rng.randint(0, min(64, nbytes // es - 1))
        seg_len = es * rng.randint(1, nbytes // es - seg_off // es)
        c = {"kind": rng.choice(["sm", "ce", "nvls"]), "dtype": dtype, "nbytes": nbytes, "seg_off": seg_off,
             "seg_len": seg_len}
        r = rng.random()
        if r < 0.2:
            c["fail_chunk"] = rng.randint(0, 3)
        elif r < 0.35:
            c["chunk_begin"] = rng.randint(0, 2)
        cases.append(c)
    return cases


@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_rails_randomized(world):
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cases = random_rail_cases(100 + world)
    res = spawn(world, os.path.join(ROOT, "tests", "workers", "rail_worker.py"), [json.dumps(cases)], timeout=300)
    for rank_res in res:
        for r in rank_res["results"]:
            assert r["watchdog"] == 0 and r["mismatch"] == 0 and r["outside_nonzero"] == 0, (r, cases[r["case"]])
