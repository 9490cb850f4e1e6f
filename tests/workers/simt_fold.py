"""Host-harness worker (tests/test_host_harness.py): the SM / CE rail fold
kernel (K2 / K3, csrc/cuda/kernels.cuh, through nz_emulate_fold) on host
fibers over the GPU suite's emulated-fold cases plus randomized awkward
geometries — chunks of a few elements (runs shorter than a 16-byte vector,
so vectors straddle runs), chunks smaller than N elements (q = 0), ragged
heads / tails, explicit grids that cut runs between CTAs — every rank's
output bit-exact against the oracle. argv: seed. Prints one JSON line.

Run only with NEZHA_TEST_HOST_HARNESS_LIB set (the harness build): "device"
pointers are host memory there.
"""
import ctypes
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
from paper_2405_17870_b200 import emulate_fold  # noqa: E402
from tests.test_gpu_rails import EMU_CASES, shard_of  # noqa: E402


def bits(a):
    return a.view(np.uint16) if a.dtype == np.uint16 else a.view(np.uint32)


def run_case(h, world, dtype, nbytes, seg_off, seg_len, chunk, mode, grid, seed):
    es = 2 if dtype == oracle.BF16 else 4
    inputs = [oracle.synthetic_input(dtype, r, nbytes, seed_base=seed + r) for r in range(world)]
    outs = [np.zeros(nbytes // es, dtype=inputs[0].dtype) for _ in range(world)]
    lo, hi = seg_off, seg_off + seg_len
    for r in range(world):
        dst = [o.ctypes.data for o in outs] if mode == "sm" else [outs[r].ctypes.data]
        emulate_fold(world, r, dtype, [x.ctypes.data for x in inputs], dst, seg_off, seg_len, chunk, lo, hi, grid=grid)
    assert h.cudaDeviceSynchronize() == 0
    want = oracle.reduce_range(inputs, dtype, seg_off, seg_len, chunk, lo, hi)
    bad = 0
    for r in range(world):
        if mode == "sm":
            bad += int(np.sum(bits(outs[r]) != bits(want)))
        else:
            s, e = shard_of(lo, hi, r, world)
            bad += int(np.sum(bits(outs[r][s // es:e // es]) != bits(want[s // es:e // es])))
    return bad


def main() -> None:
    seed = int(sys.argv[1])
    h = ctypes.CDLL(os.environ["NEZHA_TEST_HOST_HARNESS_LIB"])
    cases = []
    for world, dtype, nbytes, seg_off, seg_len, chunked in EMU_CASES:
        if nbytes > (4 << 20):
            continue  # the large ones run through the rails already
        for mode in ("sm", "ce"):
            cases.append((world, dtype, nbytes, seg_off, seg_len, oracle.default_chunk_bytes(seg_len, world, chunked),
                          mode, 0))
    rng = random.Random(seed)
    for _ in range(40):
        world = rng.randint(2, 8)
        dtype = rng.choice([oracle.F32, oracle.BF16, oracle.I32])
        es = 2 if dtype == oracle.BF16 else 4
        n = rng.choice([rng.randint(1, 64), rng.randint(64, 4096), rng.randint(4096, 60_000)])
        seg_off = es * rng.randint(0, 9)
        nbytes = seg_off + es * n + es * rng.randint(0, 9)
        chunk = es * rng.choice([rng.randint(1, 2 * world), rng.randint(world, 12 * world), rng.randint(1, n)])
        grid = rng.choice([0, 1, 2, 3, 7, 16])
        cases.append((world, dtype, nbytes, seg_off, es * n, chunk, rng.choice(["sm", "ce"]), grid))
    bad = []
    for i, c in enumerate(cases):
        m = run_case(h, *c, seed=oracle.SEED_BASE + 31 * i)
        if m:
            bad.append({"case": list(c), "mismatch": m})
    print(json.dumps({"cases": len(cases), "bad": bad}))


if __name__ == "__main__":
    main()
