"""Host-harness worker (tests/test_host_harness.py): the loopback rails' GPU
parity cases with the product's CUDA kernel source running on host fibers
(tests/fakecuda/simt.h). argv: world, seed of the random cases; prints one
JSON line with the number of grids / CUDA threads the fibers ran.

Run only with NEZHA_TEST_HOST_HARNESS_LIB set (the harness build).
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from tests.test_gpu_vranks import RAIL_CASES, _check_rails, _rails, random_rail_cases  # noqa: E402


def main() -> None:
    world, seed = int(sys.argv[1]), int(sys.argv[2])
    _check_rails(_rails(world, RAIL_CASES), RAIL_CASES)
    cases = random_rail_cases(seed, 8)
    for rank_res in _rails(world, cases):
        for r in rank_res["results"]:
            assert r["watchdog"] == 0 and r["mismatch"] == 0 and r["outside_nonzero"] == 0, (r, cases[r["case"]])
    cases = RAIL_CASES + cases
    h = ctypes.CDLL(os.environ["NEZHA_TEST_HOST_HARNESS_LIB"])
    h.fakecuda_simt_grids.restype = ctypes.c_uint64
    h.fakecuda_simt_threads.restype = ctypes.c_uint64
    print(json.dumps({"world": world, "cases": len(cases), "grids": h.fakecuda_simt_grids(),
                      "threads": h.fakecuda_simt_threads()}))


if __name__ == "__main__":
    main()
