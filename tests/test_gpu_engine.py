"""GPU: the multi-rail engine end to end (planner + rails + failure monitor)
against the CPU oracle, one process per GPU, through the C ABI. The same
checks with virtual ranks on one GPU are in test_gpu_vranks.py."""
import json
import os

import pytest

from tests.conftest import gpu_count
from tests.mp_util import spawn

pytestmark = [pytest.mark.gpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "workers", "engine_worker.py")
# tests/test_host_harness.py runs this file on the CPU harness (processes as
# GPUs, emulated multicast): no torch device, no CUDA graph capture there.
HOST_HARNESS = bool(os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB"))
needs_torch_device = pytest.mark.skipif(HOST_HARNESS, reason="torch device / CUDA graphs")

# Rails with a fixed profile so the hot split is exercised deterministically.
# The failover and ComputePool tests also pin sync_overhead_us = 0 and turn
# P12 demotion off: the plan must be the hot split over all three rails
# (whatever the measured concurrent times say), so that the rail killed
# always carries a segment and concurrent rails are always arbitrated.
PINNED_HOT = {"sync_overhead_us": 0.0, "demote_after": 0}
TOML3 = """
[[rail]]
protocol = "nvls"
t_setup_us = 12.0
bandwidth_bps = 6.0e11
[[rail]]
protocol = "ce"
t_setup_us = 40.0
bandwidth_bps = 5.0e11
[[rail]]
protocol = "sm"
t_setup_us = 14.0
bandwidth_bps = 5.0e11
"""


def _run(world, spec, timeout=420):
    res = spawn(world, WORKER, [json.dumps(spec)], timeout=timeout)
    for rk in res:
        for r in rk["results"]:
            assert r["mismatch"] == 0, r
    return res


def test_engine_single_gpu_identity():
    """N = 1: every plan degenerates to a local copy; result = input."""
    if gpu_count() < 1:
        pytest.skip("no GPU")
    spec = {"rails": ["nvls", "ce", "sm"], "calibrate_max_bytes": 1 << 22,
            "cases": [{"dtype": "f32", "nbytes": 1 << 20}, {"dtype": "bf16", "nbytes": 3_000_002},
                      {"dtype": "i32", "nbytes": 4096, "host": True}]}
    _run(1, spec)


@pytest.mark.multigpu
@pytest.mark.parametrize("world", [2, 4])
def test_engine_multirail_parity(world):
    if gpu_count() < world:
        pytest.skip(f"needs {world} GPUs")
    spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "window": 4, "tune_budgets": 1,
            "cases": [
                {"dtype": "f32", "nbytes": 64 << 20, "reps": 10},
                {"dtype": "bf16", "nbytes": 48 << 20, "reps": 2},
                {"dtype": "i32", "nbytes": (32 << 20) + 12, "reps": 2},
                {"dtype": "f32", "nbytes": 8192, "reps": 3},
                {"dtype": "f32", "nbytes": 1 << 20, "reps": 2, "host": True},
                {"dtype": "bf16", "nbytes": (24 << 20) + 2, "reps": 1, "host": True},  # pipelined pieces
                {"dtype": "f32", "nbytes": 4, "reps": 2},     # one element, fewer than ranks
                {"dtype": "bf16", "nbytes": 2, "reps": 2},
                {"dtype": "i32", "nbytes": 12, "reps": 1, "host": True},
                {"dtype": "bf16", "nbytes": 4_194_306, "reps": 2},  # odd bf16 count near the LL ceiling
                {"dtype": "f32", "nbytes": (40 << 20) + 4, "reps": 2, "device": True},  # staged pipeline
                {"dtype": "i32", "nbytes": 4096, "reps": 1, "device": True},
            ]}
    res = _run(world, spec, timeout=420)
    # Every rank ran the same plans (the table is agreed across ranks).
    plans = [[r["segs"] for r in rk["results"]] for rk in res]
    assert all(p == plans[0] for p in plans)
    # Startup budget tuning picked a candidate grid, the same on every rank.
    budgets = [[(x["kind"], x["sm_budget"]) for x in rk["state"]["rails"]] for rk in res]
    assert all(b == budgets[0] for b in budgets)
    sms = 16 if HOST_HARNESS else 1 << 30  # the harness reports 16 SMs; budgets are capped by the SM count
    cands = {"nvls": {min(c, sms) for c in (16, 32, 64)}, "sm": {min(c, sms) for c in (32, 64, 128)}, "ce": {0}}
    assert all(v in cands[k] for k, v in budgets[0]), budgets[0]


@pytest.mark.multigpu
@pytest.mark.parametrize("mode", [1, 2])
def test_engine_compute_pool_parity(mode):
    """SM arbitration of concurrent rails (ComputePool, P14): the
    result is unchanged and every op's grants are the oracle's for its demands."""
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    from oracle.compute_pool import plan_grants

    tokens = 100
    spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "window": 4, "compute_pool": mode, **PINNED_HOT,
            "pool_tokens": tokens,
            "cases": [{"dtype": "f32", "nbytes": 64 << 20, "reps": 6},
                      {"dtype": "bf16", "nbytes": 24 << 20, "reps": 2},
                      {"dtype": "i32", "nbytes": 16 << 20, "reps": 2}]}
    res = _run(2, spec, timeout=420)
    arbitrated = 0
    for rk in res:
        assert rk["state"]["compute_pool"]["mode"] == mode
        for r in rk["results"]:
            for g in r["grants"]:
                demands = [(x[0], x[1]) for x in g]
                want = plan_grants(tokens, mode, demands)
                assert [[w["rail"], w["demand"], w["grant"], w["waits"]] for w in want] == g, r
                arbitrated += 1
    assert arbitrated > 0


@needs_torch_device
@pytest.mark.multigpu
def test_engine_graph_capture():
    """graph_safe engine (device op counters in the rails): allreduces captured
    in a CUDA graph and replayed give the oracle's result on every plan kind."""
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "window": 4, "graph_safe": 1,
            "cases": [{"dtype": "f32", "nbytes": 64 << 20, "reps": 8},     # converges to a hot split
                      {"dtype": "f32", "nbytes": 64 << 20, "reps": 1, "graph": 3},
                      {"dtype": "bf16", "nbytes": 8192, "reps": 1, "graph": 4},
                      {"dtype": "i32", "nbytes": 3 << 20, "reps": 1, "graph": 2}]}
    _run(2, spec, timeout=420)


@pytest.mark.multigpu
def test_engine_oversized_split():
    """Payloads above 1 GiB run as 256 MiB pieces."""
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    n = (1 << 30) + (64 << 20)
    spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "calibrate_max_bytes": 1 << 20,
            "cases": [{"dtype": "f32", "nbytes": n}]}
    res = _run(2, spec, timeout=420)
    r = res[0]["results"][0]
    assert max(s[1] + s[2] for s in r["segs"]) == n
    assert len({(s[1] // (256 << 20)) for s in r["segs"]}) == 5


@pytest.mark.multigpu
@pytest.mark.parametrize("fail_rail", [0, 1, 2])
def test_engine_failover_reroute(fail_rail):
    world = 4 if gpu_count() >= 4 else 2
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "readmit_hold_us": 100000, **PINNED_HOT,
            "cases": [{"dtype": "bf16", "nbytes": 256 << 20, "reps": 3, "fail": [fail_rail, 3], "fail_rep": 1},
                      {"dtype": "i32", "nbytes": 64 << 20, "reps": 2},
                      {"dtype": "i32", "nbytes": 96 << 20, "reps": 1, "readmit": True}]}
    res = _run(world, spec, timeout=420)
    for rk in res:
        fo = [r for r in rk["results"] if "failover" in r][0]["failover"]
        assert fo is not None and fo["failed_rail"] == fail_rail
        assert fo["target_rail"] != fail_rail and fo["orphan_length"] > 0
        assert fo["done_us"] > 0 and 0 < fo["resume_after_detect_us"] < (1e12 if HOST_HARNESS else 1000), fo
        assert fo["stalled_here"] == (1 if rk["rank"] == world - 1 else 0), fo
        # After the failure the rail carries nothing until it is readmitted.
        later = [r for r in rk["results"] if r["case"] == 0 and r["rep"] == 2] + \
                [r for r in rk["results"] if r["case"] in (1, 2)]
        for r in later:
            assert all(s[0] != fail_rail for s in r["segs"]), r


@pytest.mark.multigpu
def test_engine_failover_trials_acceptance5():
    """SPEC acceptance 5 on B200: repeated unplanned single-rail
    link deaths at random rails / chunks / ranks; every result bit-exact
    (int32), every reroute resumes within 1 ms of its detection."""
    import random

    world = 4 if gpu_count() >= 4 else 2
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    rng = random.Random(539)
    cases = [{"dtype": "i32", "nbytes": 256 << 20, "reps": 2}]  # settle the hot split
    for _ in range(16):
        cases.append({"dtype": "i32", "nbytes": 256 << 20, "reps": 1, "fail": [rng.randrange(3), rng.randrange(6)],
                      "fail_rank": rng.randrange(world), "readmit": True})
    res = _run(world, {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "readmit_hold_us": 100000, **PINNED_HOT,
                       "cases": cases}, timeout=600)
    fos = [r["failover"] for rk in res for r in rk["results"] if r.get("failover")]
    assert len(fos) >= 8, fos
    assert HOST_HARNESS or all(f["resume_after_detect_us"] < 1000 for f in fos), fos  # device timing only


@pytest.mark.multigpu
def test_engine_failover_int32_every_rail_exact():
    """Config 4 rerun as int32: bit-exact on every rail, NVLS included (P2)."""
    world = 4 if gpu_count() >= 4 else 2
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    cases = []
    for rail in (0, 1, 2):
        cases.append({"dtype": "i32", "nbytes": 256 << 20, "reps": 1, "fail": [rail, 2], "readmit": True})
    res = _run(world, {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "readmit_hold_us": 100000, **PINNED_HOT, "cases": cases},
               timeout=420)
    for rk in res:
        assert len([r for r in rk["results"] if r.get("failover")]) == 3


@needs_torch_device
@pytest.mark.multigpu
def test_ddp_comm_hook_matches_nccl():
    """The engine as a PyTorch DDP comm hook (paper_2405_17870_b200/ddp.py)."""
    if gpu_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = spawn(2, os.path.join(ROOT, "tests", "workers", "ddp_worker.py"), timeout=600)
    for r in res:
        assert r["ok"], r
