"""CPU suite: the product's HOST logic end to end, without a GPU.

tests/fakecuda links the product's own object files (the same ones as
libnezha_b200.so) against a host stand-in for the CUDA runtime whose kernel
launches run the product's CUDA kernel source itself on host fibers
(tests/fakecuda/simt.h: one fiber per CUDA thread, per-CTA __syncthreads,
cross-rank polls that yield; barrier epochs, LL flags, launch status, gates
and injected stalls are the kernels' own code). Running the loopback GPU
tests (tests/test_gpu_vranks.py) against it exercises, on CPU: the
virtual-rank communicator and combined launches, the rails' waves, chunk
windows and copy-engine pipelining, the engine's hot split / Timer / staged
host path, the failure monitor's detection, two-round agreement, reroute and
readmit — and checks every result against the oracle.

It checks host logic and the kernel SOURCE (arithmetic, order, walking,
protocols). It says nothing about the compiled SASS, cross-GPU memory
ordering, NVLink or timing (the GPU suite's job), and it is never the product: the
harness library is loaded only by the subprocesses started here
(NEZHA_TEST_HOST_HARNESS_LIB, accepted by _lib.py for this file name only).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "tests", "fakecuda", "build", "libnezha_b200_hostharness.so")

# A cross-section of tests/test_gpu_vranks.py (its rail parity cases run in
# test_kernel_source_on_host_fibers below) (the full file, ~7 min, is `python -m pytest
# tests/test_gpu_vranks.py -m gpu` with the same environment).
SELECTION = " or ".join([
    "test_loopback_unplanned_link_death_detected and sm-4",
    "test_loopback_unplanned_link_death_detected and ce-2",
    "test_loopback_engine_multirail_parity and 4",
    "test_loopback_engine_unplanned_failover and 1",
    "test_loopback_engine_compute_pool_parity and 1",
    "test_loopback_engine_calibrated",
    "test_loopback_config1_hash",
])


@pytest.fixture(scope="module")
def harness():
    r = subprocess.run(["make", "-j8", "-C", os.path.join(ROOT, "tests", "fakecuda")], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail("harness build failed:\n" + r.stdout[-3000:] + r.stderr[-3000:])
    return HARNESS


def test_loopback_suite_host_logic(harness):
    env = dict(os.environ)
    env.update({"NEZHA_TEST_HOST_HARNESS_LIB": harness, "NEZHA_WATCHDOG_MS": "5000",
                "NEZHA_DETECT_US": "2000000", "PYTHONPATH": ROOT})
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_vranks.py"), "-m", "gpu",
                        "-q", "-p", "no:cacheprovider", "-n", "3", "--timeout", "600", "-k", SELECTION, "-rfE"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = r.stdout[-6000:] + r.stderr[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "skipped" not in r.stdout.split("passed")[0][-20:], tail


def test_harness_is_not_the_product(harness):
    """The harness build is accepted only under its own name, and the product
    library never exports the stand-in's runtime."""
    env = dict(os.environ)
    env["NEZHA_TEST_HOST_HARNESS_LIB"] = os.path.join(ROOT, "paper_2405_17870_b200", "libnezha_b200.so")
    r = subprocess.run([sys.executable, "-c", "import paper_2405_17870_b200 as p; p.lib()"], cwd=ROOT, env=env,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "must name the test harness build" in r.stderr
    nm = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2405_17870_b200", "libnezha_b200.so")],
                        capture_output=True, text=True).stdout
    assert " fakecuda_launches" not in nm and " T cudaLaunchKernel" not in nm


def test_multiprocess_engine_nvls_host_logic(harness):
    """The engine across processes with the NVLS rail (emulated multicast):
    cold plans on NVLS, the staged host and device paths, an unplanned NVLS
    link death rerouted to a survivor, readmit — exact on every rank."""
    import json

    from tests.mp_util import spawn
    from tests.test_gpu_engine import TOML3

    spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "window": 4, "readmit_hold_us": 100000,
            "cases": [{"dtype": "f32", "nbytes": 24 << 20, "reps": 3},
                      {"dtype": "bf16", "nbytes": (6 << 20) + 2, "reps": 1, "host": True},
                      {"dtype": "i32", "nbytes": 12, "reps": 1},
                      {"dtype": "bf16", "nbytes": 64 << 20, "reps": 2, "fail": [0, 3], "fail_rep": 1},
                      {"dtype": "i32", "nbytes": 16 << 20, "reps": 1, "readmit": True},
                      {"dtype": "f32", "nbytes": (8 << 20) + 4, "reps": 1, "device": True}]}
    env = _env(harness)
    env["FAKECUDA_MULTICAST"] = "1"
    res = spawn(2, os.path.join(ROOT, "tests", "workers", "engine_worker.py"), [json.dumps(spec)], timeout=600,
                extra_env=env)
    for rk in res:
        for r in rk["results"]:
            assert r["mismatch"] == 0, r
        fos = [r["failover"] for r in rk["results"] if r.get("failover")]
        assert len(fos) == 1 and fos[0]["failed_rail"] == 0 and fos[0]["target_rail"] != 0, fos
        assert fos[0]["orphan_length"] > 0, fos


def _env(harness):
    return {"NEZHA_TEST_HOST_HARNESS_LIB": harness, "NEZHA_WATCHDOG_MS": "5000", "NEZHA_DETECT_US": "2000000"}


@pytest.mark.parametrize("world,multicast", [(2, 0), (3, 0), (2, 1), (4, 1)])
def test_multiprocess_rails_host_logic(harness, world, multicast):
    """One process per rank (nz_comm_init: abstract-socket bootstrap, VMM fds
    over SCM_RIGHTS, peer mappings), the rails' direct launches: the
    multi-GPU path's host side and kernel source, checked against the oracle.
    multicast=1 emulates the NVSwitch multicast object (FAKECUDA_MULTICAST:
    a bound team table, an inaccessible window, multimem accesses resolved to
    every member and trapping when misaligned), so the NVLS rail's kernel
    (K1) runs too."""
    import json

    from tests.mp_util import spawn
    from tests.test_gpu_rails import MULTI

    # No CUDA graph capture here: the graph cases run their graph-safe rails
    # eagerly (epochs / LL flags from the device launch counter).
    cases = [dict({k: v for k, v in c.items() if k != "graph"}, graph_safe=True) if c.get("graph") else c
             for c in MULTI if multicast or c["kind"] != "nvls"]
    env = _env(harness)
    env["FAKECUDA_MULTICAST"] = str(multicast)
    res = spawn(world, os.path.join(ROOT, "tests", "workers", "rail_worker.py"), [json.dumps(cases)], timeout=600,
                extra_env=env)
    for rank_res in res:
        assert len(rank_res["results"]) == len(cases)
        for r in rank_res["results"]:
            assert r["watchdog"] == 0 and r["mismatch"] == 0 and r["outside_nonzero"] == 0, r
            assert r["progress"] == r["stop"] and r.get("graph_mismatch", 0) == 0, r


def test_multiprocess_engine_failover_host_logic(harness):
    """The engine across processes: hot split, staged host path, an unplanned
    link death agreed by the monitors over their own socket channel, the
    orphan rerouted, readmit after the hold — results exact on every rank."""
    import json

    from tests.mp_util import spawn
    from tests.test_gpu_vranks import KINDS3, TOML_LOOP

    spec = {"rails": KINDS3, "rails_toml": TOML_LOOP, "sync_overhead_us": 0.0, "readmit_hold_us": 100000,
            "cases": [{"dtype": "f32", "nbytes": 24 << 20, "reps": 2},
                      {"dtype": "bf16", "nbytes": 64 << 20, "reps": 2, "fail": [2, 3], "fail_rep": 1},
                      {"dtype": "f32", "nbytes": (1 << 20) + 4, "reps": 1, "host": True},
                      {"dtype": "i32", "nbytes": 16 << 20, "reps": 1, "readmit": True}]}
    res = spawn(2, os.path.join(ROOT, "tests", "workers", "engine_worker.py"), [json.dumps(spec)], timeout=600,
                extra_env=_env(harness))
    for rk in res:
        for r in rk["results"]:
            assert r["mismatch"] == 0, r
        fos = [r["failover"] for r in rk["results"] if r.get("failover")]
        assert len(fos) == 1 and fos[0]["failed_rail"] == 2 and fos[0]["orphan_length"] > 0, fos


def test_smoke_host_logic(harness):
    """The driver's smoke() minus its torch-only kernel check: the 4-virtual-
    rank engine (hot split, unplanned failover) and the N = 1 engine."""
    env = dict(os.environ)
    env.update(_env(harness))
    env["PYTHONPATH"] = ROOT
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g._smoke_engine(); g._smoke_single(); "
                        "print('smoke host logic ok')"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "smoke host logic ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("grace_us,spurious", [(1_000_000, False), (0, True)])
def test_straggler_is_not_a_rail_failure(harness, grace_us, spurious):
    """One process per rank; one rank's host issues its allreduce 0.6 s late,
    so the other's launch waits at its start barrier for longer than three
    missed heartbeats (150 ms). Within the start grace that wait is not a rail
    failure: no failover, the rail stays in the table. With the grace off the
    heartbeat detector fires on the straggler (the behaviour the grace
    removes); the result is exact either way."""
    from tests.mp_util import spawn

    env = _env(harness)
    env["NEZHA_START_GRACE_US"] = str(grace_us)
    res = spawn(2, os.path.join(ROOT, "tests", "workers", "straggler_worker.py"), ["0.6"], timeout=300, extra_env=env)
    for r in res:
        assert r["monitor_on"] and r["mismatch"] == 0, r
        assert (r["failovers"] > 0) == spurious, r


@pytest.mark.parametrize("mode", ["processes", "virtual"])
def test_ops_on_two_caller_streams_stay_ordered(harness, mode):
    """Cold and hot ops issued on two caller streams in turn, never
    synchronised in between: each rail's launches stay ordered (orderBefore /
    orderAfter) and every result is exact. (With the ordering removed this
    run hangs or fails: the rails' pads and LL slots are shared.)"""
    from tests.mp_util import spawn

    env = _env(harness)
    script = os.path.join(ROOT, "tests", "workers", "streams_worker.py")
    if mode == "processes":
        res = spawn(2, script, [], timeout=300, extra_env=env)
    else:
        full = dict(os.environ)
        full.update(env)
        full["PYTHONPATH"] = ROOT
        r = subprocess.run([sys.executable, script, "3"], cwd=ROOT, env=full, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        import json

        res = json.loads(r.stdout.strip().splitlines()[-1])
    for rk in res:
        assert rk["mismatch"] == 0 and rk["hot_ops"] > 0 and rk["ops"] == 24, rk


def test_bench_loopback_line_host_logic(harness):
    """bench.py's N = 1 path end to end (config 1, 8 virtual ranks, e2e,
    failover section) with torch replaced by tests/fakecuda/torch_stub.py:
    the JSON line carries every field of the contract. Numbers are the
    emulation's and mean nothing; the code path is what is checked."""
    import json

    env = dict(os.environ)
    env.update(_env(harness))
    env.update({"PYTHONPATH": ROOT, "NEZHA_HEARTBEAT_US": "5000000", "NEZHA_WATCHDOG_MS": "20000"})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fakecuda", "run_bench.py"), "--steps", "2",
                        "--warmup", "3", "--no-cpu"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["ranks"] == 8 and line["config"]["same_config"]
    assert [s[2] for s in line["config"]["plan"]] == [32 << 20, 32 << 20]  # config 1's static 50/50
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["achieved"] > 0 and 0 < rf["frac"] and "traffic" in rf
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == e2e["d2h_bytes_per_step"] == 8 * (64 << 20)
    assert "failover" in line and line["failover"]["failed_rail"] in ("sm", "ce"), line.get("failover_error")


def test_bench_multi_rank_line_host_logic(harness):
    """bench.py's N > 1 path (one process per rank, as torchrun runs it):
    config-1 headline, e2e, 8 KiB latency, failover + readmit; NCCL and the
    size sweep left out (no torch.distributed / time on the harness)."""
    import json

    from tests.mp_util import spawn

    env = _env(harness)
    env.update({"NEZHA_HEARTBEAT_US": "5000000", "NEZHA_WATCHDOG_MS": "20000"})
    res = spawn(2, os.path.join(ROOT, "tests", "fakecuda", "run_bench.py"),
                ["--gpus", "2", "--steps", "2", "--warmup", "3", "--no-nccl", "--no-sweep", "--latency-ops", "20",
                 "--tune-ops", "2"], timeout=1200, extra_env=env)
    line = res[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0, line
    assert line["roofline"]["bound"] == "nvlink" and line["e2e"]["h2d_bytes_per_step"] == 64 << 20
    assert set(line["latency_8k"]) >= {"ops", "engine", "ce_alone", "sm_alone"}
    assert "failover" in line and "readmit_error" not in line, (line.get("failover_error"), line.get("readmit_error"))
    assert res[1] == {}  # only rank 0 prints the line


@pytest.mark.parametrize("world,preempt", [(2, 0), (8, 0), (5, 20)])
def test_kernel_source_on_host_fibers(harness, world, preempt):
    """The rails' CUDA kernels themselves (csrc/cuda/kernels.cuh compiled for
    the host SIMT stand-in, tests/fakecuda/simt.h: one fiber per CUDA thread,
    per-CTA __syncthreads, yielding cross-rank polls) run the loopback rail
    cases — SM two-shot fold with its barriers, LL one-shot, CE barriers and
    reduce, ragged bf16 / i32 geometries, chunk windows, trace-form failures,
    random geometries — bit-exact against the oracle. preempt > 0 fuzzes the
    schedule: random yields at every data load / store and a shuffled fiber
    order per pass."""
    import json

    env = dict(os.environ)
    env.update(_env(harness))
    env.update({"FAKECUDA_SIMT": "1", "FAKECUDA_SIMT_PREEMPT": str(preempt), "FAKECUDA_SIMT_SEED": str(world),
                "PYTHONPATH": ROOT})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "workers", "simt_rails.py"), str(world),
                        str(300 + world)], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    out = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert out["grids"] > 0 and out["threads"] >= out["grids"] * 32, out  # the kernels ran, on fibers


@pytest.mark.parametrize("seed", [1, 2])
def test_fold_kernel_awkward_geometries_on_host_fibers(harness, seed):
    """The SM / CE fold kernel (K2 / K3 source) through nz_emulate_fold on
    host fibers: the GPU suite's emulated-fold cases plus 40 random awkward
    geometries (runs shorter than a vector, chunks of fewer than N elements,
    ragged heads / tails, grids that cut runs between CTAs), bit-exact."""
    import json

    env = dict(os.environ)
    env.update(_env(harness))
    env["PYTHONPATH"] = ROOT
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "workers", "simt_fold.py"), str(seed)], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    out = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert out["cases"] >= 60 and out["bad"] == [], out


def test_multiprocess_link_death_and_watchdog_host_logic(harness):
    """One rank's link dies mid-op on each rail, NVLS included (emulated
    multicast), the other rank not told: every rank's launch fails, the
    completed waves are exact, and after revive the op is exact; then a peer
    that never arrives at all: the waiting kernel leaves at the watchdog."""
    import json

    from tests.mp_util import spawn

    env = _env(harness)
    env["FAKECUDA_MULTICAST"] = "1"
    cases = [{"kind": k, "dtype": "f32", "nbytes": 160 << 20, "stall": [1, 3], "detect_us": 2000}
             for k in ("sm", "nvls", "ce")]
    res = spawn(2, os.path.join(ROOT, "tests", "workers", "rail_worker.py"), [json.dumps(cases)], timeout=600,
                extra_env=env)
    for rank_res in res:
        for r in rank_res["results"]:
            assert r["failed"] and r["mismatch"] == 0 and r["after_revive_mismatch"] == 0, r
            assert r["stalled_here"] == (rank_res["rank"] == 1) and r["detected_here"] == (rank_res["rank"] == 0), r
    for kind in ("sm", "nvls"):
        res = spawn(2, os.path.join(ROOT, "tests", "workers", "watchdog_worker.py"), [kind], timeout=120,
                    extra_env=dict(env, NEZHA_WATCHDOG_MS="300"))
        r0 = [r for r in res if r["rank"] == 0][0]
        assert r0["watchdog"] == 1 and r0["seconds"] < 30, r0


def test_multi_gpu_suites_on_harness(harness):
    """tests/test_gpu_rails.py and tests/test_gpu_engine.py as written, the
    harness standing in for a 4-GPU NVSwitch box (NEZHA_TEST_HARNESS_GPUS:
    one process per GPU, multicast emulated): a fast cross-section here; the
    whole of both files passes the same way (tools/harness_report.py)."""
    env = dict(os.environ)
    env.update(_env(harness))
    env.update({"NEZHA_TEST_HARNESS_GPUS": "4", "FAKECUDA_MULTICAST": "1", "PYTHONPATH": ROOT})
    sel = ("test_multi_gpu_rails or test_watchdog_instead_of_hang or test_engine_single_gpu_identity or "
           "test_engine_compute_pool_parity")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_rails.py"),
                        os.path.join(ROOT, "tests", "test_gpu_engine.py"), "-m", "gpu", "-q", "-p", "no:cacheprovider",
                        "-n", "3", "--timeout", "900", "-k", sel, "-rfE"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-3000:]
    assert " passed" in r.stdout, r.stdout[-3000:]
