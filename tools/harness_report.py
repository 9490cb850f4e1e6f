#!/usr/bin/env python3
"""CPU parity record of the kernel SOURCE (no GPU): runs the rail kernels of
csrc/cuda/kernels.cuh on the host harness's fibers (tests/fakecuda, DESIGN.md
§6d) over the GPU suite's rail cases at every world size, the fold kernel's
awkward geometries, fuzzed schedules and the multi-process rails with the
emulated NVSwitch multicast (NVLS K1), and writes the outcome to
profiles/r02/host_harness_parity.json.

    python tools/harness_report.py

This is NOT a hardware record: it proves the kernels' arithmetic, order,
walking and protocols as written, not the compiled SASS, NVLink ordering or
timing.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
HARNESS = os.path.join(ROOT, "tests", "fakecuda", "build", "libnezha_b200_hostharness.so")
ENV = {"NEZHA_TEST_HOST_HARNESS_LIB": HARNESS, "NEZHA_WATCHDOG_MS": "5000", "NEZHA_DETECT_US": "2000000",
       "PYTHONPATH": ROOT}


def last_json(out: str) -> dict:
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


def run(args, extra=None, timeout=1200):
    env = dict(os.environ)
    env.update(ENV)
    env.update(extra or {})
    t0 = time.time()
    r = subprocess.run([sys.executable] + args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    rec = {"cmd": " ".join(os.path.relpath(a, ROOT) if a.startswith(ROOT) else a for a in args),
           "env": {k: v for k, v in (extra or {}).items()}, "rc": r.returncode, "seconds": round(time.time() - t0, 1)}
    if r.returncode == 0:
        rec["result"] = last_json(r.stdout)
    else:
        rec["tail"] = (r.stdout[-1500:] + r.stderr[-1500:])
    print(json.dumps(rec), flush=True)
    return rec


def rails_multiprocess(world: int, multicast: int) -> dict:
    from tests.mp_util import spawn
    from tests.test_gpu_rails import MULTI

    cases = [c for c in MULTI if (multicast or c["kind"] != "nvls") and not c.get("graph")]
    env = dict(ENV)
    env["FAKECUDA_MULTICAST"] = str(multicast)
    t0 = time.time()
    res = spawn(world, os.path.join(ROOT, "tests", "workers", "rail_worker.py"), [json.dumps(cases)], timeout=1200,
                extra_env=env)
    bad = 0
    kinds = {}
    for rk in res:
        for r in rk["results"]:
            ok = r["watchdog"] == 0 and r["mismatch"] == 0 and r["outside_nonzero"] == 0 and r["progress"] == r["stop"]
            bad += not ok
            k = cases[r["case"]]["kind"]
            kinds[k] = kinds.get(k, 0) + 1
    rec = {"cmd": f"tests/workers/rail_worker.py x {world} processes", "env": {"FAKECUDA_MULTICAST": multicast},
           "rc": 0, "seconds": round(time.time() - t0, 1),
           "result": {"world": world, "cases": len(cases), "rank_results_by_kind": kinds, "bad": bad}}
    print(json.dumps(rec), flush=True)
    return rec


def engine_multiprocess(world: int) -> dict:
    """Config-4 shape on the emulated NVSwitch box: 256 MiB bf16 through the
    engine (NVLS + CE + SM), one rank's NVLS link dies mid-op (unplanned),
    the ranks agree and reroute, then readmit (int32, exact on every rail)."""
    from tests.mp_util import spawn
    from tests.test_gpu_engine import TOML3

    spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "readmit_hold_us": 100000,
            "cases": [{"dtype": "bf16", "nbytes": 256 << 20, "reps": 2, "fail": [0, 3], "fail_rep": 1},
                      {"dtype": "i32", "nbytes": 64 << 20, "reps": 1, "readmit": True},
                      {"dtype": "f32", "nbytes": 8192, "reps": 2}]}
    env = dict(ENV)
    env["FAKECUDA_MULTICAST"] = "1"
    t0 = time.time()
    res = spawn(world, os.path.join(ROOT, "tests", "workers", "engine_worker.py"), [json.dumps(spec)], timeout=1800,
                extra_env=env)
    bad = sum(r["mismatch"] != 0 for rk in res for r in rk["results"])
    fos = [{k: f[k] for k in ("failed_rail", "target_rail", "orphan_offset", "orphan_length", "orphan_chunk")}
           for rk in res[:1] for r in rk["results"] if (f := r.get("failover"))]
    rec = {"cmd": f"tests/workers/engine_worker.py x {world} processes (config-4 shape)",
           "env": {"FAKECUDA_MULTICAST": 1}, "rc": 0, "seconds": round(time.time() - t0, 1),
           "result": {"world": world, "ops": sum(len(rk["results"]) for rk in res), "bad": bad, "failovers_rank0": fos}}
    print(json.dumps(rec), flush=True)
    return rec


def engine_failover_each_rail(world: int) -> dict:
    """tests/test_gpu_engine.py::test_engine_failover_reroute's spec on the
    emulated NVSwitch box: a hot split over NVLS + CE + SM (pinned), one
    rank's link of rail 0, 1, then 2 dies mid-op, reroute, readmit."""
    from tests.mp_util import spawn
    from tests.test_gpu_engine import PINNED_HOT, TOML3

    env = dict(ENV)
    env["FAKECUDA_MULTICAST"] = "1"
    t0 = time.time()
    out = []
    bad = 0
    for fr in (0, 1, 2):
        spec = {"rails": ["nvls", "ce", "sm"], "rails_toml": TOML3, "readmit_hold_us": 100000, **PINNED_HOT,
                "cases": [{"dtype": "bf16", "nbytes": 256 << 20, "reps": 3, "fail": [fr, 3], "fail_rep": 1},
                          {"dtype": "i32", "nbytes": 64 << 20, "reps": 2},
                          {"dtype": "i32", "nbytes": 96 << 20, "reps": 1, "readmit": True}]}
        res = spawn(world, os.path.join(ROOT, "tests", "workers", "engine_worker.py"), [json.dumps(spec)], timeout=1800,
                    extra_env=env)
        bad += sum(r["mismatch"] != 0 for rk in res for r in rk["results"])
        fos = [[r["failover"] for r in rk["results"] if r.get("failover")] for rk in res]
        ok = all(len(f) == 1 and f[0]["failed_rail"] == fr and f[0]["target_rail"] != fr and f[0]["orphan_length"] > 0
                 for f in fos)
        bad += not ok
        f0 = fos[0][0] if fos[0] else {}
        out.append({k: f0.get(k) for k in ("failed_rail", "target_rail", "orphan_offset", "orphan_length",
                                           "orphan_chunk")})
    rec = {"cmd": f"tests/workers/engine_worker.py x {world} processes (failover of each rail, hot split)",
           "env": {"FAKECUDA_MULTICAST": 1}, "rc": 0, "seconds": round(time.time() - t0, 1),
           "result": {"world": world, "bad": bad, "failovers_rank0": out}}
    print(json.dumps(rec), flush=True)
    return rec


def gpu_suites_on_harness() -> dict:
    """tests/test_gpu_rails.py + tests/test_gpu_engine.py as written, on the
    harness standing in for a 4-GPU box (multicast emulated)."""
    env = dict(os.environ)
    env.update(ENV)
    env.update({"NEZHA_TEST_HARNESS_GPUS": "4", "FAKECUDA_MULTICAST": "1"})
    t0 = time.time()
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_rails.py", "tests/test_gpu_engine.py", "-m", "gpu",
                        "-q", "-p", "no:cacheprovider", "--timeout", "1800", "-rfE"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=5400)
    summary = [l for l in r.stdout.splitlines() if " passed" in l or " failed" in l][-1:]
    rec = {"cmd": "pytest tests/test_gpu_rails.py tests/test_gpu_engine.py -m gpu (4 harness GPUs)",
           "env": {"NEZHA_TEST_HARNESS_GPUS": 4, "FAKECUDA_MULTICAST": 1}, "rc": r.returncode,
           "seconds": round(time.time() - t0, 1),
           "result": {"summary": summary[0] if summary else r.stdout[-300:],
                      "skipped_by_design": "in-process torch device buffers, CUDA graph capture, DDP (torch)",
                      "bad": 0 if r.returncode == 0 else 1}}
    print(json.dumps(rec), flush=True)
    return rec


def main() -> None:
    subprocess.run(["make", "-j8", "-C", os.path.join(ROOT, "tests", "fakecuda")], check=True, capture_output=True)
    head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True, text=True).stdout.strip()
    runs = []
    for w in range(2, 9):
        runs.append(run([os.path.join(ROOT, "tests", "workers", "simt_rails.py"), str(w), str(300 + w)]))
    for w, seed in ((3, 1), (6, 2), (8, 3)):
        runs.append(run([os.path.join(ROOT, "tests", "workers", "simt_rails.py"), str(w), str(400 + w)],
                        {"FAKECUDA_SIMT_PREEMPT": "30", "FAKECUDA_SIMT_SEED": str(seed)}))
    for seed in (1, 2, 3, 4):
        runs.append(run([os.path.join(ROOT, "tests", "workers", "simt_fold.py"), str(seed)]))
    for w, mc in ((2, 0), (2, 1), (3, 1), (4, 1), (8, 1)):
        runs.append(rails_multiprocess(w, mc))
    runs.append(engine_multiprocess(8))
    runs.append(engine_failover_each_rail(4))
    runs.append(gpu_suites_on_harness())
    ok = all(r["rc"] == 0 and not r["result"].get("bad") for r in runs)
    out = {"what": "rail kernels of csrc/cuda/kernels.cuh run from source on host fibers (tests/fakecuda/simt.h), "
                   "checked against the CPU oracle; NOT a hardware record",
           "git_head": head, "all_ok": ok, "runs": runs}
    path = os.path.join(ROOT, "profiles", "r02", "host_harness_parity.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, "all_ok", ok)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
