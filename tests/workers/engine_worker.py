"""One rank of an engine run: a process per GPU (tests/mp_util.spawn, argv[1]
= JSON spec, prints one JSON line) or a thread per virtual rank on one GPU
(``run`` through paper_2405_17870_b200.run_ranks).

spec = {"rails": [...kinds], "cases": [...]} where each case is
{"dtype", "nbytes", "reps", "fail": [rail, chunk] | null, "fail_rank": r,
 "fail_rep": i, "host": bool, "device": bool, "graph": n, "readmit": bool}.
Every op's output is compared with the CPU oracle evaluated on the plan the
engine reports it ran (nz_engine_last_plan_json): bit-exact on CE/SM
segments and int32, NVLS fp32 within 1e-6 of sum|x|, NVLS bf16 within 1 ulp.

A failure case kills ONE rank's link of the rail (``fail_rank``, default the
last rank) at the chunk, unplanned (nz_engine_inject_failure on that rank
only): every rank's monitor must detect it, agree on the orphan and reroute
it, so the result is still the oracle's — the orphan reduced by the target
rail with the failed segment's geometry (P9/P10) — and the report carries
the failover times.
"""
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
from paper_2405_17870_b200 import Comm, Engine, SymmetricBuffer  # noqa: E402
from paper_2405_17870_b200._lib import DTYPES  # noqa: E402

ES = {oracle.F32: 4, oracle.BF16: 2, oracle.I32: 4}
_cache: dict = {}
_cache_lock = threading.Lock()


def clear_cache() -> None:
    with _cache_lock:
        _cache.clear()


def evict_case(ci) -> None:
    """Drops case ci's inputs and oracle results (every rank is past it)."""
    with _cache_lock:
        for k in [k for k in _cache if len(k) > 1 and k[1] == ci]:
            del _cache[k]


def cached(key, fn):
    with _cache_lock:
        ev = _cache.get(key)
        if ev is None:
            ev = _cache[key] = [threading.Event(), None]
            owner = True
        else:
            owner = False
    if owner:
        try:
            ev[1] = fn()
        finally:
            ev[0].set()
    else:
        ev[0].wait()
    return ev[1]


def check_segment(kind, dt, got, inputs, off, length, chunk):
    return check_segment_range(kind, dt, got, inputs, off, length, chunk, off, off + length)


def _want(dt, inputs, n, off, length, chunk, lo, hi, key):
    def make():
        want = np.zeros(n // ES[dt], dtype=oracle.NP_DTYPE[dt])
        oracle.reduce_range(inputs, dt, off, length, chunk, lo, hi, want)
        return want
    return cached(("want", key, off, length, chunk, lo, hi), make) if key is not None else make()


def check_segment_range(kind, dt, got, inputs, off, length, chunk, lo, hi, key=None):
    """Mismatches of bytes [lo, hi) of a segment with geometry (off, length, chunk)."""
    es = ES[dt]
    if hi <= lo:
        return 0
    want = _want(dt, inputs, got.size * es, off, length, chunk, lo, hi, key)
    a, b = lo // es, hi // es
    g, w = got[a:b], want[a:b]
    if kind != "nvls" or dt == oracle.I32:
        ib = np.uint16 if dt == oracle.BF16 else np.uint32
        return int(np.count_nonzero(g.view(ib) != w.view(ib)))
    if dt == oracle.F32:
        scale = np.sum([np.abs(x[a:b].astype(np.float64)) for x in inputs], axis=0)
        err = np.abs(g.astype(np.float64) - w.astype(np.float64)) / np.maximum(scale, 1e-30)
        return int(np.count_nonzero(err > 1e-6))
    gi, wi = g.astype(np.int64), w.astype(np.int64)
    same_sign = ((gi ^ wi) & 0x8000) == 0
    ulp = np.where(same_sign, np.abs(gi - wi), 2 * (g != w))
    return int(np.count_nonzero(ulp > 1))


def run(comm, spec) -> dict:
    rank, world = comm.rank, comm.world
    kinds = spec["rails"]
    over = {"kinds": kinds}
    for k in ("window", "eta", "demote_after", "calibrate_max_bytes", "calibrate_iters", "compute_pool", "pool_tokens",
              "graph_safe", "tune_budgets", "monitor", "detect_us", "heartbeat_us", "readmit_hold_us", "algorithm",
              "sync_overhead_us"):
        if k in spec:
            over[k] = spec[k]
    if "rails_toml" in spec:
        over["rails_toml"] = spec["rails_toml"]
    if os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB"):
        # tests/fakecuda emulates launches on the host, far slower than the
        # device: the monitor's heartbeat budget stretches with it.
        over["heartbeat_us"] = max(over.get("heartbeat_us", 50000.0), 50000.0) * 100
    eng = Engine(comm, **over)
    cap = max(c["nbytes"] for c in spec["cases"])
    bin_, bout = SymmetricBuffer(comm, cap), SymmetricBuffer(comm, cap)
    out = []
    for ci, c in enumerate(spec["cases"]):
        dt = DTYPES[c["dtype"]]
        n = c["nbytes"]
        inputs = cached(("in", ci, dt, n, world),
                        lambda: [oracle.synthetic_input(dt, r, n, seed_base=oracle.SEED_BASE + 131 * ci)
                                 for r in range(world)])
        for rep in range(c.get("reps", 1)):
            failing = bool(c.get("fail")) and rep == c.get("fail_rep", 0)
            if failing:  # every rank checks, so none is left waiting for the injecting one
                mon = eng.state()["monitor"]
                assert mon["on"], f"failure monitor off: {mon.get('off_reason')}"
            n_fo = len(eng.failovers())
            if failing and rank == c.get("fail_rank", world - 1):
                eng.inject_failure(eng.op_seq, c["fail"][0], c["fail"][1])
            got = np.zeros(n // ES[dt], dtype=oracle.NP_DTYPE[dt])
            if c.get("host"):
                eng.allreduce_host(inputs[rank], got, n, dt)
            elif c.get("graph"):  # graph-safe engine: capture `graph` allreduces, replay, check
                import torch
                torch.cuda.set_device(comm.device)
                bin_.write(inputs[rank], n)
                comm.barrier()
                eng.allreduce(bin_, bout, n, dt)  # eager warm-up (sizes CE staging)
                eng.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=torch.cuda.Stream()):
                    for _ in range(c["graph"]):
                        eng.allreduce(bin_, bout, n, dt, torch.cuda.current_stream())
                bout.zero()
                torch.cuda.synchronize()
                comm.barrier()
                g.replay()
                g.replay()
                torch.cuda.synchronize()
                eng.synchronize()
                bout.read(got, n)
            elif c.get("device") and os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB"):
                # tests/fakecuda: "device" memory is host memory there
                dev = inputs[rank].view(np.uint8).copy()
                comm.barrier()
                eng.allreduce_device(dev, dev, n, dt)
                eng.synchronize()
                got = dev.view(got.dtype).copy()
            elif c.get("device"):  # caller-owned device memory, in place (nz_engine_allreduce_device)
                import torch
                torch.cuda.set_device(comm.device)
                dev = torch.from_numpy(inputs[rank].view(np.uint8).copy()).cuda()
                comm.barrier()
                eng.allreduce_device(dev, dev, n, dt)
                eng.synchronize()
                got = dev.cpu().numpy().view(got.dtype).copy()
            else:
                bin_.write(inputs[rank], n)
                bout.zero()
                comm.barrier()
                eng.allreduce(bin_, bout, n, dt)
                eng.synchronize()
                bout.read(got, n)
            plans = eng.last_plans()
            fos = eng.failovers()[n_fo:]
            bad = 0
            segs = []
            for p in plans:
                for rail_id, off, length, chunk in p["segs"]:
                    kind = kinds[rail_id]
                    fo = next((f for f in fos if f["op_seq"] == p["op"] and f["failed_rail"] == rail_id), None)
                    if fo and fo["orphan_length"]:
                        # Chunks before the orphan: the failed rail's result; the
                        # orphan: the target rail's result, same geometry (P10).
                        k = fo["orphan_offset"]
                        bad += check_segment_range(kind, dt, got, inputs, off, length, chunk, off, k, key=ci)
                        bad += check_segment_range(kinds[fo["target_rail"]], dt, got, inputs, off, length, chunk, k,
                                                   off + length, key=ci)
                    else:
                        bad += check_segment_range(kind, dt, got, inputs, off, length, chunk, off, off + length,
                                                   key=ci)
                    segs.append([rail_id, off, length, chunk])
            rec = {"case": ci, "rep": rep, "dtype": c["dtype"], "nbytes": n, "mismatch": bad, "segs": segs,
                   "grants": [p["grants"] for p in plans if "grants" in p]}
            if failing:
                rec["failover"] = fos[0] if fos else None
                rec["failovers"] = fos
            out.append(rec)
        if c.get("readmit") and c.get("fail"):
            st = eng.state()
            if c["fail"][0] in st["monitor"]["failed"]:
                eng.readmit(c["fail"][0])
        # Every rank (process or virtual-rank thread) is done with case ci:
        # its inputs and oracle results (N x payload each) can go.
        comm.barrier()
        evict_case(ci)
    state = eng.state()
    eng.close()
    bin_.free()
    bout.free()
    return {"rank": rank, "results": out, "state": {"sync": state["sync_overhead_us"], "rails": state["rails"],
                                                     "compute_pool": state.get("compute_pool"),
                                                     "monitor": state.get("monitor")}}


def main():
    spec = json.loads(sys.argv[1])
    comm = Comm.from_env(session=os.environ["NZ_SESSION"])
    out = run(comm, spec)
    comm.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
