"""One rank of a rail parity run.

Two launch forms, the same checks:
  * a process per GPU (spawned by tests/mp_util.spawn): argv[1] = JSON cases,
    prints one JSON line;
  * a thread per virtual rank on one GPU (tests call ``run`` through
    paper_2405_17870_b200.run_ranks, nz_comm_init_loopback).

Each case reduces one segment geometry on one rail and compares this rank's
output buffer with the CPU oracle: bit-exact for the CE and SM rails
(P1/P2) and for int32 on every rail; NVLS fp32 within 1e-6 of
sum(|x|) per element, NVLS bf16 within one bf16 ulp of the oracle (P2).

A case with ``"stall": [rank, chunk]`` kills that rank's link of the rail at
that chunk (nz_rail_inject_stall, unplanned: the other ranks are not told)
and checks the device-side detection: every rank's launch fails, the peers'
end-barrier waits give up within the detection budget, the chunks of the
waves completed before the failure are exact, and after nz_rail_revive on
every rank the same op is exact again.
"""
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
from paper_2405_17870_b200 import Comm, Rail, SymmetricBuffer  # noqa: E402
from paper_2405_17870_b200._lib import DTYPES, RAIL_KINDS  # noqa: E402

# Virtual ranks share one process: inputs and oracle results are computed once.
_cache: dict = {}
_cache_lock = threading.Lock()


def clear_cache() -> None:
    with _cache_lock:
        _cache.clear()


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


def compare(kind, dtype, got, want, inputs, lo, hi, es):
    a, b = lo // es, hi // es
    g, w = got[a:b], want[a:b]
    if kind != "nvls" or dtype == oracle.I32:
        ibits = {np.dtype(np.float32): np.uint32, np.dtype(np.int32): np.uint32, np.dtype(np.uint16): np.uint16}
        bad = np.nonzero(g.view(ibits[g.dtype]) != w.view(ibits[w.dtype]))[0]
        return {"exact": True, "mismatch": int(bad.size), "first_bad": int(bad[0] + a) if bad.size else -1}
    if dtype == oracle.F32:
        scale = np.sum([np.abs(x[a:b].astype(np.float64)) for x in inputs], axis=0)
        err = np.abs(g.astype(np.float64) - w.astype(np.float64))
        rel = float(np.max(err / np.maximum(scale, 1e-30))) if err.size else 0.0
        return {"exact": False, "max_rel_sum_abs": rel, "mismatch": int(np.sum(err / np.maximum(scale, 1e-30) > 1e-6)),
                "bitexact_frac": float(np.mean(g == w)) if g.size else 1.0}
    gi, wi = g.astype(np.int32), w.astype(np.int32)
    ulp = np.abs(gi - wi)  # same-sign bf16 patterns: integer distance = ulps
    sign_flip = (gi ^ wi) & 0x8000
    ulp = np.where(sign_flip != 0, np.abs(oracle.bf16_to_f32(g) - oracle.bf16_to_f32(w)) > 0, ulp)
    return {"exact": False, "max_ulp": int(ulp.max()) if ulp.size else 0, "mismatch": int(np.sum(ulp > 1)),
            "bitexact_frac": float(np.mean(g == w)) if g.size else 1.0}


def _inputs(ci, dt, nbytes, world):
    return cached(("in", ci, dt, nbytes, world),
                  lambda: [oracle.synthetic_input(dt, r, nbytes, seed_base=oracle.SEED_BASE + 97 * ci)
                           for r in range(world)])


def _want(ci, dt, nbytes, world, seg_off, seg_len, chunk, lo, hi):
    def make():
        inputs = _inputs(ci, dt, nbytes, world)
        want = np.zeros(nbytes // (2 if dt == oracle.BF16 else 4), dtype=oracle.NP_DTYPE[dt])
        if hi > lo:
            oracle.reduce_range(inputs, dt, seg_off, seg_len, chunk, lo, hi, want)
        return want
    return cached(("want", ci, dt, nbytes, world, seg_off, seg_len, chunk, lo, hi), make)


def run(comm, cases) -> dict:
    rank, world = comm.rank, comm.world
    cap = max(c["nbytes"] for c in cases)
    bin_, bout = SymmetricBuffer(comm, cap), SymmetricBuffer(comm, cap)
    rails = {}
    results = []
    for ci, c in enumerate(cases):
        kind = c["kind"]
        gsafe = bool(c.get("graph") or c.get("graph_safe"))
        key = (kind, c.get("sm_budget", 0), gsafe)
        if key not in rails:
            rails[key] = Rail(comm, RAIL_KINDS[kind], len(rails), c.get("sm_budget", 0), graph_safe=gsafe)
        rail = rails[key]
        dt = DTYPES[c["dtype"]]
        es = 2 if dt == oracle.BF16 else 4
        nbytes = c["nbytes"]
        check = c.get("check", True)
        if check:
            inputs = _inputs(ci, dt, nbytes, world)
            mine = inputs[rank]
        else:  # timing-only case: this rank's synthetic input, no oracle comparison
            inputs = None
            mine = oracle.synthetic_input(dt, rank, nbytes, seed_base=oracle.SEED_BASE + 97 * ci)
        bin_.zero()
        bout.zero()
        bin_.write(mine, nbytes)
        seg_off, seg_len = c.get("seg_off", 0), c.get("seg_len", nbytes)
        chunk = c.get("chunk") or oracle.default_chunk_bytes(seg_len, world, c.get("chunked", True))
        nch = (seg_len + chunk - 1) // chunk
        ce = min(c.get("chunk_end", nch), nch)
        cb = min(c.get("chunk_begin", 0), ce)  # a window starting past the last chunk is empty
        fail = c.get("fail_chunk", -1)
        stall = c.get("stall")
        if stall:
            rail.set_detect_us(c.get("detect_us", 2000))
        comm.barrier()
        t0 = time.time()
        if stall and stall[0] == rank:
            rail.inject_stall(stall[1])
        if c.get("armed") and fail >= 0:  # nz_rail_inject_failure instead of the fail_chunk argument
            rail.inject_failure(fail)
            rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci, chunk_begin=cb, chunk_end=ce)
        else:
            rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci, chunk_begin=cb, chunk_end=ce,
                           fail_chunk=fail)
        rail.synchronize()
        seconds = time.time() - t0
        wd = rail.watchdog()
        progress = rail.progress()
        stop = fail if 0 <= fail < ce and fail >= cb else ce
        lo, hi = seg_off + min(seg_len, cb * chunk), seg_off + min(seg_len, stop * chunk)
        res = {"case": ci, "kind": kind, "dtype": c["dtype"], "nbytes": nbytes, "lo": lo, "hi": hi, "watchdog": wd,
               "progress": progress, "stop": min(stop, nch), "seconds": round(seconds, 4)}
        if stall:
            st = rail.status()
            res["status"] = {k: int(v) for k, v in st.items()}
            res["failed"] = st["ok_tag"] != st["start_tag"]  # the call's launches did not all succeed
            res["stalled_here"] = st["fail_tag"] == st["start_tag"] and st["t_fail_ns"] > 0
            res["detected_here"] = st["det_tag"] == st["start_tag"] and st["t_det_ns"] > 0
            # Chunks of the waves that completed everywhere before the death.
            hi = seg_off + min(seg_len, progress * chunk)
            res["hi"] = hi
        if check:
            got = np.zeros(nbytes // es, dtype=oracle.NP_DTYPE[dt])
            bout.read(got, nbytes)
            want = _want(ci, dt, nbytes, world, seg_off, seg_len, chunk, lo, hi)
            res.update(compare(kind, dt, got, want, inputs, lo, hi, es))
            if not stall:
                outside = np.concatenate([got[: lo // es], got[hi // es:]])
                res["outside_nonzero"] = int(np.count_nonzero(outside))
            else:
                res["outside_nonzero"] = 0
        rec = rail.poll_fault()
        res["fault"] = None if rec is None else {"op_seq": rec.op_seq, "chunk": rec.chunk}
        if stall:
            # Every rank revives the rail; the same op is then exact again.
            comm.barrier()
            rail.revive()
            rail.set_detect_us(0)
            comm.barrier()
            bout.zero()
            comm.barrier()
            rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci, chunk_begin=cb, chunk_end=ce)
            rail.synchronize()
            got = np.zeros(nbytes // es, dtype=oracle.NP_DTYPE[dt])
            bout.read(got, nbytes)
            lo2, hi2 = seg_off + min(seg_len, cb * chunk), seg_off + min(seg_len, ce * chunk)
            want = _want(ci, dt, nbytes, world, seg_off, seg_len, chunk, lo2, hi2)
            res["after_revive_mismatch"] = compare(kind, dt, got, want, inputs, lo2, hi2, es)["mismatch"]
            res["after_revive_watchdog"] = rail.watchdog()
        if c.get("graph") and check:
            # Graph-safe rail: capture `graph` ops (the eager op above was the
            # warm-up), replay three times, then one more eager op; every
            # result must equal the oracle.
            import torch
            torch.cuda.set_device(comm.device)
            want = _want(ci, dt, nbytes, world, seg_off, seg_len, chunk, lo, hi)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=torch.cuda.Stream()):
                for _ in range(c["graph"]):
                    rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci, chunk_begin=cb, chunk_end=ce,
                                   stream=torch.cuda.current_stream())
            bad = 0
            for rep in range(4):
                bout.zero()
                torch.cuda.synchronize()
                comm.barrier()
                if rep < 3:
                    g.replay()
                else:
                    rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci, chunk_begin=cb, chunk_end=ce)
                    rail.synchronize()
                torch.cuda.synchronize()
                got = np.zeros(nbytes // es, dtype=oracle.NP_DTYPE[dt])
                bout.read(got, nbytes)
                bad += compare(kind, dt, got, want, inputs, lo, hi, es)["mismatch"]
            res["graph_mismatch"] = bad
            res["watchdog"] = max(res["watchdog"], rail.watchdog())
        if c.get("graph_safe") and check:
            # Graph-safe rail run eagerly (no capture: the host harness): the
            # barrier epochs and LL flags / parities come from the device
            # launch counter; three more ops, each equal to the oracle.
            want = _want(ci, dt, nbytes, world, seg_off, seg_len, chunk, lo, hi)
            bad = 0
            for _ in range(3):
                bout.zero()
                comm.barrier()
                rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci, chunk_begin=cb, chunk_end=ce)
                rail.synchronize()
                got = np.zeros(nbytes // es, dtype=oracle.NP_DTYPE[dt])
                bout.read(got, nbytes)
                bad += compare(kind, dt, got, want, inputs, lo, hi, es)["mismatch"]
            res["graph_mismatch"] = bad
            res["watchdog"] = max(res["watchdog"], rail.watchdog())
        iters = c.get("iters", 0)
        if iters:
            import torch
            torch.cuda.set_device(comm.device)
            st = torch.cuda.ExternalStream(rail.stream)
            for _ in range(3):
                rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci)
            comm.barrier()
            rail.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(iters):
                rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci)
            e1.record(st)
            rail.synchronize()
            t = e0.elapsed_time(e1) / iters / 1e3
            res["us"] = t * 1e6
            res["busbw_GBs"] = 2 * (world - 1) / world * seg_len / t / 1e9 if world > 1 else 0.0
            res["algbw_GBs"] = seg_len / t / 1e9
        if c.get("abort"):
            from paper_2405_17870_b200 import NezhaError
            rail.abort()
            try:
                rail.allreduce(bin_, bout, seg_off, seg_len, chunk, dt, op_seq=ci)
                res["abort_refused"] = False
            except NezhaError:
                res["abort_refused"] = True
            rails[key] = Rail(comm, RAIL_KINDS[kind], len(rails) + 10, c.get("sm_budget", 0))
            rail.close()
        results.append(res)
    for r in rails.values():
        r.close()
    bin_.free()
    bout.free()
    return {"rank": rank, "results": results}


def main():
    cases = json.loads(sys.argv[1])
    comm = Comm.from_env(session=os.environ["NZ_SESSION"])
    out = run(comm, cases)
    comm.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
