"""One rank of a multi-GPU engine run (spawned by tests/mp_util.spawn).

argv[1] = JSON {"rails": [...kinds], "cases": [...]} where each case is
{"dtype", "nbytes", "reps", "fail": [rail, chunk] | null, "host": bool}.
Every op's output is compared with the CPU oracle evaluated on the plan the
engine reports it ran (nz_engine_last_plan_json): bit-exact on CE/SM
segments and int32, NVLS fp32 within 1e-6 of sum|x|, NVLS bf16 within 1 ulp.
A failure case also checks the rerouted result and reports the failover times.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
from paper_2405_17870_b200 import Comm, Engine, SymmetricBuffer  # noqa: E402
from paper_2405_17870_b200._lib import DTYPES, RAIL_KINDS  # noqa: E402

ES = {oracle.F32: 4, oracle.BF16: 2, oracle.I32: 4}


def check_segment(kind, dt, got, inputs, off, length, chunk):
    return check_segment_range(kind, dt, got, inputs, off, length, chunk, off, off + length)


def check_segment_range(kind, dt, got, inputs, off, length, chunk, lo, hi):
    """Mismatches of bytes [lo, hi) of a segment with geometry (off, length, chunk)."""
    es = ES[dt]
    if hi <= lo:
        return 0
    want = np.zeros_like(got)
    oracle.reduce_range(inputs, dt, off, length, chunk, lo, hi, want)
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


def main():
    spec = json.loads(sys.argv[1])
    comm = Comm.from_env(session=os.environ["NZ_SESSION"])
    rank, world = comm.rank, comm.world
    kinds = spec["rails"]
    over = {"kinds": kinds}
    for k in ("window", "eta", "demote_after", "calibrate_max_bytes", "calibrate_iters", "compute_pool", "pool_tokens",
              "graph_safe", "tune_budgets"):
        if k in spec:
            over[k] = spec[k]
    if "rails_toml" in spec:
        over["rails_toml"] = spec["rails_toml"]
    eng = Engine(comm, **over)
    cap = max(c["nbytes"] for c in spec["cases"])
    bin_, bout = SymmetricBuffer(comm, cap), SymmetricBuffer(comm, cap)
    out = []
    for ci, c in enumerate(spec["cases"]):
        dt = DTYPES[c["dtype"]]
        n = c["nbytes"]
        inputs = [oracle.synthetic_input(dt, r, n, seed_base=oracle.SEED_BASE + 131 * ci) for r in range(world)]
        for rep in range(c.get("reps", 1)):
            if c.get("fail") and rep == c.get("fail_rep", 0):
                inj_seq = eng.op_seq
                eng.inject_failure(inj_seq, c["fail"][0], c["fail"][1])
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
            failing = c.get("fail") and rep == c.get("fail_rep", 0)
            fo = eng.last_failover() if failing else None
            if fo is not None and fo["op_seq"] != inj_seq:
                fo = None  # the failed rail carried nothing of this op (idle failure): no reroute
            bad = 0
            segs = []
            for p in plans:
                for rail_id, off, length, chunk in p["segs"]:
                    kind = kinds[rail_id]
                    if fo and rail_id == fo["failed_rail"] and fo["orphan_length"] and \
                            off <= fo["orphan_offset"] < off + length:
                        # Chunks before the failure: the failed rail's result; the
                        # orphan: the target rail's result, same geometry (P10).
                        k = fo["orphan_offset"]
                        bad += check_segment_range(kind, dt, got, inputs, off, length, chunk, off, k)
                        bad += check_segment_range(kinds[fo["target_rail"]], dt, got, inputs, off, length, chunk, k,
                                                   off + length)
                    else:
                        bad += check_segment(kind, dt, got, inputs, off, length, chunk)
                    segs.append([rail_id, off, length, chunk])
            rec = {"case": ci, "rep": rep, "dtype": c["dtype"], "nbytes": n, "mismatch": bad, "segs": segs,
                   "grants": [p["grants"] for p in plans if "grants" in p]}
            if failing:
                rec["failover"] = fo
            out.append(rec)
        if c.get("readmit") and c.get("fail"):
            eng.readmit(c["fail"][0])
    state = eng.state()
    eng.close()
    bin_.free()
    bout.free()
    comm.close()
    print(json.dumps({"rank": rank, "results": out, "state": {"sync": state["sync_overhead_us"],
                                                               "rails": state["rails"],
                                                               "compute_pool": state.get("compute_pool")}}))


if __name__ == "__main__":
    main()
