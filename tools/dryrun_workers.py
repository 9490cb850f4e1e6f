"""Development aid, CPU only: runs the GPU tests' worker logic
(tests/workers/rail_worker.py, engine_worker.py) against FAKE runtime objects
whose results come from the CPU oracle, so the Python paths of the loopback
tests (virtual-rank threads, stall / failover bookkeeping, checks) can be
exercised before a GPU is available. Nothing here touches the product's CUDA
path; it checks the test harness, not the library.

    python tools/dryrun_workers.py
"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import planner as P  # noqa: E402
from paper_2405_17870_b200.runtime import Planner  # noqa: E402  (CPU balancer through the ABI)

WAVE = 64 << 20
ES = {0: 4, 1: 2, 2: 4}


class Group:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.lock = threading.Lock()
        self.slots = {}


class FakeComm:
    def __init__(self, rank, group):
        self.rank, self.world, self.device, self.group = rank, group.world, 0, group
        self.loopback = True
        self.multicast = False

    def barrier(self):
        self.group.bar.wait()

    def allgather_bytes(self, data):
        g = self.group
        with g.lock:
            g.slots[self.rank] = data
        g.bar.wait()
        out = [g.slots[r] for r in range(self.world)]
        g.bar.wait()
        return out

    def gather(self, key, value):
        """Every rank's value for `key` (a collective)."""
        g = self.group
        with g.lock:
            g.slots[(key, self.rank)] = value
        g.bar.wait()
        out = [g.slots[(key, r)] for r in range(self.world)]
        g.bar.wait()
        return out

    def close(self):
        pass


class FakeBuffer:
    def __init__(self, comm, nbytes):
        self.comm, self.nbytes = comm, nbytes
        self.mem = np.zeros(nbytes, dtype=np.uint8)

    def write(self, src, nbytes, offset=0, stream=None):
        self.mem[offset:offset + nbytes] = np.asarray(src).view(np.uint8).reshape(-1)[:nbytes]

    def read(self, dst, nbytes, offset=0, stream=None):
        np.asarray(dst).view(np.uint8).reshape(-1)[:nbytes] = self.mem[offset:offset + nbytes]

    def zero(self, stream=None):
        self.mem[:] = 0

    def free(self):
        pass


def typed(buf, dt):
    return buf.mem.view(oracle.NP_DTYPE[dt])


class FakeRail:
    """One rail call = a collective over the group; results from the oracle."""

    def __init__(self, comm, kind, rail_id, sm_budget=0, graph_safe=False):
        self.comm, self.kind, self.rail_id = comm, kind, rail_id
        self.stall = None
        self.armed = -1
        self.tag = 0
        self.st = {"ok_tag": 0, "prog_tag": 0, "prog_chunk": 0, "start_tag": 0, "fail_tag": 0, "t_start_ns": 0,
                   "t_fail_ns": 0, "det_tag": 0, "abort": 0, "t_det_ns": 0}
        self.wd = 0
        self.fault = None
        self.prog = 0
        self.dead = False
        self.aborted = False
        self.stream = 0

    def allreduce(self, inp, out, seg_off, seg_len, chunk, dt, op_seq=0, chunk_begin=0, chunk_end=1 << 62,
                  fail_chunk=-1, stream=None):
        if self.aborted:
            from paper_2405_17870_b200 import NezhaError
            raise NezhaError("aborted")
        if fail_chunk < 0 and self.armed >= 0:
            fail_chunk = self.armed
        self.armed = -1
        c = self.comm
        nch = -(-seg_len // chunk)
        ce = min(chunk_end, nch)
        stop = fail_chunk if 0 <= fail_chunk < ce and fail_chunk >= chunk_begin else ce
        stall = self.stall
        self.stall = None
        stalls = c.gather(("stall", self.rail_id), (stall, self.dead))
        self.tag += 1
        self.st["start_tag"] = self.tag
        lo, hi = seg_off + min(seg_len, chunk_begin * chunk), seg_off + min(seg_len, stop * chunk)
        dead_any = [r for r, (s, d) in enumerate(stalls) if d or (s is not None and chunk_begin <= s < stop)]
        prog_end = stop
        if dead_any:
            ks = [P.completed_before_stall(chunk, chunk_begin, stop, s if s is not None else chunk_begin, WAVE)
                  for (s, d) in stalls if d or s is not None]
            prog_end = min(ks)
            if stall is not None or self.dead:
                self.st["fail_tag"], self.st["t_fail_ns"] = self.tag, 1
                self.dead = True
            else:
                self.st["det_tag"], self.st["t_det_ns"] = self.tag, 1
                self.wd = 1
            hi = seg_off + min(seg_len, prog_end * chunk)
        ins = c.gather(("in", self.rail_id, self.tag), typed(inp, dt).copy())
        if hi > lo:
            oracle.reduce_range(ins, dt, seg_off, seg_len, chunk, lo, hi, typed(out, dt))
        c.gather(("done", self.rail_id, self.tag), 0)
        self.st["prog_tag"], self.st["prog_chunk"] = self.tag, prog_end
        if not dead_any:
            self.st["ok_tag"] = self.tag
            if stop != ce:
                self.fault = {"op_seq": op_seq, "chunk": stop}
        self.prog = prog_end

    def synchronize(self):
        pass

    def watchdog(self):
        w, self.wd = self.wd, 0
        return w

    def progress(self):
        return self.prog

    def status(self):
        return dict(self.st)

    def inject_stall(self, chunk):
        self.stall = chunk

    def inject_failure(self, chunk):
        self.armed = chunk

    def revive(self):
        self.dead = False

    def set_detect_us(self, us):
        pass

    def poll_fault(self, consume=True):
        f = self.fault
        if consume:
            self.fault = None
        if f is None:
            return None
        return type("R", (), f)

    def abort(self):
        self.aborted = True

    def close(self):
        pass


class FakeEngine:
    """Plans with the product's CPU balancer; results from the oracle; an
    injected stall on one rank becomes the monitor's agreed reroute."""

    def __init__(self, comm, kinds=None, rails_toml=None, **kw):
        self.comm, self.kinds = comm, kinds
        self.planner = Planner(rails_toml, sync_overhead_us=kw.get("sync_overhead_us", 0.0) or 0.0,
                               window=kw.get("window", 100))
        self.op_seq = 0
        self.inject = {}
        self.plans = []
        self.fos = []
        self.failed = set()

    def allreduce(self, inp, out, nbytes, dt, stream=None):
        c = self.comm
        plan = self.planner.allocate(nbytes)
        inj = c.gather(("inj", self.op_seq), self.inject.pop(self.op_seq, None))
        ins = c.gather(("ein", self.op_seq), typed(inp, dt)[: nbytes // ES[dt]].copy())
        o = typed(out, dt)
        segs = []
        for rail, off, length in plan["segs"]:
            C = oracle.default_chunk_bytes(length, c.world)
            oracle.reduce_range(ins, dt, off, length, C, off, off + length, o[: nbytes // ES[dt]])
            segs.append([rail, off, length, C])
            for r_, x in enumerate(inj):
                if x and x[0] == rail:
                    nch = -(-length // C)
                    k = P.completed_before_stall(C, 0, nch, x[1], WAVE)
                    if k < nch:
                        others = [s_[0] for s_ in plan["segs"] if s_[0] != rail] or [rail]
                        self.fos.append({"op_seq": self.op_seq, "failed_rail": rail, "target_rail": others[0],
                                         "orphan_offset": off + k * C, "orphan_length": length - k * C,
                                         "orphan_chunk": k, "stalled_here": int(r_ == c.rank), "detect_us": 5000.0,
                                         "resume_after_detect_us": 120.0, "resume_us": 5100.0, "done_us": 5300.0})
                        self.failed.add(rail)
        self.plans = [{"op": self.op_seq, "hot": plan["hot"], "segs": segs}]
        self.op_seq += 1

    def allreduce_host(self, hin, hout, nbytes, dt):
        b_in, b_out = FakeBuffer(self.comm, nbytes), FakeBuffer(self.comm, nbytes)
        b_in.write(hin, nbytes)
        self.allreduce(b_in, b_out, nbytes, dt)
        b_out.read(hout, nbytes)

    def synchronize(self):
        pass

    def inject_failure(self, op_seq, rail, chunk):
        self.inject[op_seq] = (rail, chunk)

    def last_plans(self):
        return self.plans

    def failovers(self):
        return list(self.fos)

    def readmit(self, rail):
        self.failed.discard(rail)

    def state(self):
        return {"sync_overhead_us": 0.0, "rails": [], "compute_pool": None,
                "monitor": {"on": True, "off_reason": "", "failed": sorted(self.failed)}}

    def close(self):
        pass


def run_ranks(world, fn):
    g = Group(world)
    res, err = [None] * world, [None] * world

    def body(r):
        try:
            res[r] = fn(FakeComm(r, g))
        except BaseException as e:  # noqa: BLE001
            import traceback
            err[r] = traceback.format_exc()
            g.bar.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if any(err):
        raise RuntimeError("\n".join(e for e in err if e))
    return res


def main():
    from tests.workers import engine_worker, rail_worker
    import tests.test_gpu_vranks as T

    saved = {(m, n): getattr(m, n) for m in (rail_worker, engine_worker) for n in ("Rail", "SymmetricBuffer", "Engine")
             if hasattr(m, n)}
    for (m, n) in saved:
        setattr(m, n, {"Rail": FakeRail, "SymmetricBuffer": FakeBuffer, "Engine": FakeEngine}[n])
    try:
        _dry(rail_worker, engine_worker, T)
    finally:
        for (m, n), v in saved.items():  # the real objects again for anything running after this
            setattr(m, n, v)
        rail_worker.clear_cache()
        engine_worker.clear_cache()
    print("dry run ok")


def _dry(rail_worker, engine_worker, T):
    # rail parity cases (the abort case recreates rails)
    for world in (2, 4):
        res = run_ranks(world, lambda c: rail_worker.run(c, [x for x in T.RAIL_CASES if x["nbytes"] <= (8 << 20)]))
        T._check_rails(res, [x for x in T.RAIL_CASES if x["nbytes"] <= (8 << 20)])
        rail_worker.clear_cache()
    # stall cases
    for world in (2, 4):
        cases = [{"kind": "sm", "dtype": "f32", "nbytes": 160 << 20, "stall": [world - 1, 7 if world >= 4 else 3]},
                 {"kind": "sm", "dtype": "i32", "nbytes": 1 << 20, "stall": [0, 0]}]
        res = run_ranks(world, lambda c: rail_worker.run(c, cases))
        for rk in res:
            for r in rk["results"]:
                assert r["failed"] and r["mismatch"] == 0 and r["after_revive_mismatch"] == 0, r
        rail_worker.clear_cache()
    # engine failover case
    spec = {"rails": T.KINDS3, "rails_toml": T.TOML_LOOP, "sync_overhead_us": 0.0,
            "cases": [{"dtype": "bf16", "nbytes": 64 << 20, "reps": 3, "fail": [1, 5], "fail_rep": 1},
                      {"dtype": "f32", "nbytes": 1 << 20, "reps": 1, "host": True},
                      {"dtype": "i32", "nbytes": 16 << 20, "reps": 1, "readmit": True}]}
    res = run_ranks(4, lambda c: engine_worker.run(c, spec))
    for rk in res:
        for r in rk["results"]:
            assert r["mismatch"] == 0, r
    fo = [r for r in res[0]["results"] if "failover" in r][0]["failover"]
    assert fo and fo["failed_rail"] == 1, fo


if __name__ == "__main__":
    main()
