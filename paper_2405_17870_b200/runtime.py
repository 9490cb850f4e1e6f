"""Python mirror of the C ABI objects: Comm, SymmetricBuffer, Rail, Engine.

Thin wrappers: every operation is a call into libnezha_b200.so. Device memory
is the library's own symmetric VMM allocation (the UnboundBuffer); torch is
only used by callers for streams and host tensors.
"""
from __future__ import annotations

import ctypes
import json
import os
from ctypes import byref, c_void_p

from . import _lib
from ._lib import check, lib


def _ptr(x) -> int | None:
    """Accepts an int address, a ctypes pointer, a numpy array or a torch tensor."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    return ctypes.cast(x, c_void_p).value


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


class Comm:
    """One rank of the job (nz_comm_init). Replaces rendezvous() (transport.hpp:219-238).

    ``loopback=True`` (nz_comm_init_loopback): one virtual rank of a job whose
    ranks are threads of this process on one GPU (see loopback.run_ranks)."""

    def __init__(self, rank: int, world: int, device: int, session: str, timeout_ms: int = 120000,
                 loopback: bool = False):
        h = c_void_p()
        fn = lib().nz_comm_init_loopback if loopback else lib().nz_comm_init
        check(fn(rank, world, device, session.encode(), timeout_ms, byref(h)),
              "nz_comm_init_loopback" if loopback else "nz_comm_init")
        self.handle = h
        self.rank, self.world, self.device = rank, world, device
        self.loopback = loopback

    @classmethod
    def from_env(cls, session: str | None = None, timeout_ms: int = 120000) -> "Comm":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        local = int(os.environ.get("LOCAL_RANK", str(rank)))
        if session is None:
            session = f"{os.environ.get('MASTER_PORT', '0')}-{os.environ.get('TORCHELASTIC_RUN_ID', 'nz')}"
        return cls(rank, world, local, session, timeout_ms)

    @property
    def multicast(self) -> bool:
        return lib().nz_comm_multicast_supported(self.handle) == 1

    @property
    def sm_count(self) -> int:
        return lib().nz_comm_sm_count(self.handle)

    def barrier(self) -> None:
        check(lib().nz_comm_barrier(self.handle), "nz_comm_barrier")

    def allgather_bytes(self, data: bytes) -> list[bytes]:
        n = len(data)
        out = ctypes.create_string_buffer(n * self.world)
        check(lib().nz_comm_allgather(self.handle, data, n, out), "nz_comm_allgather")
        raw = out.raw
        return [raw[i * n:(i + 1) * n] for i in range(self.world)]

    def abort(self) -> None:
        """Loopback: fail every virtual rank still waiting on this group."""
        if self.handle:
            check(lib().nz_comm_abort(self.handle), "nz_comm_abort")

    def close(self) -> None:
        if self.handle:
            check(lib().nz_comm_destroy(self.handle), "nz_comm_destroy")
            self.handle = None


class SymmetricBuffer:
    """nz_buffer_alloc: the UnboundBuffer."""

    def __init__(self, comm: Comm, nbytes: int):
        h = c_void_p()
        check(lib().nz_buffer_alloc(comm.handle, nbytes, byref(h)), "nz_buffer_alloc")
        self.handle = h
        self.comm = comm
        self.nbytes = nbytes

    @property
    def ptr(self) -> int:
        return lib().nz_buffer_ptr(self.handle)

    @property
    def mc_ptr(self) -> int | None:
        return lib().nz_buffer_mc_ptr(self.handle)

    def write(self, src, nbytes: int, offset: int = 0, stream=None) -> None:
        check(lib().nz_buffer_write(self.handle, offset, _ptr(src), nbytes, _stream(stream)), "nz_buffer_write")

    def read(self, dst, nbytes: int, offset: int = 0, stream=None) -> None:
        check(lib().nz_buffer_read(self.handle, offset, _ptr(dst), nbytes, _stream(stream)), "nz_buffer_read")

    def zero(self, stream=None) -> None:
        check(lib().nz_buffer_fill_zero(self.handle, _stream(stream)), "nz_buffer_fill_zero")

    def free(self) -> None:
        if self.handle:
            check(lib().nz_buffer_free(self.handle), "nz_buffer_free")
            self.handle = None


class Rail:
    """One rail's executor on this rank (nz_rail_create)."""

    def __init__(self, comm: Comm, kind: int, rail_id: int, sm_budget: int = 0, graph_safe: bool = False):
        h = c_void_p()
        check(lib().nz_rail_create_ex(comm.handle, kind, rail_id, sm_budget, 1 if graph_safe else 0, byref(h)),
              "nz_rail_create_ex")
        self.handle = h
        self.kind = kind
        self.rail_id = rail_id

    @property
    def stream(self) -> int:
        return lib().nz_rail_stream(self.handle)

    def allreduce(self, inp: SymmetricBuffer, out: SymmetricBuffer, seg_off: int, seg_len: int, chunk_bytes: int,
                  dtype: int, op_seq: int = 0, chunk_begin: int = 0, chunk_end: int = 1 << 62,
                  fail_chunk: int = -1, stream=None) -> None:
        check(lib().nz_rail_allreduce(self.handle, inp.handle, out.handle, seg_off, seg_len, chunk_bytes, chunk_begin,
                                      chunk_end, dtype, op_seq, fail_chunk, _stream(stream)), "nz_rail_allreduce")

    def synchronize(self) -> None:
        check(lib().nz_rail_synchronize(self.handle), "nz_rail_synchronize")

    def poll_fault(self, consume: bool = True) -> _lib.FaultRecord | None:
        rec = _lib.FaultRecord()
        check(lib().nz_rail_poll_fault(self.handle, byref(rec), 1 if consume else 0), "nz_rail_poll_fault")
        return rec if rec.valid else None

    def watchdog(self) -> int:
        return lib().nz_rail_watchdog(self.handle)

    def inject_failure(self, chunk: int) -> None:
        """Arms a failure at `chunk` for this rank's next allreduce (nz_rail_inject_failure)."""
        check(lib().nz_rail_inject_failure(self.handle, chunk), "nz_rail_inject_failure")

    def inject_stall(self, chunk: int) -> None:
        """This rank's link dies at `chunk` of its next allreduce (nz_rail_inject_stall); peers are not told."""
        check(lib().nz_rail_inject_stall(self.handle, chunk), "nz_rail_inject_stall")

    def revive(self) -> None:
        """Clears a failed launch state on this rank (nz_rail_revive); call on every rank."""
        check(lib().nz_rail_revive(self.handle), "nz_rail_revive")

    def set_detect_us(self, us: float) -> None:
        check(lib().nz_rail_set_detect_us(self.handle, float(us)), "nz_rail_set_detect_us")

    def status(self) -> dict:
        """nz_rail_status: the launch status record this rank's kernels publish."""
        st = _lib.RailStatus()
        check(lib().nz_rail_status(self.handle, ctypes.byref(st)), "nz_rail_status")
        return {f: getattr(st, f) for f, _ in st._fields_}

    def progress(self) -> int:
        """Chunks of the last allreduce complete on this rank (nz_rail_progress)."""
        v = ctypes.c_uint64(0)
        check(lib().nz_rail_progress(self.handle, byref(v)), "nz_rail_progress")
        return v.value

    def abort(self) -> None:
        """Kills the rail on this rank (nz_rail_abort); later calls raise ChannelDownError."""
        check(lib().nz_rail_abort(self.handle), "nz_rail_abort")

    def close(self) -> None:
        if self.handle:
            check(lib().nz_rail_destroy(self.handle), "nz_rail_destroy")
            self.handle = None


def default_engine_config() -> _lib.EngineConfig:
    cfg = _lib.EngineConfig()
    lib().nz_engine_config_default(byref(cfg))
    return cfg


class Engine:
    """Multi-rail allreduce engine (nz_engine_*): planner + rails + monitor."""

    def __init__(self, comm: Comm, cfg: _lib.EngineConfig | None = None, **overrides):
        cfg = cfg or default_engine_config()
        for k, v in overrides.items():
            if k == "kinds":
                cfg.num_rails = len(v)
                for i, kind in enumerate(v):
                    cfg.kinds[i] = _lib.RAIL_KINDS[kind] if isinstance(kind, str) else kind
            elif k == "sm_budget":
                for i, b in enumerate(v):
                    cfg.sm_budget[i] = b
            elif k == "rails_toml":
                self._toml = v.encode() if isinstance(v, str) else v
                cfg.rails_toml = self._toml
            else:
                setattr(cfg, k, v)
        h = c_void_p()
        check(lib().nz_engine_create(comm.handle, byref(cfg), byref(h)), "nz_engine_create")
        self.handle = h
        self.comm = comm

    def allreduce(self, inp: SymmetricBuffer, out: SymmetricBuffer, nbytes: int, dtype: int, stream=None) -> None:
        check(lib().nz_engine_allreduce(self.handle, inp.handle, out.handle, nbytes, dtype, _stream(stream)),
              "nz_engine_allreduce")

    def allreduce_host(self, host_in, host_out, nbytes: int, dtype: int) -> None:
        check(lib().nz_engine_allreduce_host(self.handle, _ptr(host_in), _ptr(host_out), nbytes, dtype),
              "nz_engine_allreduce_host")

    def allreduce_device(self, src, dst, nbytes: int, dtype: int, stream=None) -> None:
        """Allreduce of caller-owned device memory (nz_engine_allreduce_device); src may equal dst."""
        check(lib().nz_engine_allreduce_device(self.handle, _ptr(src), _ptr(dst), nbytes, dtype, _stream(stream)),
              "nz_engine_allreduce_device")

    def inject_failure(self, op_seq: int, rail_id: int, chunk: int) -> None:
        check(lib().nz_engine_inject_failure(self.handle, op_seq, rail_id, chunk), "nz_engine_inject_failure")

    def readmit(self, rail_id: int) -> None:
        check(lib().nz_engine_readmit(self.handle, rail_id), "nz_engine_readmit")

    def synchronize(self) -> None:
        check(lib().nz_engine_synchronize(self.handle), "nz_engine_synchronize")

    @property
    def op_seq(self) -> int:
        return lib().nz_engine_op_seq(self.handle)

    def last_failover(self) -> dict | None:
        rep = _lib.FailoverReport()
        rc = lib().nz_engine_last_failover(self.handle, byref(rep))
        if rc == _lib.NZ_ERR_INVALID:
            return None
        check(rc, "nz_engine_last_failover")
        return {f: getattr(rep, f) for f, _ in rep._fields_}

    def loop_timing(self, rail_id: int, enable: bool = True) -> None:
        """Loopback: time every cross-rank grid of the rail on its own stream (nz_rail_loop_timing)."""
        check(lib().nz_rail_loop_timing(lib().nz_engine_rail(self.handle, rail_id), 1 if enable else 0),
              "nz_rail_loop_timing")

    def loop_time(self, rail_id: int) -> dict:
        """Launches and summed device time of the rail's loopback grids since the last read."""
        n, us = ctypes.c_uint64(), ctypes.c_double()
        check(lib().nz_rail_loop_time(lib().nz_engine_rail(self.handle, rail_id), byref(n), byref(us)),
              "nz_rail_loop_time")
        return {"launches": n.value, "total_us": us.value}

    def failovers(self) -> list[dict]:
        """Every failover the monitor handled so far, in order (nz_engine_failover_get)."""
        n = check(lib().nz_engine_failover_count(self.handle), "nz_engine_failover_count")
        out = []
        for i in range(n):
            rep = _lib.FailoverReport()
            check(lib().nz_engine_failover_get(self.handle, i, byref(rep)), "nz_engine_failover_get")
            out.append({f: getattr(rep, f) for f, _ in rep._fields_})
        return out

    def _json(self, fn, *args) -> dict:
        cap = 1 << 16
        while True:
            buf = ctypes.create_string_buffer(cap)
            rc = fn(self.handle, *args, buf, cap)
            if rc == _lib.NZ_ERR_BUFFER:
                cap *= 4
                continue
            check(rc)
            return json.loads(buf.value.decode())

    def state(self) -> dict:
        return self._json(lib().nz_engine_state_json)

    def plan(self, nbytes: int) -> dict:
        return self._json(lib().nz_engine_plan_json, nbytes)

    def last_plans(self) -> list:
        return self._json(lib().nz_engine_last_plan_json)

    def rail_stats(self, rail_id: int) -> dict:
        ops, us, nbytes = ctypes.c_uint64(), ctypes.c_double(), ctypes.c_uint64()
        check(lib().nz_engine_rail_stats(self.handle, rail_id, byref(ops), byref(us), byref(nbytes)),
              "nz_engine_rail_stats")
        return {"ops": ops.value, "total_us": us.value, "bytes": nbytes.value}

    def stats_reset(self) -> None:
        check(lib().nz_engine_stats_reset(self.handle), "nz_engine_stats_reset")

    def save_state(self) -> str:
        """AllocationTable + profiles as JSON (--balancer-state)."""
        return json.dumps(self._json(lib().nz_engine_save_state))

    def load_state(self, text: str) -> None:
        check(lib().nz_engine_load_state(self.handle, text.encode()), "nz_engine_load_state")

    def close(self) -> None:
        if self.handle:
            check(lib().nz_engine_destroy(self.handle), "nz_engine_destroy")
            self.handle = None


def kernel_launch_count() -> int:
    """Kernels libnezha_b200.so has launched in this process (nz_kernel_launch_count)."""
    return int(lib().nz_kernel_launch_count())


def run_trace(scenario: str) -> str:
    """Planner decisions for a scenario (nz_planner_run_trace), CPU only."""
    cap = 1 << 20
    while True:
        buf = ctypes.create_string_buffer(cap)
        rc = lib().nz_planner_run_trace(scenario.encode(), buf, cap)
        if rc == _lib.NZ_ERR_BUFFER:
            cap *= 8
            continue
        check(rc, "nz_planner_run_trace")
        return buf.value.decode()


def emulate_fold(world: int, rank: int, dtype: int, srcs: list[int], dsts: list[int], seg_off: int, seg_len: int,
                 chunk_bytes: int, lo: int, hi: int, grid: int = 0, stream=None) -> None:
    """Single-GPU emulation of one rank of the SM / CE rail fold kernels (nz_emulate_fold)."""
    s = (c_void_p * len(srcs))(*srcs)
    d = (c_void_p * len(dsts))(*dsts)
    check(lib().nz_emulate_fold(world, rank, dtype, s, d, len(dsts), seg_off, seg_len, chunk_bytes, lo, hi, grid,
                                _stream(stream)), "nz_emulate_fold")


class ComputePool:
    """Per-phase compute tokens (nz_pool_*, include/nezha/compute_pool.hpp).

    Mirrors acquire_phase_tokens / release_phase_tokens: phase 0 io, 1
    communication, 2 computation. ``try_acquire`` returns None when
    ``acquire`` would block."""

    IO, COMMUNICATION, COMPUTATION = 0, 1, 2

    def __init__(self, total_tokens: int):
        self._h = None
        h = c_void_p()
        check(lib().nz_pool_create(total_tokens, ctypes.byref(h)), "nz_pool_create")
        self._h = h

    def close(self) -> None:
        if self._h:
            lib().nz_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def declare(self, rail_id: int, computation: int, io: int = 1, communication: int = 1) -> None:
        check(lib().nz_pool_declare(self._h, rail_id, io, communication, computation), "nz_pool_declare")

    def _acquire(self, rail_id: int, phase: int, blocking: int) -> int:
        g = ctypes.c_int(0)
        check(lib().nz_pool_acquire(self._h, rail_id, phase, blocking, ctypes.byref(g)), "nz_pool_acquire")
        return g.value

    def acquire(self, rail_id: int, phase: int) -> int:
        return self._acquire(rail_id, phase, 1)

    def try_acquire(self, rail_id: int, phase: int) -> int | None:
        g = self._acquire(rail_id, phase, 0)
        return None if g < 0 else g

    def release(self, rail_id: int, phase: int) -> None:
        check(lib().nz_pool_release(self._h, rail_id, phase), "nz_pool_release")

    @property
    def outstanding(self) -> int:
        return check(lib().nz_pool_outstanding(self._h), "nz_pool_outstanding")

    @property
    def waiting(self) -> int:
        return check(lib().nz_pool_waiting(self._h), "nz_pool_waiting")


def plan_compute_grants(total_tokens: int, mode: int, demands: list[tuple[int, int]]) -> list[dict]:
    """The engine's per-op SM arbitration (nz_pool_plan): per rail {rail, demand, grant, waits}."""
    n = len(demands)
    ids = (ctypes.c_int * max(n, 1))(*[r for r, _ in demands])
    dem = (ctypes.c_int * max(n, 1))(*[d for _, d in demands])
    grants = (ctypes.c_int * max(n, 1))()
    masks = (ctypes.c_uint32 * max(n, 1))()
    check(lib().nz_pool_plan(total_tokens, mode, n, ids, dem, grants, masks), "nz_pool_plan")
    out = []
    for i, (r, d) in enumerate(demands):
        waits = [rr for rr, _ in demands[:i] if masks[i] >> rr & 1]
        out.append({"rail": r, "demand": d, "grant": grants[i], "waits": waits})
    return out


def calibrate(samples: list[tuple[int, float]]) -> dict:
    """calibrate(samples) -> CalibratedProfile (nz_core_calibrate)."""
    n = len(samples)
    xs = (ctypes.c_uint64 * max(n, 1))(*[int(x) for x, _ in samples])
    ys = (ctypes.c_double * max(n, 1))(*[float(y) for _, y in samples])
    t, bw, mr = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    it = ctypes.c_int()
    check(lib().nz_core_calibrate(xs, ys, n, byref(t), byref(bw), byref(it), byref(mr)), "nz_core_calibrate")
    return {"t_setup_us": t.value, "bandwidth_bps": bw.value, "interpolated": bool(it.value),
            "max_rel_residual": mr.value}


class Planner:
    """The engine's balancer driven op by op (nz_balancer_*), no GPU.

    ``agree(bucket, rail_ids, means) -> means`` is the multi-rank flush
    agreement (the engine: max over ranks); None = single process."""

    def __init__(self, rails_toml: str, tau: float = 5.0, eta: float = 0.05, sync_overhead_us: float = 0.0,
                 window: int = 100, demote_after: int = 0, agree=None):
        self._h = None
        h = c_void_p()
        self._toml = rails_toml.encode()
        check(lib().nz_balancer_create(self._toml, tau, eta, sync_overhead_us, window, demote_after, byref(h)),
              "nz_balancer_create")
        self._h = h
        self._cb = None
        if agree is not None:
            def _cb(_ctx, bucket, n, ids, means):
                try:
                    new = agree(bucket, [ids[i] for i in range(n)], [means[i] for i in range(n)])
                    for i in range(n):
                        means[i] = float(new[i])
                    return 0
                except Exception:  # pragma: no cover - surfaced as NZ_ERR_SYSTEM by the library
                    return 1
            self._cb = _lib.AGREE_FN(_cb)
            check(lib().nz_balancer_set_agreement(self._h, self._cb, None), "nz_balancer_set_agreement")

    def close(self) -> None:
        if self._h:
            lib().nz_balancer_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def allocate(self, nbytes: int) -> dict:
        buf = ctypes.create_string_buffer(1 << 16)
        check(lib().nz_balancer_allocate(self._h, nbytes, buf, len(buf)), "nz_balancer_allocate")
        return json.loads(buf.value.decode())

    def record(self, latencies: dict) -> bool:
        ids = sorted(latencies)
        arr_i = (ctypes.c_int * max(len(ids), 1))(*ids)
        arr_d = (ctypes.c_double * max(len(ids), 1))(*[latencies[i] for i in ids])
        fl = ctypes.c_int(0)
        check(lib().nz_balancer_record(self._h, len(ids), arr_i, arr_d, byref(fl)), "nz_balancer_record")
        return bool(fl.value)

    def table(self) -> dict:
        buf = ctypes.create_string_buffer(1 << 20)
        check(lib().nz_balancer_table_json(self._h, buf, len(buf)), "nz_balancer_table_json")
        return json.loads(buf.value.decode())
