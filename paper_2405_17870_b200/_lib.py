"""ctypes binding of libnezha_b200.so (the C ABI in include/nezha_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2405_17870_b200/csrc`). There is no fallback: if the library is
missing, importing the runtime raises, so a GPU run can never silently take a
non-CUDA path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_size_t, c_uint32, c_uint64, c_void_p

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnezha_b200.so")

NZ_OK = 0
NZ_ERR_INVALID = -1
NZ_ERR_CUDA = -2
NZ_ERR_SYSTEM = -3
NZ_ERR_UNSUPPORTED = -4
NZ_ERR_RAIL_DOWN = -5
NZ_ERR_UNRECOVERABLE = -6
NZ_ERR_TIMEOUT = -7
NZ_ERR_BUFFER = -8

F32, BF16, I32 = 0, 1, 2
DTYPES = {"f32": F32, "bf16": BF16, "i32": I32}
ELEM_SIZE = {F32: 4, BF16: 2, I32: 4}
NVLS, CE, SM = 0, 1, 2
RAIL_KINDS = {"nvls": NVLS, "ce": CE, "sm": SM}
ALGO_RING, ALGO_RING_CHUNKED = 0, 1


class NezhaError(RuntimeError):
    """Base of the errors mapped from ABI return codes (error.hpp:11-60)."""

    code = -100


class InvalidArgument(NezhaError, ValueError):
    code = NZ_ERR_INVALID


class CudaError(NezhaError):
    code = NZ_ERR_CUDA


class SystemFailure(NezhaError):
    code = NZ_ERR_SYSTEM


class Unsupported(NezhaError):
    code = NZ_ERR_UNSUPPORTED


class ChannelDownError(NezhaError):
    code = NZ_ERR_RAIL_DOWN


class UnrecoverableError(NezhaError):
    code = NZ_ERR_UNRECOVERABLE


class RendezvousTimeoutError(NezhaError):
    code = NZ_ERR_TIMEOUT


class BufferTooSmall(NezhaError):
    code = NZ_ERR_BUFFER


_BY_CODE = {c.code: c for c in (InvalidArgument, CudaError, SystemFailure, Unsupported, ChannelDownError,
                                UnrecoverableError, RendezvousTimeoutError, BufferTooSmall)}


class FaultRecord(ctypes.Structure):
    _fields_ = [("valid", c_uint32), ("op_seq", c_uint32), ("chunk", c_uint64), ("t_fail_ns", c_uint64)]


class EngineConfig(ctypes.Structure):
    _fields_ = [
        ("num_rails", c_int),
        ("kinds", c_int * 3),
        ("sm_budget", c_int * 3),
        ("algorithm", c_int),
        ("tau", c_double),
        ("eta", c_double),
        ("convergence_eps", c_double),
        ("sync_overhead_us", c_double),
        ("window", c_int),
        ("max_iters", c_int),
        ("demote_after", c_int),
        ("rails_toml", c_char_p),
        ("calibrate_iters", c_int),
        ("calibrate_max_bytes", c_uint64),
        ("timer_lag", c_int),
        ("compute_pool", c_int),
        ("pool_tokens", c_int),
        ("tune_budgets", c_int),
        ("graph_safe", c_int),
        ("monitor", c_int),
        ("detect_us", c_double),
        ("heartbeat_us", c_double),
        ("readmit_hold_us", c_double),
    ]


class FailoverReport(ctypes.Structure):
    _fields_ = [
        ("op_seq", c_uint32),
        ("failed_rail", c_int),
        ("target_rail", c_int),
        ("orphan_offset", c_uint64),
        ("orphan_length", c_uint64),
        ("detect_us", c_double),
        ("resume_us", c_double),
        ("done_us", c_double),
        ("host_detect_us", c_double),
        ("device_detect_us", c_double),
        ("resume_after_detect_us", c_double),
        ("orphan_chunk", c_uint64),
        ("stalled_here", c_int),
    ]


class RailStatus(ctypes.Structure):
    """nz_rail_status_t: launch status a rail's kernels publish."""

    _fields_ = [
        ("ok_tag", c_uint32),
        ("prog_tag", c_uint32),
        ("prog_chunk", c_uint64),
        ("start_tag", c_uint32),
        ("fail_tag", c_uint32),
        ("t_start_ns", c_uint64),
        ("t_fail_ns", c_uint64),
        ("det_tag", c_uint32),
        ("abort", c_uint32),
        ("t_det_ns", c_uint64),
        ("run_tag", c_uint32),
        ("reserved", c_uint32),
        ("t_run_ns", c_uint64),
    ]


AGREE_FN = ctypes.CFUNCTYPE(c_int, c_void_p, c_int, c_int, POINTER(c_int), POINTER(c_double))

_SIGS = {
    "nz_last_error": (c_char_p, []),
    "nz_abi_version": (c_int, []),
    "nz_abi_sizeof": (c_int, [c_char_p]),
    "nz_has_cuda_kernels": (c_int, []),
    "nz_comm_init": (c_int, [c_int, c_int, c_int, c_char_p, c_int, POINTER(c_void_p)]),
    "nz_comm_init_loopback": (c_int, [c_int, c_int, c_int, c_char_p, c_int, POINTER(c_void_p)]),
    "nz_comm_is_loopback": (c_int, [c_void_p]),
    "nz_comm_abort": (c_int, [c_void_p]),
    "nz_comm_destroy": (c_int, [c_void_p]),
    "nz_comm_rank": (c_int, [c_void_p]),
    "nz_comm_world": (c_int, [c_void_p]),
    "nz_comm_device": (c_int, [c_void_p]),
    "nz_comm_sm_count": (c_int, [c_void_p]),
    "nz_comm_multicast_supported": (c_int, [c_void_p]),
    "nz_comm_barrier": (c_int, [c_void_p]),
    "nz_comm_allgather": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "nz_buffer_alloc": (c_int, [c_void_p, c_size_t, POINTER(c_void_p)]),
    "nz_buffer_free": (c_int, [c_void_p]),
    "nz_buffer_ptr": (c_void_p, [c_void_p]),
    "nz_buffer_peer_ptr": (c_void_p, [c_void_p, c_int]),
    "nz_buffer_mc_ptr": (c_void_p, [c_void_p]),
    "nz_buffer_size": (c_size_t, [c_void_p]),
    "nz_buffer_write": (c_int, [c_void_p, c_uint64, c_void_p, c_uint64, c_void_p]),
    "nz_buffer_read": (c_int, [c_void_p, c_uint64, c_void_p, c_uint64, c_void_p]),
    "nz_buffer_fill_zero": (c_int, [c_void_p, c_void_p]),
    "nz_rail_create": (c_int, [c_void_p, c_int, c_int, c_int, POINTER(c_void_p)]),
    "nz_rail_create_ex": (c_int, [c_void_p, c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    "nz_rail_destroy": (c_int, [c_void_p]),
    "nz_rail_kind": (c_int, [c_void_p]),
    "nz_rail_stream": (c_void_p, [c_void_p]),
    "nz_rail_synchronize": (c_int, [c_void_p]),
    "nz_rail_allreduce": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64, c_uint64, c_uint64, c_uint64, c_uint64,
                                  c_int, c_uint32, c_int64, c_void_p]),
    "nz_rail_poll_fault": (c_int, [c_void_p, POINTER(FaultRecord), c_int]),
    "nz_rail_watchdog": (c_int, [c_void_p]),
    "nz_rail_inject_failure": (c_int, [c_void_p, c_uint64]),
    "nz_rail_progress": (c_int, [c_void_p, POINTER(c_uint64)]),
    "nz_rail_abort": (c_int, [c_void_p]),
    "nz_rail_status": (c_int, [c_void_p, c_void_p]),
    "nz_rail_loop_timing": (c_int, [c_void_p, c_int]),
    "nz_rail_loop_time": (c_int, [c_void_p, POINTER(c_uint64), POINTER(c_double)]),
    "nz_engine_rail": (c_void_p, [c_void_p, c_int]),
    "nz_rail_inject_stall": (c_int, [c_void_p, c_uint64]),
    "nz_rail_revive": (c_int, [c_void_p]),
    "nz_rail_set_detect_us": (c_int, [c_void_p, c_double]),
    "nz_event_elapsed_us": (c_int, [c_void_p, c_void_p, POINTER(c_double)]),
    "nz_engine_config_default": (None, [POINTER(EngineConfig)]),
    "nz_engine_create": (c_int, [c_void_p, POINTER(EngineConfig), POINTER(c_void_p)]),
    "nz_engine_destroy": (c_int, [c_void_p]),
    "nz_engine_allreduce": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64, c_int, c_void_p]),
    "nz_engine_allreduce_host": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64, c_int]),
    "nz_engine_allreduce_device": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64, c_int, c_void_p]),
    "nz_engine_inject_failure": (c_int, [c_void_p, c_uint32, c_int, c_uint64]),
    "nz_engine_readmit": (c_int, [c_void_p, c_int]),
    "nz_engine_synchronize": (c_int, [c_void_p]),
    "nz_engine_op_seq": (c_uint32, [c_void_p]),
    "nz_engine_last_failover": (c_int, [c_void_p, POINTER(FailoverReport)]),
    "nz_engine_failover_count": (c_int, [c_void_p]),
    "nz_engine_failover_get": (c_int, [c_void_p, c_int, POINTER(FailoverReport)]),
    "nz_engine_state_json": (c_int, [c_void_p, c_char_p, c_size_t]),
    "nz_engine_plan_json": (c_int, [c_void_p, c_uint64, c_char_p, c_size_t]),
    "nz_engine_last_plan_json": (c_int, [c_void_p, c_char_p, c_size_t]),
    "nz_engine_rail_stats": (c_int, [c_void_p, c_int, POINTER(c_uint64), POINTER(c_double), POINTER(c_uint64)]),
    "nz_engine_stats_reset": (c_int, [c_void_p]),
    "nz_engine_save_state": (c_int, [c_void_p, c_char_p, c_size_t]),
    "nz_engine_load_state": (c_int, [c_void_p, c_char_p]),
    "nz_kernel_launch_count": (c_uint64, []),
    "nz_planner_run_trace": (c_int, [c_char_p, c_char_p, c_size_t]),
    "nz_emulate_fold": (c_int, [c_int, c_int, c_int, POINTER(c_void_p), POINTER(c_void_p), c_int, c_uint64, c_uint64,
                                c_uint64, c_uint64, c_uint64, c_int, c_void_p]),
    "nz_balancer_create": (c_int, [c_char_p, c_double, c_double, c_double, c_int, c_int, POINTER(c_void_p)]),
    "nz_balancer_destroy": (c_int, [c_void_p]),
    "nz_balancer_set_agreement": (c_int, [c_void_p, AGREE_FN, c_void_p]),
    "nz_balancer_allocate": (c_int, [c_void_p, c_uint64, c_char_p, c_size_t]),
    "nz_balancer_record": (c_int, [c_void_p, c_int, POINTER(c_int), POINTER(c_double), POINTER(c_int)]),
    "nz_balancer_table_json": (c_int, [c_void_p, c_char_p, c_size_t]),
    "nz_pool_create": (c_int, [c_int, POINTER(c_void_p)]),
    "nz_pool_destroy": (c_int, [c_void_p]),
    "nz_pool_declare": (c_int, [c_void_p, c_int, c_int, c_int, c_int]),
    "nz_pool_acquire": (c_int, [c_void_p, c_int, c_int, c_int, POINTER(c_int)]),
    "nz_pool_release": (c_int, [c_void_p, c_int, c_int]),
    "nz_pool_outstanding": (c_int, [c_void_p]),
    "nz_pool_waiting": (c_int, [c_void_p]),
    "nz_pool_plan": (c_int, [c_int, c_int, c_int, POINTER(c_int), POINTER(c_int), POINTER(c_int), POINTER(c_uint32)]),
    "nz_core_ring_volume": (c_uint64, [c_int, c_uint64]),
    "nz_core_bucket_of": (c_int, [c_uint64]),
    "nz_core_default_chunk_bytes": (c_uint64, [c_uint64, c_int, c_int]),
    "nz_core_calibrate": (c_int, [POINTER(c_uint64), POINTER(c_double), c_int, POINTER(c_double), POINTER(c_double),
                                  POINTER(c_int), POINTER(c_double)]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded product library; raises if it was never built."""
    global _lib
    if _lib is None:
        path = LIB_PATH
        harness = os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB")
        if harness:
            # CPU test suite only (tests/test_host_harness.py): the product's
            # host code linked against tests/fakecuda's host stand-in for the
            # CUDA runtime, to exercise host logic without a GPU. It is never
            # the product: only that test sets this, only for its own
            # subprocesses, and only this one file name is accepted.
            if os.path.basename(harness) != "libnezha_b200_hostharness.so":
                raise ImportError(f"NEZHA_TEST_HOST_HARNESS_LIB must name the test harness build, not {harness}")
            path = harness
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        l = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name, None)
            if fn is None:
                continue  # exports are verified separately by tests/test_abi.py
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(rc: int, what: str = "") -> int:
    if rc >= 0:
        return rc
    msg = (lib().nz_last_error() or b"").decode(errors="replace")
    cls = _BY_CODE.get(rc, NezhaError)
    raise cls(f"{what}: {msg}" if what else msg)
