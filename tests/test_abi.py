"""The drop-in boundary: libnezha_b200.so loads without a GPU and exports every
function include/nezha_b200.h declares; the core ABI answers the reference's
known answers (proj/tests/test_core.cpp:12-19, :111-118). CPU only."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nezha_b200.h")
LIB = os.path.join(ROOT, "paper_2405_17870_b200", "libnezha_b200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nz_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    for must in ("nz_comm_init", "nz_buffer_alloc", "nz_rail_create", "nz_rail_allreduce", "nz_rail_poll_fault",
                 "nz_engine_create", "nz_engine_allreduce", "nz_engine_allreduce_host", "nz_engine_inject_failure",
                 "nz_planner_run_trace", "nz_core_ring_volume", "nz_last_error", "nz_comm_init_loopback",
                 "nz_rail_inject_stall", "nz_rail_status", "nz_rail_revive", "nz_engine_failover_get"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: __graft_entry__.build()"
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_core_known_answers_through_the_abi():
    from paper_2405_17870_b200 import lib

    l = lib()
    assert l.nz_core_ring_volume(2, 1024) == 1024
    assert l.nz_core_ring_volume(4, 4 << 20) == 6 << 20
    assert l.nz_core_ring_volume(16, 0) == 0
    assert l.nz_core_bucket_of(4096) == 12 and l.nz_core_bucket_of(8191) == 12 and l.nz_core_bucket_of(8192) == 13
    assert l.nz_core_default_chunk_bytes(64 << 20, 8, 1) == 4 << 20
    assert l.nz_abi_version() == 3 and l.nz_has_cuda_kernels() == 1


def test_errors_map_to_codes_without_gpu():
    from paper_2405_17870_b200 import Comm, lib
    from paper_2405_17870_b200._lib import NezhaError

    with pytest.raises(NezhaError):
        Comm(0, 9, 0, "too-many-ranks")  # world > 8 is a precondition violation
    l = lib()
    assert l.nz_comm_abort(None) == -1  # NZ_ERR_INVALID, no CUDA call made


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (not just PTX) for the rail kernels."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([tool, "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([tool, "-sass", LIB], capture_output=True, text=True).stdout
    assert "LDGMC" in sass or "multimem" in sass.lower()  # NVLS ld_reduce made it to SASS


def test_ctypes_struct_layouts_match_the_header():
    """The Python mirror lays the ABI structs out exactly as the library does."""
    import ctypes

    from paper_2405_17870_b200 import _lib, lib

    l = lib()
    for name, cls in (("engine_config", _lib.EngineConfig), ("failover_report", _lib.FailoverReport),
                      ("rail_status", _lib.RailStatus), ("fault_record", _lib.FaultRecord)):
        assert l.nz_abi_sizeof(name.encode()) == ctypes.sizeof(cls), name
    assert l.nz_abi_sizeof(b"nope") < 0


def test_engine_config_defaults():
    """Round-2 defaults: failure monitor on, Timer lag 16, SPEC heartbeats
    (50 ms) and readmit hold (1 s), profiles measured at startup."""
    from paper_2405_17870_b200 import default_engine_config

    c = default_engine_config()
    assert (c.num_rails, list(c.kinds)) == (3, [0, 1, 2])
    assert c.monitor == 1 and c.timer_lag == 16 and c.heartbeat_us == 50000 and c.readmit_hold_us == 1e6
    assert c.detect_us == 0 and c.sync_overhead_us < 0 and c.window == 100 and c.tau == 5.0
    assert c.graph_safe == 0 and c.compute_pool == 0 and c.tune_budgets == 0
