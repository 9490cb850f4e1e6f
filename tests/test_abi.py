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
                 "nz_planner_run_trace", "nz_core_ring_volume", "nz_last_error"):
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
    assert l.nz_abi_version() == 2 and l.nz_has_cuda_kernels() == 1


def test_errors_map_to_codes_without_gpu():
    from paper_2405_17870_b200 import Comm
    from paper_2405_17870_b200._lib import NezhaError

    with pytest.raises(NezhaError):
        Comm(0, 9, 0, "too-many-ranks")  # world > 8 is a precondition violation


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
