"""Compiles and runs the C++ doctest-style suites (CPU only):
  - tests/cpp/test_product.cpp: product C++ API known answers;
  - the reference's own suites (proj/tests/test_core.cpp, test_toml.cpp)
    against OUR include/nezha headers and sources (drop-in check),
    when /root/reference is present (built by oracle/Makefile)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2405_17870_b200", "csrc", "host")
SRCS = [os.path.join(HOST, f) for f in ("core.cpp", "collective.cpp", "balancer.cpp", "faults.cpp", "toml.cpp", "rails_config.cpp", "balancer_state.cpp", "json.cpp", "compute_pool.cpp", "calibration.cpp")]
REF_TESTS = "/root/reference/proj/tests"
FLAGS = ["-std=c++20", "-O1", "-pthread", "-ffp-contract=off", f"-I{ROOT}/include", f"-I{ROOT}/oracle/shim"]


def _build_run(tmp_path, name, sources):
    exe = str(tmp_path / name)
    cxx = shutil.which("g++")
    r = subprocess.run([cxx, *FLAGS, "-o", exe, *sources], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def test_product_cpp_api(tmp_path):
    out = _build_run(tmp_path, "test_product", [os.path.join(ROOT, "tests", "cpp", "test_product.cpp"), *SRCS])
    assert "0 failed" in out


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="/root/reference not mounted")
@pytest.mark.parametrize("suite,extra", [("test_core.cpp", []), ("test_toml.cpp", [])])
def test_reference_suites_against_our_headers(tmp_path, suite, extra):
    out = _build_run(tmp_path, suite[:-4], [os.path.join(REF_TESTS, suite), *SRCS, *extra])
    assert "0 failed" in out


def test_gpu_header_compiles_and_maps_errors(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2405_17870_b200")
    if not os.path.exists(os.path.join(lib_dir, "libnezha_b200.so")):
        pytest.skip("library not built")
    exe = str(tmp_path / "test_gpu_header")
    r = subprocess.run([shutil.which("g++"), *FLAGS, "-o", exe, os.path.join(ROOT, "tests", "cpp", "test_gpu_header.cpp"),
                        f"-L{lib_dir}", "-lnezha_b200", f"-Wl,-rpath,{lib_dir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


def test_product_host_code_under_tsan(tmp_path):
    """The product's host C++ (planner, faults, ComputePool incl. its blocking
    multi-threaded tests) under ThreadSanitizer."""
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    exe = str(tmp_path / "test_product_tsan")
    r = subprocess.run([cxx, *FLAGS, "-g", "-fsanitize=thread", "-o", exe,
                        os.path.join(ROOT, "tests", "cpp", "test_product.cpp"), *SRCS], capture_output=True, text=True)
    if r.returncode != 0 and "tsan" in r.stderr:
        pytest.skip("no ThreadSanitizer runtime")
    assert r.returncode == 0, r.stderr[-3000:]
    run = subprocess.run([exe], capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, TSAN_OPTIONS="halt_on_error=1"))
    assert run.returncode == 0 and "ThreadSanitizer" not in run.stdout + run.stderr, (run.stdout + run.stderr)[-3000:]
