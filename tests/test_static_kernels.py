"""Static properties of the shipped sm_100a kernels (CPU only, no GPU).

Reads the product library with cuobjdump, the way profiles/r01/sass_summary.txt
was made (tools/sass_summary.sh), and pins what the rail designs rely on
(DESIGN.md §3): the NVLS rail reduces inside the switch with vector
multimem.ld_reduce, the fold / copy paths move 128-bit vectors, the instances
the 2-, 4- and 8-GPU sweep launches keep everything in registers (no local
memory), and every virtual-rank (loopback) instance exists for N = 2..8.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2405_17870_b200", "libnezha_b200.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

pytestmark = pytest.mark.skipif(
    not (os.path.exists(LIB) and os.path.exists(CUOBJDUMP)),
    reason="needs the built library (make -C paper_2405_17870_b200/csrc) and cuobjdump",
)


def _run(*args):
    return subprocess.run([CUOBJDUMP, *args, LIB], check=True, capture_output=True, text=True).stdout


@pytest.fixture(scope="module")
def resources():
    """mangled kernel name -> {REG, STACK, LOCAL, ...}"""
    out, res, fn = _run("-res-usage"), {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
        elif fn and "REG:" in line:
            res[fn] = {k: int(v) for k, v in re.findall(r"(\w+):(\d+)", line)}
            fn = None
    assert res, "cuobjdump -res-usage listed no kernels"
    return res


@pytest.fixture(scope="module")
def sass():
    """mangled kernel name -> set of SASS opcodes"""
    out, ops, fn = _run("-sass"), {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            fn = m.group(1)
            ops[fn] = set()
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
        if fn and m:
            ops[fn].add(m.group(1))
    return ops


def _family(table, prefix):
    hits = {k: v for k, v in table.items() if k.startswith(prefix)}
    assert hits, f"no kernel named {prefix}* in {LIB}"
    return hits


# Itanium mangling of the templates in csrc/cuda/kernels.cuh.
DTYPES = {"F32": "3F32", "BF16": "4BF16", "I32": "3I32"}


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dt", sorted(DTYPES))
def test_sweep_instances_have_no_local_memory(resources, n, dt):
    """LL, NVLS and fold instances for N in {2, 4, 8}."""
    d = DTYPES[dt]
    prefixes = [
        f"_ZN2nz9ll_kernelINS_{d}ELi{n}EEEvNS_6LLArgsE",
        f"_ZN2nz11nvls_kernelINS_{d}ELi{n}E",
        f"_ZN2nz11fold_kernelINS_{d}ELi{n}E",
    ]
    for p in prefixes:
        for name, r in _family(resources, p).items():
            assert r.get("LOCAL", 0) == 0 and r.get("STACK", 0) == 0, f"{name}: {r}"


def test_copy_kernel_is_spill_free(resources):
    # The launch-status prologue keeps one 32-bit value across the copy loop
    # on the stack at the (512, 2) register cap: at most 8 bytes, never more.
    for name, r in _family(resources, "_ZN2nz11copy_kernel").items():
        assert r.get("LOCAL", 0) <= 8, f"{name}: {r}"


@pytest.mark.parametrize("n", range(2, 9))
def test_loopback_instances_exist(resources, n):
    """Virtual-rank grids (nz_comm_init_loopback) for every rail kernel with a cross-rank wait."""
    for dt, d in DTYPES.items():
        _family(resources, f"_ZN2nz14fold_kernel_vrINS_{d}ELi{n}ELi{n}E")
        _family(resources, f"_ZN2nz12ll_kernel_vrINS_{d}ELi{n}E")
    _family(resources, f"_ZN2nz17barrier_kernel_vrILi{n}E")


def test_pruned_variants_are_gone(resources):
    """Round-2 pruning: no multicast-push LL, no TMA or one-shot SM kernels ship."""
    for name in resources:
        assert "sm_tma_kernel" not in name and "oneshot_kernel" not in name, name
        assert not name.startswith("_ZN2nz9ll_kernel") or "ELb1E" not in name, name


@pytest.mark.parametrize(
    "dt,op",
    [("F32", "LDGMC.E.ADD.F32x4"), ("BF16", "LDGMC.E.HPADD.BF16x8"), ("I32", "LDGMC.E.ADD.32")],
)
def test_nvls_reduces_in_the_switch(sass, dt, op):
    for name, ops in _family(sass, f"_ZN2nz11nvls_kernelINS_{DTYPES[dt]}E").items():
        assert any(o.startswith(op) for o in ops), f"{name}: no {op}"
        assert any(o.startswith("STG.E.128") for o in ops), f"{name}: no 128-bit multimem.st"


@pytest.mark.parametrize("prefix", ["_ZN2nz11fold_kernel", "_ZN2nz11copy_kernel"])
def test_vector_paths_are_128_bit(sass, prefix):
    for name, ops in _family(sass, prefix).items():
        assert "LDG.E.NA.128" in ops or any(o.startswith("LDG.E.128") for o in ops), f"{name}: no 128-bit load"
        assert any(o.startswith("STG.E.128") for o in ops), f"{name}: no 128-bit store"
