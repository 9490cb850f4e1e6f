"""CPU oracle for the Nezha allreduce path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package, and only as the checker or
the timed CPU baseline. The product (paper_2405_17870_b200/) never imports it.

  nezha_oracle.c  -> build/liboracle.so   ring-order fold (P1/P2),
                                           synthetic inputs
  ring_inmem.cpp  -> _ref/libnezha_inmem_oracle.so  the literal SPEC ring on
                                           the reference's InMemoryFabric
  planner.py      -> balancer / faults decisions
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_int, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")
INMEM_LIB = os.path.join(HERE, "_ref", "libnezha_inmem_oracle.so")

F32, BF16, I32 = 0, 1, 2
NP_DTYPE = {F32: np.float32, BF16: np.uint16, I32: np.int32}
SEED_BASE = 0x4E5A0000

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing: run `make -C oracle`")
        l = ctypes.CDLL(LIB)
        l.nzo_reduce_range.argtypes = [c_int, c_int, ctypes.POINTER(c_void_p), c_void_p, c_uint64, c_uint64, c_uint64,
                                       c_uint64, c_uint64]
        l.nzo_reduce_range.restype = c_int
        l.nzo_fill_input.argtypes = [c_int, c_int, c_uint64, c_void_p, c_uint64]
        l.nzo_fill_input.restype = c_int
        l.nzo_default_chunk_bytes.argtypes = [c_uint64, c_int, c_int]
        l.nzo_default_chunk_bytes.restype = c_uint64
        l.nzo_f32_to_bf16.argtypes = [c_void_p, c_void_p, c_uint64]
        l.nzo_f32_to_bf16.restype = None
        _lib = l
    return _lib


def default_chunk_bytes(seg_len: int, world: int, chunked: bool = True) -> int:
    return int(lib().nzo_default_chunk_bytes(seg_len, world, 1 if chunked else 0))


def synthetic_input(dtype: int, rank: int, nbytes: int, seed_base: int = SEED_BASE) -> np.ndarray:
    """Rank `rank`'s synthetic payload: mt19937_64(seed_base + rank)."""
    es = 2 if dtype == BF16 else 4
    n = nbytes // es
    a = np.empty(n, dtype=NP_DTYPE[dtype])
    if lib().nzo_fill_input(dtype, rank, seed_base, a.ctypes.data, n) != 0:
        raise ValueError("bad dtype")
    return a


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty(a.shape, dtype=np.uint16)
    lib().nzo_f32_to_bf16(a.ctypes.data, out.ctypes.data, a.size)
    return out


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def reduce_range(inputs: list[np.ndarray], dtype: int, seg_off: int, seg_len: int, chunk_bytes: int, lo: int, hi: int,
                 out: np.ndarray | None = None) -> np.ndarray:
    """Ring-order allreduce of bytes [lo, hi) with geometry (seg_off, seg_len, chunk_bytes).

    Elements outside [lo, hi) are left as they were in `out` (zeros if new).
    """
    world = len(inputs)
    ins = [np.ascontiguousarray(x) for x in inputs]
    if out is None:
        out = np.zeros_like(ins[0])
    arr = (c_void_p * world)(*[x.ctypes.data for x in ins])
    rc = lib().nzo_reduce_range(world, dtype, arr, out.ctypes.data, seg_off, seg_len, chunk_bytes, lo, hi)
    if rc != 0:
        raise ValueError("oracle: bad geometry")
    return out


_inmem = None


def inmem_available() -> bool:
    return os.path.exists(INMEM_LIB)


def inmem_lib():
    global _inmem
    if _inmem is None:
        if not os.path.exists(INMEM_LIB):
            raise ImportError(f"{INMEM_LIB} missing: run `make -C oracle ref` where /root/reference exists")
        l = ctypes.CDLL(INMEM_LIB)
        P = ctypes.POINTER
        l.nzi_multirail_allreduce.argtypes = [c_int, c_int, c_int, P(c_void_p), P(c_void_p), c_uint64, c_int,
                                              P(c_int), P(c_uint64), P(c_uint64), c_int, c_int, c_uint64,
                                              ctypes.c_uint32, P(ctypes.c_double), P(c_uint64)]
        l.nzi_multirail_allreduce.restype = c_int
        _inmem = l
    return _inmem


def inmem_allreduce(inputs: list[np.ndarray], dtype: int, segments: list[tuple[int, int, int]], nrails: int,
                    chunked: bool = True, fail_rail: int = -1, fail_chunk: int = 0, op_seq: int = 1,
                    outputs: list[np.ndarray] | None = None):
    """The literal SPEC ring on the reference InMemoryFabric (oracle/ring_inmem.cpp).

    segments: (rail, offset, length). Returns (outputs per rank, elapsed_us, rank0 data bytes).
    """
    world = len(inputs)
    ins = [np.ascontiguousarray(x) for x in inputs]
    outs = outputs if outputs is not None else [np.zeros_like(ins[0]) for _ in range(world)]
    n = len(segments)
    rails = (c_int * n)(*[s[0] for s in segments])
    offs = (c_uint64 * n)(*[s[1] for s in segments])
    lens = (c_uint64 * n)(*[s[2] for s in segments])
    el = ctypes.c_double()
    sent = c_uint64()
    rc = inmem_lib().nzi_multirail_allreduce(world, dtype, 1 if chunked else 0,
                                             (c_void_p * world)(*[x.ctypes.data for x in ins]),
                                             (c_void_p * world)(*[x.ctypes.data for x in outs]),
                                             ins[0].nbytes, n, rails, offs, lens, nrails, fail_rail, fail_chunk,
                                             op_seq, ctypes.byref(el), ctypes.byref(sent))
    if rc != 0:
        raise RuntimeError(f"inmem oracle failed rc={rc}")
    return outs, el.value, sent.value


def reduce_segments(inputs: list[np.ndarray], dtype: int, segments: list[tuple[int, int, int]]) -> np.ndarray:
    """Full allreduce result for a list of (offset, length, chunk_bytes) segments covering the buffer."""
    out = np.zeros_like(inputs[0])
    for off, length, chunk in segments:
        if length:
            reduce_range(inputs, dtype, off, length, chunk, off, off + length, out)
    return out
