"""TEST HARNESS ONLY: the few torch calls bench.py makes, over numpy and the
host harness's stand-in CUDA runtime (tests/fakecuda), so that bench.py's
own code paths — the loopback headline, its JSON line, e2e, the failover
section — can run on CPU (tests/test_host_harness.py). "cuda" tensors are
host arrays here, as device memory is host memory in the harness. Nothing
here is imported outside that test.
"""
from __future__ import annotations

import ctypes
import types

import numpy as np

from paper_2405_17870_b200._lib import lib


class _DType:
    def __init__(self, name, np_dtype):
        self.name, self.np = name, np_dtype


uint8 = _DType("uint8", np.uint8)
float32 = _DType("float32", np.float32)
bfloat16 = _DType("bfloat16", np.uint16)  # bf16 bits


class Tensor:
    def __init__(self, arr: np.ndarray, dtype: _DType):
        self.a, self.dtype = arr, dtype

    def data_ptr(self) -> int:
        return self.a.ctypes.data

    def __mul__(self, k):
        return Tensor(self.a * np.float32(k), self.dtype)

    def __sub__(self, k):
        return Tensor(self.a - np.float32(k), self.dtype)

    def to(self, dtype):
        if dtype is bfloat16:
            u = self.a.astype(np.float32).view(np.uint32)
            return Tensor(((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16), bfloat16)
        raise NotImplementedError(dtype.name)

    def view(self, dtype):
        return Tensor(self.a.view(dtype.np), dtype)

    def __getitem__(self, k):
        return Tensor(self.a[k], self.dtype)

    def cpu(self):
        return self

    def pin_memory(self):
        return self

    def copy_(self, other):
        np.copyto(self.a, other.a.view(self.a.dtype).reshape(self.a.shape))
        return self


class Generator:
    def __init__(self, device=None):
        self.rng = np.random.default_rng(0)

    def manual_seed(self, s):
        self.rng = np.random.default_rng(s)
        return self


def rand(n, device=None, generator=None):
    g = generator.rng if generator else np.random.default_rng()
    return Tensor(g.random(n, dtype=np.float32), float32)


def empty(n, dtype=float32):
    return Tensor(np.empty(n, dtype=dtype.np), dtype)


class _Stream:
    def __init__(self):
        s = ctypes.c_void_p()
        assert lib().cudaStreamCreateWithFlags(ctypes.byref(s), 1) == 0
        self.cuda_stream = s.value


class _Event:
    def __init__(self, enable_timing=False):
        e = ctypes.c_void_p()
        assert lib().cudaEventCreate(ctypes.byref(e)) == 0
        self.e = e

    def record(self, stream=None):
        assert lib().cudaEventRecord(self.e, ctypes.c_void_p(stream.cuda_stream if stream else None)) == 0

    def synchronize(self):
        assert lib().cudaEventSynchronize(self.e) == 0

    def elapsed_time(self, other) -> float:
        ms = ctypes.c_float()
        assert lib().cudaEventElapsedTime(ctypes.byref(ms), self.e, other.e) == 0
        return ms.value


cuda = types.SimpleNamespace(
    set_device=lambda d: None,
    init=lambda: None,
    is_available=lambda: True,
    device_count=lambda: 1,
    synchronize=lambda: lib().cudaDeviceSynchronize(),
    Stream=_Stream,
    Event=_Event,
)
