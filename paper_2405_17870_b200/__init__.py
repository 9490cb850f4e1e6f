"""B200-native multi-rail allreduce (Nezha, arxiv 2405.17870).

The product is libnezha_b200.so (C ABI: include/nezha_b200.h; C++ API:
include/nezha/*.hpp). This package is the Python mirror of that ABI used by
the tests and bench.py.
"""
from ._lib import BF16, CE, F32, I32, NVLS, SM, NezhaError, lib  # noqa: F401
from .runtime import Comm, ComputePool, Engine, Rail, SymmetricBuffer, default_engine_config, emulate_fold, run_trace  # noqa: F401
from .loopback import RankFailure, run_ranks  # noqa: F401

__all__ = ["Comm", "ComputePool", "Engine", "Rail", "SymmetricBuffer", "default_engine_config", "emulate_fold", "run_trace",
           "run_ranks", "RankFailure",
           "F32", "BF16", "I32", "NVLS", "CE", "SM", "NezhaError", "lib"]
