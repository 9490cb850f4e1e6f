import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# Bounded device waits for the whole test session: a rail kernel whose peer
# never arrives gives up after 5 s instead of the production 20 s (read once
# by the library, so it is set before anything loads it).
os.environ.setdefault("NEZHA_WATCHDOG_MS", "5000")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs in one box")


def gpu_count() -> int:
    # The CPU host harness (tests/test_host_harness.py) can
    # stand in for an N-GPU box: one process per "GPU", multicast emulated.
    if os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB") and os.environ.get("NEZHA_TEST_HARNESS_GPUS"):
        return int(os.environ["NEZHA_TEST_HARNESS_GPUS"])
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.fixture(scope="session")
def n_gpus() -> int:
    return gpu_count()
