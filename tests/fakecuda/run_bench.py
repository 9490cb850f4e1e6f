"""TEST HARNESS ONLY: runs bench.py's loopback path on CPU — torch replaced by
tests/fakecuda/torch_stub.py, the product library by the host harness (set
NEZHA_TEST_HOST_HARNESS_LIB). Checks bench.py's own code, not performance.
    python tests/fakecuda/run_bench.py [bench.py args]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
assert os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB"), "host harness only"

import torch_stub  # noqa: E402

sys.modules["torch"] = torch_stub
import bench  # noqa: E402

sys.argv = ["bench.py"] + sys.argv[1:]
sys.exit(bench.main())
