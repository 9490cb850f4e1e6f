"""CPU: the GPU tests' worker logic (virtual-rank threads, stall and failover
bookkeeping, checks) runs end to end against oracle-backed fakes of the
runtime objects (tools/dryrun_workers.py). It guards the test harness — the
code that will judge the device path — not the library itself."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_worker_logic_dry_run():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import dryrun_workers

    dryrun_workers.main()
