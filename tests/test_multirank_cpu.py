"""N > 1 host logic on CPU (gloo, world size 2): the multi-rank flush
agreement keeps every rank's planner decisions and table identical even when
each rank measures different latencies (DESIGN.md §4 "Multi-rank agreement")."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "workers", "planner_rank_worker.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_planner_agreement_gloo_world2():
    port, world = _free_port(), 2
    procs = [subprocess.Popen([sys.executable, WORKER], cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True, env=dict(os.environ, RANK=str(r), WORLD_SIZE=str(world),
                                                  MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PYTHONPATH=ROOT))
             for r in range(world)]
    outs = []
    try:
        for p in procs:
            o, e = p.communicate(timeout=240)
            assert p.returncode == 0, e[-3000:]
            outs.append(json.loads([l for l in o.splitlines() if l.startswith("{")][-1]))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for o in outs:
        a, l = o["results"]["agree"], o["results"]["local"]
        assert a["same_plans"] and a["same_table"], o
        assert a["measured_buckets"] >= 3 and a["hot_ops"] > 100, o
        # Sensitivity: without agreement the ranks' tables drift apart.
        assert not (l["same_plans"] and l["same_table"]), o
