"""Spawns one worker process per rank (the torchrun layout, without torchrun)."""
from __future__ import annotations

import json
import os
import subprocess
import sys
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def spawn(world: int, script: str, args: list[str] | None = None, timeout: float = 300.0,
          extra_env: dict | None = None) -> list[dict]:
    """Runs `script` as `world` ranks; returns each rank's last JSON stdout line.

    Raises AssertionError with the ranks' output when any rank fails.
    """
    session = uuid.uuid4().hex[:12]
    procs = []
    for r in range(world):
        env = dict(os.environ)
        env.update({"RANK": str(r), "WORLD_SIZE": str(world), "LOCAL_RANK": str(r), "NZ_SESSION": session,
                    "MASTER_ADDR": "127.0.0.1", "PYTHONPATH": ROOT + os.pathsep + env.get("PYTHONPATH", "")})
        if extra_env:
            env.update(extra_env)
        procs.append(subprocess.Popen([sys.executable, script] + (args or []), cwd=ROOT, env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    import time

    outs = []
    failed = False
    deadline = time.monotonic() + timeout  # one deadline for the whole job
    for p in procs:
        try:
            o, e = p.communicate(timeout=max(1.0, deadline - time.monotonic()))
        except subprocess.TimeoutExpired:
            p.kill()
            o, e = p.communicate()
            failed = True
        outs.append((p.returncode, o, e))
        failed |= p.returncode != 0
    if failed:
        msg = "\n".join(f"--- rank {i} rc={rc}\n{o[-4000:]}\n{e[-4000:]}" for i, (rc, o, e) in enumerate(outs))
        raise AssertionError(f"worker failure:\n{msg}")
    res = []
    for rc, o, e in outs:
        lines = [l for l in o.splitlines() if l.startswith("{")]
        res.append(json.loads(lines[-1]) if lines else {})
    return res
