"""python tools/run_spawn.py WORLD script.py [args...]: spawn ranks, print their outputs."""
import os, sys, subprocess, uuid
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
world = int(sys.argv[1]); session = uuid.uuid4().hex[:10]
ps = []
for r in range(world):
    env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), NZ_SESSION=session,
               PYTHONPATH=ROOT)
    ps.append(subprocess.Popen([sys.executable] + sys.argv[2:], env=env, cwd=ROOT))
rc = max(p.wait() for p in ps)
sys.exit(rc)
