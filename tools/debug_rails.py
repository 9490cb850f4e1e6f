"""Runs each multi-GPU rail case in its own job to localise failures."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.mp_util import spawn
from tests.test_gpu_rails import MULTI
world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sel = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else range(len(MULTI))
for i in sel:
    try:
        res = spawn(world, "tests/workers/rail_worker.py", [json.dumps([MULTI[i]])], timeout=120,
                    extra_env={"CUDA_LAUNCH_BLOCKING": os.environ.get("CUDA_LAUNCH_BLOCKING", "0")})
        print(i, MULTI[i], "OK", json.dumps(res[0]["results"][0]))
    except AssertionError as e:
        print(i, MULTI[i], "FAIL", str(e)[-1500:])
    sys.stdout.flush()
