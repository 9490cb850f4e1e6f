"""Rank 1 never joins rank 0's rail op: rank 0's kernel must give up after
NEZHA_WATCHDOG_MS, flag the watchdog and exit (no GPU hang); the engine-level
synchronize then reports the rail down on every rank."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2405_17870_b200 import Comm, Rail, SymmetricBuffer
from paper_2405_17870_b200._lib import F32, RAIL_KINDS
comm = Comm.from_env(session=os.environ["NZ_SESSION"])
kind = sys.argv[1]
b1, b2 = SymmetricBuffer(comm, 1 << 22), SymmetricBuffer(comm, 1 << 22)
r = Rail(comm, RAIL_KINDS[kind], 0)
t0 = time.time()
if comm.rank == 0:
    r.allreduce(b1, b2, 0, 1 << 22, 1 << 20, F32)  # two-shot path (> LL ceiling at N=2 for NVLS)
    r.synchronize()
wd = r.watchdog()
dt = time.time() - t0
comm.barrier()
r.close(); b1.free(); b2.free(); comm.close()
print(json.dumps({"rank": comm.rank, "watchdog": wd, "seconds": round(dt, 3)}))
