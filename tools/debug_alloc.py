"""Allocation probe: symmetric buffers of growing size with/without multicast."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_17870_b200 import Comm, SymmetricBuffer
comm = Comm.from_env(session=os.environ["NZ_SESSION"])
bufs = []
for mb in [1, 64, 256, 1024, 1024, 64, 2048]:
    try:
        bufs.append(SymmetricBuffer(comm, mb << 20))
        print(comm.rank, "ok", mb, file=sys.stderr)
    except Exception as e:
        print(comm.rank, "FAIL", mb, e, file=sys.stderr)
        break
print(json.dumps({"rank": comm.rank, "n": len(bufs), "mc": comm.multicast}))
