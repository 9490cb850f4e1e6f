"""Forced-hot probe: the engine with two rails and a TOML that makes the hot
split win in the model, to measure real concurrent throughput vs each rail."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17870_b200 import Comm, Engine, SymmetricBuffer
from paper_2405_17870_b200._lib import F32
comm = Comm.from_env(session=os.environ["NZ_SESSION"])
torch.cuda.set_device(comm.device)
kinds = sys.argv[1].split(",")
alpha0 = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
pool_mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # ComputePool: 0 off, 1 block, 2 shrink
toml = ""
for k in kinds:
    toml += f'[[rail]]\nprotocol = "{k}"\nt_setup_us = 10.0\nbandwidth_bps = 5.0e11\n'
res = {}
for S in [64 << 20, 256 << 20, 1 << 30]:
    eng = Engine(comm, kinds=kinds, rails_toml=toml, sync_overhead_us=0.0, window=10, eta=0.3, demote_after=0,
                 compute_pool=pool_mode)
    bi, bo = SymmetricBuffer(comm, S), SymmetricBuffer(comm, S)
    st = torch.cuda.Stream()
    for _ in range(300):
        eng.allreduce(bi, bo, S, F32, st)
    eng.synchronize()
    comm.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20):
        eng.allreduce(bi, bo, S, F32, st)
    b.record(st)
    b.synchronize()
    eng.synchronize()
    t = a.elapsed_time(b) / 1e3 / 20
    w = comm.world
    res[S] = {"busbw": round(2 * (w - 1) / w * S / t / 1e9, 1), "plan": eng.last_plans()[0]["segs"]}
    eng.close(); bi.free(); bo.free()
print(json.dumps({"rank": comm.rank, "kinds": kinds, "compute_pool": pool_mode, "res": {str(k): v for k, v in res.items()}}))
comm.close()
