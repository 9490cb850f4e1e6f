"""Debug the DDP hook: direct hook calls on known tensors, then DDP grads vs NCCL."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2405_17870_b200.ddp import NezhaHookState, nezha_allreduce_hook
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29655")
torch.cuda.set_device(rank)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
state = NezhaHookState.create(capacity=8 << 20, calibrate_max_bytes=1 << 22, calibrate_iters=4)
class B:
    def __init__(self, t): self.t = t
    def buffer(self): return self.t
res = {}
for n in [1000, 65536, 262144, 1 << 20, 3 << 20]:
    x = torch.arange(n, device="cuda", dtype=torch.float32) * (rank + 1)
    y = nezha_allreduce_hook(state, B(x.clone())).wait()
    torch.cuda.synchronize()
    want = torch.arange(n, device="cuda", dtype=torch.float32) * sum(range(1, world + 1)) / world
    res[n] = float((y - want).abs().max())
# grads from one DDP backward, hook vs nccl
def grads(hook):
    torch.manual_seed(0)
    m = torch.nn.Sequential(torch.nn.Linear(256, 1024), torch.nn.ReLU(), torch.nn.Linear(1024, 64)).cuda()
    d = torch.nn.parallel.DistributedDataParallel(m, device_ids=[rank], bucket_cap_mb=1)
    if hook: d.register_comm_hook(state, nezha_allreduce_hook)
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    x = torch.randn(32, 256, device="cuda", generator=g)
    d(x).square().mean().backward()
    torch.cuda.synchronize()
    return [p.grad.clone() for p in m.parameters()]
a, b = grads(False), grads(True)
res["grad_diff"] = [float((u - v).abs().max()) for u, v in zip(a, b)]
res["grad_mag"] = [float(u.abs().max()) for u in a]
print(json.dumps({"rank": rank, **{str(k): v for k, v in res.items()}}))
state.close(); dist.destroy_process_group()
