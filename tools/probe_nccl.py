"""Quick torch/NCCL allreduce busbw probe (baseline context only)."""
import os, torch, torch.distributed as dist, json
dist.init_process_group("nccl")
r = dist.get_rank(); w = dist.get_world_size()
torch.cuda.set_device(r)
res = []
for sz in [8192, 1<<20, 64<<20, 256<<20, 1<<30]:
    x = torch.ones(sz//4, device="cuda")
    for _ in range(5): dist.all_reduce(x)
    torch.cuda.synchronize()
    it = 50 if sz < (64<<20) else 10
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    dist.barrier(); s.record()
    for _ in range(it): dist.all_reduce(x)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e)/it/1e3
    res.append({"bytes": sz, "us": t*1e6, "busbw": 2*(w-1)/w*sz/t/1e9})
if r == 0: print("NCCL", json.dumps(res))
dist.destroy_process_group()
