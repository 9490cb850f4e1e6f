"""One rank of the DDP comm-hook check: the same tiny model trained 3 steps
with NCCL's allreduce and with the Nezha engine hook must end with the same
parameters (fp32, different summation order: rtol 1e-5)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_17870_b200.ddp import NezhaHookState, nezha_allreduce_hook  # noqa: E402


def train(use_hook, rank, state=None):
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(256, 1024), torch.nn.ReLU(), torch.nn.Linear(1024, 64)).cuda()
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[rank], bucket_cap_mb=1)
    if use_hook:
        ddp.register_comm_hook(state, nezha_allreduce_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.1)
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    for _ in range(3):
        x = torch.randn(32, 256, device="cuda", generator=g)
        loss = ddp(x).square().mean()
        opt.zero_grad()
        loss.backward()
        opt.step()
    torch.cuda.synchronize()
    return [p.detach().clone() for p in model.parameters()]


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29600 + int(os.environ["NZ_SESSION"][:4], 16) % 300))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    ref = train(False, rank)
    state = NezhaHookState.create(capacity=8 << 20, calibrate_max_bytes=1 << 22, calibrate_iters=4)
    got = train(True, rank, state)
    worst = max(float(((a - b).abs() / (b.abs() + 1e-6)).max()) for a, b in zip(got, ref))
    ok = all(torch.allclose(a, b, rtol=1e-5, atol=1e-6) for a, b in zip(got, ref))
    state.close()
    dist.destroy_process_group()
    print(json.dumps({"rank": rank, "ok": ok, "max_rel": worst}))


if __name__ == "__main__":
    main()
