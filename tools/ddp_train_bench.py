"""Real DDP training steps: ResNet-50 and BERT-large with
random init and synthetic data, NCCL's default allreduce vs the Nezha engine
comm hook, ms per iteration (CUDA events on the default stream, max over
ranks). Launch one process per GPU:
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
      tools/ddp_train_bench.py [resnet50,bert] [iters]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_17870_b200.ddp import NezhaHookState, nezha_allreduce_hook  # noqa: E402


def make(name):
    if name == "resnet50":
        import torchvision
        m = torchvision.models.resnet50(weights=None)
        x = torch.randn(64, 3, 224, 224)
        y = torch.randint(0, 1000, (64,))
        return m, lambda mm: torch.nn.functional.cross_entropy(mm(x.cuda(non_blocking=True)), y.cuda()), x, y
    from transformers import BertConfig, BertForPreTraining
    cfg = BertConfig(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16, intermediate_size=4096)
    m = BertForPreTraining(cfg)
    ids = torch.randint(0, cfg.vocab_size, (8, 128))
    lab = ids.clone()
    nsp = torch.zeros(8, dtype=torch.long)

    def loss(mm):
        out = mm(input_ids=ids.cuda(), labels=lab.cuda(), next_sentence_label=nsp.cuda())
        return out.loss
    return m, loss, ids, lab


def run(name, hook_state, iters, rank):
    torch.manual_seed(0)
    model, loss_fn, _, _ = make(name)
    model = model.cuda()
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[rank])
    if hook_state is not None:
        ddp.register_comm_hook(hook_state, nezha_allreduce_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=1e-3)
    for _ in range(5):
        opt.zero_grad(set_to_none=True)
        loss_fn(ddp).backward()
        opt.step()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        opt.zero_grad(set_to_none=True)
        loss_fn(ddp).backward()
        opt.step()
    b.record()
    b.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / iters], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def main():
    rank = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["resnet50", "bert"]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    state = NezhaHookState.create(capacity=64 << 20, calibrate_max_bytes=1 << 26)
    res = {}
    for n in names:
        res[n] = {"nccl_ms": round(run(n, None, iters, rank), 3), "nezha_ms": round(run(n, state, iters, rank), 3)}
    state.close()
    if dist.get_rank() == 0:
        print(json.dumps({"world": dist.get_world_size(), "iters": iters, "ms_per_iter": res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
