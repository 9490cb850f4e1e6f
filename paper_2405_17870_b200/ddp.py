"""PyTorch DDP communication hook backed by the multi-rail engine.

The paper's end users are data-parallel trainers (Gloo apps, Horovod, vTrain;
PAPER.md:528-531). This hook lets `torch.nn.parallel.DistributedDataParallel`
reduce its gradient buckets through libnezha_b200.so instead of NCCL:

    state = NezhaHookState.create(process_group)      # one Engine per rank
    ddp_model.register_comm_hook(state, nezha_allreduce_hook)

Each bucket goes through nz_engine_allreduce_device: staged piecewise into
the engine's symmetric UnboundBuffer, all-reduced by the rails and copied
back with the copies pipelined against the NVLink work, then averaged — all
on the hook's own communication stream, which first waits for the stream that
produced the gradients. The returned CUDA-aware future carries an event on
that communication stream, so backward compute of the next buckets overlaps
the reduction (as with NCCL's stream) and DDP's consumers wait for it.
torch is only the caller here; the reduction is the C ABI.
"""
import os
from dataclasses import dataclass

import torch

from ._lib import BF16, F32, I32
from .runtime import Comm, Engine

# Gradient dtypes the hook averages. int32 is an engine dtype (sum with
# wraparound) but a mean of integers is not a gradient: it is refused up front,
# before anything is reduced.
_DTYPES = {torch.float32: F32, torch.bfloat16: BF16}
_ENGINE_ONLY = {torch.int32: I32}


@dataclass
class NezhaHookState:
    comm: Comm
    engine: Engine
    world: int
    stream: torch.cuda.Stream = None

    @classmethod
    def create(cls, process_group=None, capacity: int = 256 << 20, rails=("nvls", "ce", "sm"),
               **engine_overrides) -> "NezhaHookState":
        """`capacity` sizes the startup calibration (and so the first staging
        buffer) unless `calibrate_max_bytes` is given; larger buckets grow it."""
        import torch.distributed as dist

        rank = dist.get_rank(process_group)
        world = dist.get_world_size(process_group)
        # Same session string on every rank: agree on it through the process group.
        token = [f"ddp-{os.getpid()}-{torch.randint(0, 1 << 30, (1,)).item()}"]
        dist.broadcast_object_list(token, src=0, group=process_group)
        device = torch.cuda.current_device()
        comm = Comm(rank, world, device, token[0])
        if world > 1 and not comm.multicast:
            rails = tuple(r for r in rails if r != "nvls") or ("sm",)
        engine_overrides.setdefault("calibrate_max_bytes", capacity)
        engine = Engine(comm, kinds=list(rails), **engine_overrides)
        return cls(comm, engine, world, torch.cuda.Stream(priority=-1))

    def close(self) -> None:
        self.engine.close()
        self.comm.close()


def nezha_allreduce_hook(state: NezhaHookState, bucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: mean all-reduce of `bucket.buffer()` through the engine."""
    t = bucket.buffer()
    dtype = _DTYPES.get(t.dtype)
    if dtype is None:
        why = " (integer buckets have no mean; use Engine.allreduce_device for a sum)" if t.dtype in _ENGINE_ONLY else ""
        raise TypeError(f"nezha hook: unsupported gradient dtype {t.dtype}{why}")
    nbytes = t.numel() * t.element_size()
    stream = state.stream or torch.cuda.current_stream()
    stream.wait_stream(torch.cuda.current_stream())  # the gradients of this bucket are written
    with torch.cuda.stream(stream):
        state.engine.allreduce_device(t, t, nbytes, dtype, stream)
        t.div_(state.world)
        # CUDA-aware future: set_result records an event on the communication
        # stream; DDP's consumers wait on it before reading the bucket.
        fut = torch.futures.Future(devices=[t.device])
        fut.set_result(t)
    return fut
