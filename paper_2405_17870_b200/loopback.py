"""Virtual ranks on one GPU (nz_comm_init_loopback).

``run_ranks(world, fn)`` runs ``fn(comm)`` for every rank of a ``world``-rank
job in its own host thread — the one-thread-per-rank analogue of one process
per GPU — with every rank's Comm a loopback comm on the same device. The
library runs each cross-rank kernel of the ranks as one grid (blockIdx.y =
rank), so the rails' real protocols (barriers, LL flags, copy-engine DMA
between ranks' buffers, failure detection and reroute) execute on one B200.
The calls into the library release the GIL (ctypes), so the ranks proceed
concurrently.
"""
from __future__ import annotations

import sys
import threading
import traceback
import uuid

from .runtime import Comm


class RankFailure(RuntimeError):
    """One or more virtual ranks raised; the message carries every traceback."""


def run_ranks(world: int, fn, device: int = 0, session: str | None = None, timeout: float = 600.0,
              timeout_ms: int = 120000) -> list:
    session = session or f"loop-{uuid.uuid4().hex[:12]}"
    results: list = [None] * world
    errors: list = [None] * world

    def body(rank: int) -> None:
        comm = None
        torch = sys.modules.get("torch")  # only a caller that uses torch needs its device set per thread
        if torch is not None:
            try:
                torch.cuda.set_device(device)
            except Exception:  # the library sets the device itself
                pass
        try:
            comm = Comm(rank, world, device, session, timeout_ms=timeout_ms, loopback=True)
            results[rank] = fn(comm)
        except BaseException:  # noqa: BLE001 - reported below with the rank
            errors[rank] = traceback.format_exc()
            if comm is not None:  # peers waiting on this rank fail now, not after timeout_ms
                try:
                    comm.abort()
                except BaseException:  # noqa: BLE001
                    pass
        finally:
            if comm is not None:
                try:
                    comm.close()
                except BaseException:  # noqa: BLE001
                    if errors[rank] is None:
                        errors[rank] = traceback.format_exc()

    threads = [threading.Thread(target=body, args=(r,), name=f"nz-vrank-{r}", daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    import time

    deadline = time.monotonic() + timeout  # one deadline for the whole job
    for t in threads:
        t.join(max(0.0, deadline - time.monotonic()))
    hung = [r for r, t in enumerate(threads) if t.is_alive()]
    if hung or any(errors):
        msg = [f"virtual rank {r} did not finish within {timeout} s" for r in hung]
        msg += [f"--- virtual rank {r}\n{e}" for r, e in enumerate(errors) if e]
        raise RankFailure("\n".join(msg))
    return results
