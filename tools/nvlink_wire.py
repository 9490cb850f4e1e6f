"""NVLink wire bytes per allreduce, per rail, from NVML counters (rank 0's GPU).

Spawn with tools/run_spawn.py N tools/nvlink_wire.py [sizes_csv]. Rank 0 reads
NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX} (KiB, cumulative) summed over all
links before / after K ops of each rail and reports bytes per op against the
model: NVLS (N+1)/N * S per direction, SM / CE 2(N-1)/N * S."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17870_b200 import Comm, Rail, SymmetricBuffer
from paper_2405_17870_b200._lib import F32, RAIL_KINDS

comm = Comm.from_env(session=os.environ["NZ_SESSION"])
rank, world = comm.rank, comm.world
torch.cuda.set_device(comm.device)
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [64 << 20, 256 << 20]
nv = None
if rank == 0:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(comm.device)

    def counters():
        tx = rx = 0
        for link in range(18):
            vals = pynvml.nvmlDeviceGetFieldValues(h, [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                       (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
            if vals[0].nvmlReturn == 0:
                tx += vals[0].value.ullVal
            if vals[1].nvmlReturn == 0:
                rx += vals[1].value.ullVal
        return tx * 1024, rx * 1024
cap = max(sizes)
bi, bo = SymmetricBuffer(comm, cap), SymmetricBuffer(comm, cap)
rows = []
for kind in ("nvls", "sm", "ce"):
    r = Rail(comm, RAIL_KINDS[kind], len(rows))
    for S in sizes:
        C = max(65536, (S // (2 * world)) & ~3)
        for _ in range(3):
            r.allreduce(bi, bo, 0, S, C, F32)
        r.synchronize()
        comm.barrier()
        K = 20
        if rank == 0:
            t0, r0 = counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.ExternalStream(r.stream)
        e0.record(st)
        for _ in range(K):
            r.allreduce(bi, bo, 0, S, C, F32)
        e1.record(st)
        r.synchronize()
        comm.barrier()
        if rank == 0:
            t1, r1 = counters()
            dt = e0.elapsed_time(e1) / 1e3 / K
            model = (world + 1) / world * S if kind == "nvls" else 2 * (world - 1) / world * S
            rows.append({"world": world, "rail": kind, "bytes": S, "tx_per_op": (t1 - t0) / K,
                         "rx_per_op": (r1 - r0) / K, "model_per_dir": model,
                         "tx_over_model": round((t1 - t0) / K / model, 3), "rx_over_model": round((r1 - r0) / K / model, 3),
                         "wire_tx_GBs": round((t1 - t0) / K / dt / 1e9, 1), "wire_rx_GBs": round((r1 - r0) / K / dt / 1e9, 1),
                         "busbw_GBs": round(2 * (world - 1) / world * S / dt / 1e9, 1)})
    r.close()
if rank == 0:
    for row in rows:
        print(json.dumps(row))
bi.free(); bo.free(); comm.close()
