"""Config 1 with 8 virtual ranks on one GPU (bench.py's N = 1 headline) for an
ncu capture of its dominant kernel, the SM rail's two-shot fold grid:
  ncu --set full --clock-control none --import-source on -k regex:fold_kernel_vr -s 2 -c 1 \\
      -f -o gpurun_out/ncu_fold_vr python tools/ncu_loopback.py
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \\
      python tools/ncu_loopback.py
then here: python tools/ncu_traffic.py gpurun_out/ncu_fold_vr.ncu-rep fold_kernel_vr 536870912
(per-launch algorithmic bytes: 2 x 8 ranks x 32 MiB, bench.py cfg1_hbm_bytes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17870_b200 import Engine, SymmetricBuffer, run_ranks
from paper_2405_17870_b200._lib import F32

V = int(sys.argv[1]) if len(sys.argv) > 1 else 8
OPS = int(sys.argv[2]) if len(sys.argv) > 2 else 4
S = 64 << 20
TOML = "".join(f'[[rail]]\nprotocol = "{k}"\nt_setup_us = 20.0\nbandwidth_bps = 5.0e11\n' for k in ("sm", "ce"))
torch.cuda.set_device(0)


def body(comm):
    torch.cuda.set_device(0)
    # Profiles and sync overhead given: no startup calibration launches.
    eng = Engine(comm, kinds=["sm", "ce"], rails_toml=TOML, algorithm=0, window=1 << 30, sync_overhead_us=0.0)
    bi, bo = SymmetricBuffer(comm, S), SymmetricBuffer(comm, S)
    x = torch.rand(S // 4, device="cuda")
    bi.write(x.data_ptr(), S)
    torch.cuda.synchronize()
    for _ in range(OPS):
        eng.allreduce(bi, bo, S, F32)
    eng.synchronize()
    plan = eng.last_plans()[0]["segs"]
    eng.close()
    bi.free()
    bo.free()
    return plan


print("ok", run_ranks(V, body, timeout=900)[0])
