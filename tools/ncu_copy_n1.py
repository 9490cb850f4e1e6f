"""N = 1 engine allreduce (the bench's N=1 hot kernel, copy_kernel) for an
ncu --set full capture:
  ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 1 -c 1 \\
      -o gpurun_out/ncu_copy_n1 python tools/ncu_copy_n1.py
then here: python tools/ncu_traffic.py gpurun_out/ncu_copy_n1.ncu-rep copy_kernel 2147483648"""
import os, sys, uuid
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17870_b200 import Comm, Engine, SymmetricBuffer
from paper_2405_17870_b200._lib import F32
S = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
torch.cuda.set_device(0)
comm = Comm(0, 1, 0, session=uuid.uuid4().hex[:8])
# Profiles given, sync overhead given: no startup calibration, so the only
# copy_kernel launches are the 1 GiB ones below (ncu -s 1 -c 1 takes the 2nd).
TOML = "".join(f'[[rail]]\nprotocol = "{k}"\nt_setup_us = 10.0\nbandwidth_bps = 1.0e12\n' for k in ("nvls", "ce", "sm"))
eng = Engine(comm, kinds=["nvls", "ce", "sm"], rails_toml=TOML, sync_overhead_us=0.0)
bi, bo = SymmetricBuffer(comm, S), SymmetricBuffer(comm, S)
for _ in range(5):
    eng.allreduce(bi, bo, S, F32)
eng.synchronize()
print("ok", eng.last_plans()[0]["segs"])
eng.close(); bi.free(); bo.free(); comm.close()
