"""Single-GPU kernel probe for ncu: the SM-rail fold (NDST = N) and the CE-rail
local reduce (NDST = 1) for N virtual ranks over S bytes, all buffers on cuda:0.
usage: ncu_emulate.py N S_bytes [sm|ce] [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17870_b200 import emulate_fold
from paper_2405_17870_b200._lib import F32
N, S = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "sm"
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
torch.cuda.set_device(0)
ins = [torch.rand(S // 4, device="cuda") for _ in range(N)]
outs = [torch.zeros(S // 4, device="cuda") for _ in range(N)]
chunk = max(65536, (S // (2 * N)) & ~3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(iters + 1):
    if it == 1:
        e0.record()
    for r in range(N):
        dst = [o.data_ptr() for o in outs] if mode == "sm" else [outs[r].data_ptr()]
        emulate_fold(N, r, F32, [t.data_ptr() for t in ins], dst, 0, S, chunk, 0, S)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 1e3 / iters / N  # per virtual-rank launch
# HBM bytes per launch: read N shards of S/N, write NDST shards of S/N.
ndst = N if mode == "sm" else 1
byts = (N + ndst) * S / N
print(f"mode={mode} N={N} S={S} per-launch {t*1e6:.1f} us, {byts/t/1e9:.0f} GB/s HBM-equivalent")
