"""Ops of one engine issued on two caller streams in turn, never synchronised
in between (cold LL-size ops run on the caller's stream, hot ones fork onto
the rails' streams): every rail launch must still be ordered after the rail's
previous one (rails.cu orderBefore / orderAfter). Each op
reduces its own buffer pair; all results are checked against the oracle at
the end. One process per rank (tests.mp_util.spawn) or virtual ranks."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (the checker)
from paper_2405_17870_b200 import Engine, SymmetricBuffer, run_ranks  # noqa: E402
from paper_2405_17870_b200._lib import F32, I32  # noqa: E402

TOML = ('[[rail]]\nprotocol = "ce"\nt_setup_us = 30.0\nbandwidth_bps = 5.0e11\n'
        '[[rail]]\nprotocol = "sm"\nt_setup_us = 15.0\nbandwidth_bps = 5.0e11\n')
SIZES = [8192, 24 << 20, 4096, 16 << 20, 65536, 6 << 20, 16384, 20 << 20]


def new_stream():
    if os.environ.get("NEZHA_TEST_HOST_HARNESS_LIB"):
        import ctypes

        from paper_2405_17870_b200._lib import lib

        s = ctypes.c_void_p()
        assert lib().cudaStreamCreateWithFlags(ctypes.byref(s), 1) == 0
        return s.value
    import torch

    return torch.cuda.Stream()


def body(comm):
    world = comm.world
    eng = Engine(comm, kinds=["ce", "sm"], rails_toml=TOML, sync_overhead_us=0.0, window=2)
    streams = [new_stream(), new_stream()]
    bufs, ins = [], []
    for i, n in enumerate(SIZES):
        dt = I32 if i % 2 else F32
        x = [oracle.synthetic_input(dt, r, n, seed_base=oracle.SEED_BASE + 7 * i) for r in range(world)]
        bi, bo = SymmetricBuffer(comm, n), SymmetricBuffer(comm, n)
        bi.write(x[comm.rank], n)
        bufs.append((bi, bo, dt, n))
        ins.append(x)
    comm.barrier()
    plans = []
    for rep in range(3):
        for i, (bi, bo, dt, n) in enumerate(bufs):
            eng.allreduce(bi, bo, n, dt, streams[(i + rep) % 2])
            plans.append(eng.last_plans()[0]["segs"])
    eng.synchronize()
    bad = 0
    for i, (bi, bo, dt, n) in enumerate(bufs):
        got = np.zeros(n // 4, dtype=oracle.NP_DTYPE[dt])
        bo.read(got, n)
        for _, off, length, c in plans[-len(bufs) + i]:
            w = np.zeros_like(got)
            oracle.reduce_range(ins[i], dt, off, length, c, off, off + length, w)
            a, b = off // 4, (off + length) // 4
            bad += int(np.count_nonzero(got[a:b].view(np.uint32) != w[a:b].view(np.uint32)))
    hot = sum(1 for p in plans if len(p) > 1)
    eng.close()
    for bi, bo, _, _ in bufs:
        bi.free()
        bo.free()
    return {"rank": comm.rank, "mismatch": bad, "hot_ops": hot, "ops": len(plans)}


def main():
    if "RANK" in os.environ:
        from paper_2405_17870_b200 import Comm

        comm = Comm.from_env(session=os.environ["NZ_SESSION"])
        out = body(comm)
        comm.close()
        print(json.dumps(out))
    else:
        print(json.dumps(run_ranks(int(sys.argv[1]) if len(sys.argv) > 1 else 2, body, timeout=300)))


if __name__ == "__main__":
    main()
