"""One rank issues its allreduce late (a host-side straggler): with one
process per rank the others' launches wait at their start barrier. Prints the failovers seen and
whether the results are exact. Used by tests/test_host_harness.py (and valid
on a GPU: python tests/workers/straggler_worker.py DELAY_S)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (the checker)
from paper_2405_17870_b200 import Engine, SymmetricBuffer, run_ranks  # noqa: E402
from paper_2405_17870_b200._lib import F32  # noqa: E402

TOML = ('[[rail]]\nprotocol = "ce"\nt_setup_us = 30.0\nbandwidth_bps = 5.0e11\n'
        '[[rail]]\nprotocol = "sm"\nt_setup_us = 15.0\nbandwidth_bps = 5.0e11\n')


def main():
    delay = float(sys.argv[1])
    world, n = 2, 4 << 20
    ins = [oracle.synthetic_input(F32, r, n) for r in range(world)]

    def body(comm):
        eng = Engine(comm, kinds=["ce", "sm"], rails_toml=TOML, sync_overhead_us=0.0)
        bi, bo = SymmetricBuffer(comm, n), SymmetricBuffer(comm, n)
        bi.write(ins[comm.rank], n)
        comm.barrier()
        if comm.rank == world - 1:
            time.sleep(delay)
        eng.allreduce(bi, bo, n, F32)
        eng.synchronize()
        got = np.zeros(n // 4, dtype=np.float32)
        bo.read(got, n)
        segs = eng.last_plans()[0]["segs"]
        bad = 0
        for _, off, length, c in segs:
            w = np.zeros_like(got)
            oracle.reduce_range(ins, F32, off, length, c, off, off + length, w)
            a, b = off // 4, (off + length) // 4
            bad += int(np.count_nonzero(got[a:b].view(np.uint32) != w[a:b].view(np.uint32)))
        fos = eng.failovers()
        mon = eng.state()["monitor"]
        eng.close()
        bi.free()
        bo.free()
        return {"rank": comm.rank, "mismatch": bad, "failovers": len(fos), "monitor_on": mon["on"],
                "failed": mon["failed"]}

    if "RANK" in os.environ:  # one process per rank (tests.mp_util.spawn / torchrun layout)
        from paper_2405_17870_b200 import Comm

        comm = Comm.from_env(session=os.environ["NZ_SESSION"])
        out = body(comm)
        comm.close()
        print(json.dumps(out))
    else:  # virtual ranks: a late rank's host thread holds the combined launch, nothing waits on the device
        print(json.dumps(run_ranks(world, body, timeout=300)))


if __name__ == "__main__":
    main()
