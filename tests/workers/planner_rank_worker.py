"""One rank of the CPU multi-rank planner check (tests/test_multirank_cpu.py).

gloo process group of world 2 on 127.0.0.1. Every rank drives the engine's
Balancer (nz_balancer_*) over the same op stream with its OWN measured
latencies (rank-specific noise), exactly as each GPU rank's engine would.
With the engine's agreement (flush means -> max over ranks, here an
all_reduce(MAX) over gloo) every rank must make identical decisions and end
with an identical table; without it the tables drift apart. Prints one JSON
line per rank."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_17870_b200.runtime import Planner  # noqa: E402

TOML = """
[[rail]]
protocol = "nvls"
t_setup_us = 12.0
bandwidth_bps = 6.0e11
[[rail]]
protocol = "ce"
t_setup_us = 40.0
bandwidth_bps = 5.0e11
[[rail]]
protocol = "sm"
t_setup_us = 14.0
bandwidth_bps = 5.0e11
"""
TRUTH = {0: (15.0, 5.2e11), 1: (45.0, 4.1e11), 2: (16.0, 4.6e11)}  # what the rails "really" do


def agree_max(bucket, ids, means):
    t = torch.tensor(means, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def drive(planner, rank, ops=1500):
    sizes = np.random.default_rng(7).integers(13, 29, ops)  # same stream on every rank
    noise = np.random.default_rng(1000 + rank)              # this rank's own measurements
    plans = []
    for k in range(ops):
        S = 1 << int(sizes[k])
        p = planner.allocate(S)
        lat = {}
        for rid, _, length in p["segs"]:
            a, b = TRUTH[rid]
            lat[rid] = (a + length / b * 1e6) * (1.0 + 0.25 * noise.random())
        planner.record(lat)
        plans.append([p["hot"], p["segs"]])
    return plans


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{os.environ['MASTER_PORT']}", rank=rank,
                            world_size=world)
    res = {}
    for mode in ("agree", "local"):
        pl = Planner(TOML, window=10, eta=0.2, sync_overhead_us=2.0, agree=agree_max if mode == "agree" else None)
        plans = drive(pl, rank)
        table = pl.table()
        pl.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, {"plans": plans, "table": table})
        res[mode] = {"same_plans": all(g["plans"] == gathered[0]["plans"] for g in gathered),
                     "same_table": all(g["table"] == gathered[0]["table"] for g in gathered),
                     "measured_buckets": sum(1 for b in table["buckets"] if b["measured"]),
                     "hot_ops": sum(1 for h, _ in plans if h)}
    dist.destroy_process_group()
    print(json.dumps({"rank": rank, "results": res}))


if __name__ == "__main__":
    main()
