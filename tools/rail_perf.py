"""Per-rail busbw / latency sweep at N GPUs (development probe, not the bench).
usage: rail_perf.py WORLD [kind[:sm_budget],...] [sizes_csv]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.mp_util import spawn
world = int(sys.argv[1])
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["nvls", "sm", "ce"]
sizes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else \
    [8192, 65536, 262144, 1 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30]
cases = []
for k in kinds:
    kind, _, budget = k.partition(":")
    for s in sizes:
        it = 200 if s <= (1 << 20) else (50 if s <= (64 << 20) else 10)
        cases.append({"kind": kind, "sm_budget": int(budget or 0), "dtype": "f32", "nbytes": s, "iters": it,
                      "check": False})
res = spawn(world, "tests/workers/rail_worker.py", [json.dumps(cases)], timeout=900)
rows = {}
for rr in res:
    for r in rr["results"]:
        key = (cases[r["case"]]["kind"] + ":" + str(cases[r["case"]]["sm_budget"]), r["nbytes"])
        rows[key] = max(rows.get(key, 0), r["us"])
for (k, s), us in sorted(rows.items()):
    bus = 2 * (world - 1) / world * s / (us * 1e-6) / 1e9
    print(json.dumps({"world": world, "rail": k, "bytes": s, "us_max_over_ranks": round(us, 2), "busbw_GBs": round(bus, 1)}))
