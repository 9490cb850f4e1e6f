"""Condenses bench.py JSON lines (files or a log containing them) into the
numbers profiles/README.md quotes. usage: summarize_bench.py FILE [FILE...]"""
import json
import sys


def lines(path):
    for l in open(path):
        l = l.strip()
        if l.startswith("{") and '"metric"' in l:
            try:
                yield json.loads(l)
            except ValueError:
                pass


def main():
    for path in sys.argv[1:]:
        for d in lines(path):
            n = d.get("n_gpus")
            print(f"== {path}: impl={d.get('impl', 'ours')} N={n} value={d.get('value')} {d.get('unit')} "
                  f"ms/step={d.get('ms_per_step')}")
            if d.get("impl") == "reference":
                continue
            r = d.get("roofline") or {}
            print(f"   roofline {r.get('kernel')}: {r.get('achieved')}/{r.get('peak')} {r.get('unit')} "
                  f"frac={r.get('frac')} traffic={r.get('traffic')}")
            e = d.get("e2e") or {}
            print(f"   e2e {e.get('value')} {e.get('unit')}; nccl headline {d.get('nccl_busbw_GBs')}; "
                  f"clocks {d.get('clocks')}; launches {d.get('gpu_launches')}")
            print(f"   8KiB p50 {d.get('latency_8k_p50_us')}")
            for row in d.get("sweep", []):
                print(f"   {row['bytes']:>11} ours {row.get('us'):>9} us {row.get('busbw_GBs'):>8} GB/s rails "
                      f"{row.get('rails')} | nccl {row.get('nccl_us')} us {row.get('nccl_busbw_GBs')} GB/s"
                      + (f" graph {row['nccl_graph_us']}" if "nccl_graph_us" in row else ""))
            for k in ("failover", "config3", "config5", "graph_replay_us", "nccl_algos_busbw_GBs"):
                if k in d:
                    print(f"   {k}: {json.dumps(d[k])[:400]}")


if __name__ == "__main__":
    main()
