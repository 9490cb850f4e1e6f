#!/usr/bin/env python3
"""Benchmark of the B200 multi-rail allreduce (Nezha, arxiv 2405.17870).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Metric (BASELINE.json): 8-GPU allreduce busbw GB/s vs size (4KB-1GB); 8KB p50
latency; failover ms. A "step" is one engine allreduce of the headline payload
(1 GiB fp32, synthetic) on the configured rails (default: the configs[2]
rail set NVLS + copy-engine + SM under the cold/hot state machine, swept
4 KiB-1 GiB as configs[1] specifies; `--rails nvls,ce` is configs[1] itself). `value` = busbw = ringVolume(N, S) / t with
t the max over ranks of the device time per step (N = 1: algbw S / t, no
NVLink exchange exists). Inputs are 1 GiB, larger than the 126 MB L2, so no
flush is needed between steps. Rank 0 prints one JSON line.

Reference arm (--impl reference): the CPU baseline — the SPEC ring restated on
the reference's own InMemoryFabric (oracle/_ref, compiled from
/root/reference/proj/src), ranks as threads, timed on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "8-GPU allreduce busbw GB/s vs size (4KB–1GB); 8KB p50 latency; failover ms"
NVLINK_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md; 900 nominal)
GiB = 1 << 30


def ring_volume(n: int, s: int) -> int:
    return (2 * (n - 1) * s + n // 2) // n if n >= 2 else 0


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", os.environ.get("RANK", "0"))))


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(kernel: str, per_launch_bytes: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` summary (profiles/ncu_traffic.json), when it
    was captured at this launch size; else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[kernel]
    except Exception:
        return None
    return t["dram_bytes"] if t.get("per_launch_bytes") == per_launch_bytes else None


def wire_bytes(kind: str, world: int, seg: int) -> int:
    """Bytes one GPU must send over NVLink per op of `seg` bytes on a rail (per
    direction): ring-equivalent rails 2(N-1)/N*S (Eq. 1); NVLS (N+1)/N*S — the
    switch reads every rank's copy once and multicasts the reduced shards."""
    if kind == "nvls":
        return (world + 1) * seg // world
    return ring_volume(world, seg)


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.path = f"/tmp/nezha_clocks_{os.getpid()}_{device}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)  # first sample lands before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            try:
                self.lines = [l.strip() for l in open(self.path) if l.strip()]
                os.unlink(self.path)
            except OSError:
                self.lines = []

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            p = [x.strip() for x in l.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline ---
def cpu_baseline(world_sim: int = 8, nbytes: int = 64 << 20, budget_s: float = 20.0):
    """Config 1 of BASELINE.json on the host: world_sim simulated ranks (threads)
    on the reference InMemoryFabric, 2 identical rails, static 50/50 split, Ring,
    64 KiB frames, fp32. Returns the busbw GB/s and the sample description."""
    import numpy as np

    import oracle  # CPU baseline leg: the only bench use of oracle/

    if not oracle.inmem_available():
        return None
    inputs = [oracle.synthetic_input(oracle.F32, r, nbytes) for r in range(world_sim)]
    outs = [np.zeros_like(inputs[0]) for _ in range(world_sim)]
    half = (nbytes // 2) & ~3
    segs = [(0, 0, half), (1, half, nbytes - half)]
    oracle.inmem_allreduce(inputs, oracle.F32, segs, 2, chunked=False, outputs=outs)  # warm-up
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < 3 or (time.perf_counter() < t_end and len(times) < 20):
        _, us, _ = oracle.inmem_allreduce(inputs, oracle.F32, segs, 2, chunked=False, outputs=outs)
        times.append(us * 1e-6)
    t = statistics.mean(times)
    threads = world_sim * 2
    return {"value": round(ring_volume(world_sim, nbytes) / t / 1e9, 4), "unit": "GB/s", "cores": threads,
            "host_cpus": len(os.sched_getaffinity(0)), "kind": "port",
            "sample": f"config 1: {world_sim} simulated ranks x 2 rails (threads), fp32 {nbytes >> 20} MiB, static "
                      f"50/50, Ring, 64 KiB frames, {len(times)} timed ops (mean {t * 1e3:.1f} ms/op); SPEC ring "
                      f"restated on the reference InMemoryFabric compiled from /root/reference/proj/src"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    world_sim = max(2, world)
    nbytes = 64 << 20
    res = cpu_baseline(world_sim, nbytes, budget_s=max(5.0, 3.0 * args.steps))
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return 0
    v = res["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ring_volume(world_sim, nbytes) / (v * 1e9) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"CPU allreduce, {world_sim} simulated ranks, 2 rails 50/50, 64 MiB fp32 sample",
                       "bytes_per_rank": nbytes, "ranks": f"{world_sim} simulated (threads)"},
            "cpu_baseline": res,
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- our arm ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rails", default="nvls,ce,sm",
                    help="comma list of nvls|ce|sm (configs[1] = nvls,ce; configs[2] = nvls,ce,sm)")
    ap.add_argument("--bytes", type=int, default=GiB)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16", "i32"])
    ap.add_argument("--tune-ops", type=int, default=200, help="balancer convergence ops before timing")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-failover", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep-max", type=int, default=GiB)
    ap.add_argument("--tune", action="store_true",
                    help="engine measures its CTA budgets and protocol crossovers at startup (tune_budgets=1)")
    ap.add_argument("--graph", action="store_true",
                    help="small sizes replayed from CUDA graphs: a graph_safe engine vs NCCL (device time per op)")
    ap.add_argument("--nccl-graph", action="store_true",
                    help="also time NCCL at <= 1 MiB from a captured CUDA graph (no host launch overhead)")
    ap.add_argument("--nccl-algos", action="store_true",
                    help="also time NCCL with NCCL_ALGO=NVLS and =Ring (SURVEY.md 8d) at a few sizes")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    from paper_2405_17870_b200 import Comm, Engine, Rail, SymmetricBuffer
    from paper_2405_17870_b200._lib import DTYPES, RAIL_KINDS
    from paper_2405_17870_b200.runtime import kernel_launch_count

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    session = f"bench-{os.environ.get('MASTER_PORT', '0')}-{os.environ.get('TORCHELASTIC_RUN_ID', str(os.getppid()))}"
    comm = Comm(rank, world, local, session)
    kinds = args.rails.split(",")
    if world > 1 and not comm.multicast and "nvls" in kinds:  # no NVSwitch multicast on this box
        kinds = [k for k in kinds if k != "nvls"] or ["sm"]
    dt = DTYPES[args.dtype]
    S = args.bytes
    eng = Engine(comm, kinds=kinds, window=5, eta=0.2, demote_after=1, calibrate_max_bytes=min(GiB, max(S, 1 << 20)),
                 tune_budgets=1 if args.tune else 0)

    def max_over_ranks(x: float) -> float:
        vals = comm.allgather_bytes(json.dumps(x).encode().ljust(32))
        return max(json.loads(v.decode().strip()) for v in vals)

    cap = max(S, args.sweep_max if not args.no_sweep else 0, 8192)
    bin_, bout = SymmetricBuffer(comm, cap), SymmetricBuffer(comm, cap)
    g = torch.Generator(device="cuda").manual_seed(0x4E5A0000 + rank)
    tdt = {0: torch.float32, 1: torch.bfloat16, 2: torch.int32}[dt]
    if dt == 2:
        x = torch.randint(-(1 << 20), 1 << 20, (cap // 4,), device="cuda", generator=g, dtype=torch.int32)
    else:
        x = (torch.rand(cap // x_es(dt), device="cuda", generator=g) * 2 - 1).to(tdt)
    bin_.write(x.data_ptr(), cap)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()

    def timed(nbytes, iters, warm):
        for _ in range(warm):
            eng.allreduce(bin_, bout, nbytes, dt, stream)
        eng.synchronize()
        comm.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            eng.allreduce(bin_, bout, nbytes, dt, stream)
        e1.record(stream)
        e1.synchronize()
        eng.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / iters
        return max_over_ranks(t)

    # Balancer convergence on the headline size (one-time, like NCCL tuning).
    for _ in range(args.tune_ops):
        eng.allreduce(bin_, bout, S, dt, stream)
    eng.synchronize()

    # ---- headline: K timed steps of S bytes --------------------------------
    for _ in range(max(args.warmup, 3)):
        eng.allreduce(bin_, bout, S, dt, stream)
    eng.synchronize()
    t_est = timed(S, 3, warm=0)
    soak_ops = max(1, min(2000, int(0.4 / max(t_est, 1e-6))))
    eng.stats_reset()
    comm.barrier()
    torch.cuda.synchronize()
    launches0 = kernel_launch_count()
    with ClockSampler(local) as clk:
        # Keep the GPU under the same load for ~0.4 s so the sampler sees it
        # running, then time exactly K steps back to back.
        for _ in range(soak_ops):  # same count on every rank (collective)
            eng.allreduce(bin_, bout, S, dt, stream)
        eng.synchronize()
        comm.barrier()
        eng.stats_reset()
        launches0 = kernel_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            eng.allreduce(bin_, bout, S, dt, stream)
        e1.record(stream)
        e1.synchronize()
    launches = kernel_launch_count() - launches0
    eng.synchronize()
    t_step = max_over_ranks(e0.elapsed_time(e1) / 1e3 / args.steps)
    busbw = ring_volume(world, S) / t_step / 1e9
    algbw = S / t_step / 1e9
    value = busbw if world > 1 else algbw
    plan = eng.last_plans()[0] if eng.last_plans() else {}
    # Dominant rail (largest share): its per-op time on its own stream.
    peaks = measured_peaks()
    stats = {k: eng.rail_stats(i) for i, k in enumerate(kinds)}
    dom = max(range(len(kinds)), key=lambda i: stats[kinds[i]]["bytes"])
    st = stats[kinds[dom]]
    roofline = None
    if st["ops"] == 0 and plan.get("segs"):
        # Cold plan: one rail carried the whole step on the caller's stream.
        dom = plan["segs"][0][0]
        st = {"ops": args.steps, "total_us": t_step * 1e6 * args.steps, "bytes": S * args.steps}
    if st["ops"]:
        t_rail = max_over_ranks(st["total_us"] / st["ops"] * 1e-6)
        seg = st["bytes"] / st["ops"]
        if world > 1:
            wb = wire_bytes(kinds[dom], world, int(seg))
            ach = wb / t_rail / 1e9
            roofline = {"bound": "nvlink", "kernel": f"{kinds[dom]} rail", "achieved": round(ach, 1),
                        "peak": NVLINK_GBS, "unit": "GB/s", "frac": round(ach / NVLINK_GBS, 4), "traffic": None,
                        "per_launch_bytes": wb,
                        "note": "achieved = NVLink bytes one GPU must send per op (ring rails 2(N-1)/N*S, NVLS "
                                "(N+1)/N*S) / rail time per op (CUDA events on the rail stream); peak = measured "
                                "peer copy 770 GB/s per direction (B200_PROFILING.md; 900 nominal). traffic: ncu "
                                "cannot replay kernels with cross-GPU barriers (profiles/README.md)"}
        else:
            hbm = peaks.get("hbm_gbs", 6650.0)
            ach = 2 * seg / t_rail / 1e9
            roofline = {"bound": "hbm", "kernel": f"{kinds[dom]} rail (N=1 copy)", "achieved": round(ach, 1),
                        "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                        "traffic": ncu_traffic("copy_kernel", int(2 * seg)),
                        "per_launch_bytes": int(2 * seg),
                        "note": "N=1: the allreduce is a copy in->out, 2S HBM bytes; peak = MEASURED_PEAKS.json "
                                "hbm_gbs" + ("" if "hbm_gbs" in peaks else " (fallback)")}

    out = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
           "config": {"workload": f"multi-rail ({'+'.join(kinds)}) state-machine {args.dtype} allreduce of "
                                  f"{S} B per rank (value = busbw at this size; N=1: algbw)",
                      "bytes_per_rank": S, "ranks": world,
                      "l2": "inputs (1 GiB) larger than the 126 MB L2; no flush",
                      "algbw_GBs": round(algbw, 2), "busbw_GBs": round(busbw, 2), "plan": plan},
           "roofline": roofline, "gpu_launches": launches, "clocks": clk.summary()}

    # ---- NCCL on the same sizes --------------------------------------------
    nccl = {}
    pg = None
    if world > 1 and not args.no_nccl:
        import torch.distributed as dist
        saved = os.dup(1)
        os.dup2(2, 1)  # NCCL prints its banner on stdout; keep stdout for the one JSON line
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            pg = dist
            warm = torch.ones(1, device="cuda")
            pg.all_reduce(warm)
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover
            out["nccl_error"] = str(e)[:200]
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)

    def nccl_time(nbytes, iters, group=None):
        t = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
        for _ in range(5):
            pg.all_reduce(t, group=group)
        torch.cuda.synchronize()
        pg.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            pg.all_reduce(t, group=group)
        b.record()
        b.synchronize()
        return max_over_ranks(a.elapsed_time(b) / 1e3 / iters)

    def nccl_graph_time(nbytes, per_graph=50, replays=10):
        """NCCL device time per op: `per_graph` allreduces captured in one CUDA
        graph, replayed; excludes the Python / launch overhead of nccl_time."""
        t = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                pg.all_reduce(t)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(per_graph):
                pg.all_reduce(t)
        g.replay()
        torch.cuda.synchronize()
        pg.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(replays):
            g.replay()
        b.record()
        b.synchronize()
        return max_over_ranks(a.elapsed_time(b) / 1e3 / (replays * per_graph))

    if pg is not None:
        tn = nccl_time(S, max(5, args.steps // 2))
        nccl["busbw_headline"] = round(ring_volume(world, S) / tn / 1e9, 2)
        out["nccl_busbw_GBs"] = nccl["busbw_headline"]
        if args.nccl_algos:
            # NCCL reads NCCL_ALGO when a communicator is created: one group per algorithm.
            algos = {}
            for algo in ("NVLS", "Ring"):
                old = os.environ.get("NCCL_ALGO")
                os.environ["NCCL_ALGO"] = algo
                try:
                    g = pg.new_group(backend="nccl")
                    algos[algo] = {str(sz): round(ring_volume(world, sz) / nccl_time(sz, 20 if sz > (64 << 20) else 100,
                                                                                       g) / 1e9, 2)
                                   for sz in (8192, 1 << 20, 64 << 20, S)}
                except Exception as e:  # pragma: no cover
                    algos[algo] = {"error": str(e)[:160]}
                finally:
                    if old is None:
                        os.environ.pop("NCCL_ALGO", None)
                    else:
                        os.environ["NCCL_ALGO"] = old
            out["nccl_algos_busbw_GBs"] = algos

    # ---- sweep 4 KiB .. 1 GiB ----------------------------------------------
    if not args.no_sweep:
        sweep = []
        s = 4096
        while s <= min(args.sweep_max, cap):
            it = 200 if s <= (1 << 20) else (40 if s <= (64 << 20) else 8)
            t = timed(s, it, warm=20 if s <= (64 << 20) else 12)
            row = {"bytes": s, "us": round(t * 1e6, 2), "algbw_GBs": round(s / t / 1e9, 2),
                   "busbw_GBs": round(ring_volume(world, s) / t / 1e9, 2),
                   "hot": bool(eng.last_plans()[0]["hot"]) if eng.last_plans() else None,
                   "rails": sorted({seg[0] for p in eng.last_plans() for seg in p["segs"]})}
            if pg is not None:
                tn = nccl_time(s, it)
                row["nccl_busbw_GBs"] = round(ring_volume(world, s) / tn / 1e9, 2)
                row["nccl_us"] = round(tn * 1e6, 2)
                if args.nccl_graph and s <= (1 << 20):
                    try:
                        row["nccl_graph_us"] = round(nccl_graph_time(s) * 1e6, 2)
                    except Exception as e:  # pragma: no cover
                        row["nccl_graph_error"] = str(e)[:120]
            sweep.append(row)
            s *= 2
        out["sweep"] = sweep

    # ---- 8 KiB p50 latency: engine (cold start) vs each rail alone vs NCCL --
    def p50_host(fn, n=1000):
        """Per op: every rank issues at one agreed CLOCK_MONOTONIC instant (the
        clock is system-wide, so one box shares it) and stops when its result
        is on the host's side of a synchronize; the op's latency is the max over
        ranks of (done - start), i.e. issued on all GPUs -> complete on all GPUs
        (SURVEY.md 8d). p50 over n ops. Removes the skew a plain barrier leaves."""
        import struct
        lat = []
        for _ in range(n):
            prop = time.perf_counter() + 1e-3  # well past the exchange itself
            start = max(struct.unpack("d", b)[0] for b in comm.allgather_bytes(struct.pack("d", prop)))
            while time.perf_counter() < start:
                pass
            fn()
            torch.cuda.synchronize()
            lat.append(time.perf_counter() - start)
        mine = struct.pack(f"{n}d", *lat)
        per_op = [max(v) for v in zip(*[struct.unpack(f"{n}d", b) for b in comm.allgather_bytes(mine)])]
        return statistics.median(per_op) * 1e6

    lat = {}
    lat["engine_us"] = round(p50_host(lambda: eng.allreduce(bin_, bout, 8192, dt, stream)), 2)
    if world > 1:
        for k in ("nvls", "ce", "sm"):
            if k == "nvls" and not comm.multicast:
                continue
            r = Rail(comm, RAIL_KINDS[k], 10 + len(lat))
            lat[f"{k}_alone_us"] = round(p50_host(lambda: (r.allreduce(bin_, bout, 0, 8192, 65536, dt),
                                                            r.synchronize())), 2)
            r.close()
        if pg is not None:
            t8 = torch.empty(2048, dtype=torch.float32, device="cuda")
            lat["nccl_us"] = round(p50_host(lambda: pg.all_reduce(t8)), 2)
    out["latency_8k_p50_us"] = lat

    # ---- small sizes from CUDA graphs (no host launch cost on either side) --
    if args.graph and world > 1:
        geng = Engine(comm, kinds=kinds, window=5, eta=0.2, demote_after=1, calibrate_max_bytes=1 << 22,
                      graph_safe=1)
        rows = {}
        for sz in (8192, 65536, 1 << 20):
            try:
                geng.allreduce(bin_, bout, sz, dt)  # warm-up
                geng.synchronize()
                g = torch.cuda.CUDAGraph()
                per_graph, replays = 50, 10
                with torch.cuda.graph(g, stream=torch.cuda.Stream()):
                    for _ in range(per_graph):
                        geng.allreduce(bin_, bout, sz, dt, torch.cuda.current_stream())
                g.replay()
                torch.cuda.synchronize()
                comm.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(replays):
                    g.replay()
                b.record()
                b.synchronize()
                row = {"ours_us": round(max_over_ranks(a.elapsed_time(b) * 1e3 / (replays * per_graph)), 2),
                       "rails": sorted({seg[0] for p in geng.last_plans() for seg in p["segs"]})}
                if pg is not None:
                    row["nccl_us"] = round(nccl_graph_time(sz) * 1e6, 2)
                rows[str(sz)] = row
            except Exception as e:  # pragma: no cover
                rows[str(sz)] = {"error": str(e)[:160]}
        geng.close()
        out["graph_replay_us"] = rows

    # ---- e2e through the public host API (H2D + allreduce + D2H) ------------
    if not args.no_e2e:
        hin = torch.empty(S, dtype=torch.uint8).pin_memory()
        hout = torch.empty(S, dtype=torch.uint8).pin_memory()
        hin.copy_(x.view(torch.uint8)[:S].cpu())
        for _ in range(2):
            eng.allreduce_host(hin, hout, S, dt)
        k = max(3, min(args.steps, 10))
        comm.barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            eng.allreduce_host(hin, hout, S, dt)
        te = max_over_ranks((time.perf_counter() - t0) / k)
        eng.synchronize()
        ev = (ring_volume(world, S) if world > 1 else S) / te / 1e9
        out["e2e"] = {"value": round(ev, 2), "unit": "GB/s", "h2d_bytes_per_step": S, "d2h_bytes_per_step": S,
                      "ms_per_step": round(te * 1e3, 3),
                      "note": "nz_engine_allreduce_host from pinned host memory, wall clock, max over ranks"}

    # ---- failover: config 4 shape (bf16 256 MiB, largest-alpha rail fails mid-op)
    if world > 1 and not args.no_failover and len(kinds) > 1:
        fs = min(256 << 20, cap)
        plan_f = eng.plan(fs)["pieces"][0]["plan"]
        segs = plan_f["segs"]
        if segs:
            victim = max(segs, key=lambda sgm: sgm[2])
            nch =-(-victim[2] // max(65536, (victim[2] // (2 * world)) & ~3))
            eng.inject_failure(eng.op_seq, victim[0], nch // 2)
            eng.allreduce(bin_, bout, fs, DTYPES["bf16"], stream)
            eng.synchronize()
            fo = eng.last_failover()
            if fo:
                out["failover"] = {"failed_rail": kinds[fo["failed_rail"]], "target_rail": kinds[fo["target_rail"]],
                                   "orphan_bytes": fo["orphan_length"], "detect_us": round(fo["detect_us"], 2),
                                   "host_detect_us": round(fo["host_detect_us"], 2),
                                   "resume_us": round(fo["resume_us"], 2), "done_us": round(fo["done_us"], 2),
                                   "payload": "bf16 256 MiB"}
                # failover = device fault stamp -> orphan fully reduced on the survivor
                out["failover_ms"] = round(max_over_ranks(fo["done_us"]) / 1e3, 4)
            eng.readmit(victim[0])

    # ---- config 3: mixed 8 KiB - 4 MiB stream through the state machine ------
    if not args.no_sweep:
        import random

        rnd = random.Random(7)
        n_ops = 2000
        sizes = [max(4, int(2 ** rnd.uniform(13, 22)) & ~3) for _ in range(n_ops)]
        for s_ in sizes[:50]:
            eng.allreduce(bin_, bout, s_, dt, stream)
        eng.synchronize()
        comm.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s_ in sizes:
            eng.allreduce(bin_, bout, s_, dt, stream)
        b.record(stream)
        b.synchronize()
        eng.synchronize()
        tm = max_over_ranks(a.elapsed_time(b) / 1e3)
        table = eng.state()["table"]
        hot_buckets = [e["bucket"] for e in table["buckets"] if e["hot"] and 13 <= e["bucket"] <= 22]
        out["config3_mixed_stream"] = {"ops": n_ops, "sizes": "log-uniform 8 KiB-4 MiB, seed 7",
                                       "mean_us_per_op": round(tm / n_ops * 1e6, 2),
                                       "algbw_GBs": round(sum(sizes) / tm / 1e9, 2),
                                       "hot_buckets": hot_buckets, "threshold": table["threshold"]}
        if pg is not None:
            tt = {s_: torch.empty(s_ // 4, dtype=torch.float32, device="cuda") for s_ in set(sizes)}
            torch.cuda.synchronize()
            a.record()
            for s_ in sizes:
                pg.all_reduce(tt[s_])
            b.record()
            b.synchronize()
            tn = max_over_ranks(a.elapsed_time(b) / 1e3)
            out["config3_mixed_stream"]["nccl_mean_us_per_op"] = round(tn / n_ops * 1e6, 2)
            del tt

    # ---- config 5: DDP gradient-bucket traces ----------------
    if not args.no_sweep:
        # torch 2.11's own DDP bucketing of the two models (tests/golden/make_ddp_buckets.py).
        traces = json.load(open(os.path.join(ROOT, "tests", "golden", "ddp_buckets.json")))
        c5 = {}
        for name, buckets in traces.items():
            offs, o = [], 0
            for nb in buckets:
                offs.append(o)
                o += nb
            if max(buckets) > cap:
                continue
            for _ in range(3):
                for nb in buckets:
                    eng.allreduce(bin_, bout, nb, dt, stream)
            eng.synchronize()
            comm.barrier()
            iters = 5
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(iters):
                for nb in buckets:
                    eng.allreduce(bin_, bout, nb, dt, stream)
            b.record(stream)
            b.synchronize()
            eng.synchronize()
            t_it = max_over_ranks(a.elapsed_time(b) / 1e3 / iters)
            row = {"buckets": len(buckets), "bytes": o, "ms_per_iter": round(t_it * 1e3, 3),
                   "busbw_GBs": round(ring_volume(world, o) / t_it / 1e9, 2) if world > 1 else None}
            if pg is not None:
                tb = [torch.empty(nb // 4, dtype=torch.float32, device="cuda") for nb in buckets]
                for t_ in tb:
                    pg.all_reduce(t_)
                torch.cuda.synchronize()
                a.record()
                for _ in range(iters):
                    for t_ in tb:
                        pg.all_reduce(t_)
                b.record()
                b.synchronize()
                tn = max_over_ranks(a.elapsed_time(b) / 1e3 / iters)
                row["nccl_ms_per_iter"] = round(tn * 1e3, 3)
                del tb
            c5[name] = row
        out["config5_ddp_buckets"] = c5

    # ---- CPU baseline (rank 0, N = 1 only) ----------------------------------
    if world == 1 and rank == 0 and not args.no_cpu:
        cb = cpu_baseline()
        if cb:
            out["cpu_baseline"] = cb

    st_ = eng.state()
    out["engine_state"] = {"sync_overhead_us": st_["sync_overhead_us"], "threshold": st_["table"]["threshold"],
                           "rails": [{"kind": r["kind"], "calibration": r["calibration"]} for r in st_["rails"]],
                           "concurrent": st_.get("concurrent", [])}
    eng.close()
    bin_.free()
    bout.free()
    comm.close()
    if pg is not None:
        pg.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))
    return 0


def x_es(dt: int) -> int:
    return 2 if dt == 1 else 4


if __name__ == "__main__":
    sys.exit(main())
