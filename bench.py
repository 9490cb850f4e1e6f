#!/usr/bin/env python3
"""Benchmark of the B200 multi-rail allreduce (Nezha, arxiv 2405.17870).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Metric (BASELINE.json): 8-GPU allreduce busbw GB/s vs size (4KB-1GB); 8KB p50
latency; failover ms. busbw = ringVolume(N, S) / t (Eq. 1,
proj/src/core/math.cpp:7-16), t the max over ranks of the device time per
step.

The headline workload is BASELINE config 1 — 2 rails with identical profiles
(so a static 50/50 split: [0, 32 MiB) and [32 MiB, 64 MiB)), Ring, 64 MiB fp32
per rank — run through the product's public engine API (nz_engine_allreduce),
one "step" = one allreduce of the whole job:
  * N = 1 (no torchrun): the config's 8 ranks as 8 virtual ranks on the one
    B200 (nz_comm_init_loopback, one host thread per rank; the SM and CE
    rails' own kernels and DMA, each cross-rank kernel one co-resident grid
    over the ranks). All inter-rank traffic is HBM traffic, so the roofline
    is HBM (MEASURED_PEAKS.json hbm_gbs).
  * N > 1: N real GPUs, rails NVLS + copy-engine (configs[1]'s set; SM + CE
    without multicast); roofline NVLink 900 GB/s per direction,
    plus the 4 KiB-1 GiB state-machine sweep, NCCL, 8 KiB latency, failover,
    config 3 and config 5 as secondary fields.
Inputs (8 x 64 MiB per buffer) exceed the 126 MB L2, so no flush is needed.

Reference arm (--impl reference): the CPU baseline — the SPEC ring restated on
the reference's own InMemoryFabric (oracle/_ref, compiled from
/root/reference/proj/src), the same config (8 simulated ranks at N = 1, else N),
ranks as threads, timed on this host's cores; rank 0 only.
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
NVLINK_GBS = 900.0       # NVLink 5 per direction per GPU (BASELINE.md "Roofline definitions")
NVLINK_COPY_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md), secondary
GiB = 1 << 30
CFG1_BYTES = 64 << 20
CFG1_RANKS = 8
ALGO_RING, ALGO_RING_CHUNKED = 0, 1


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


def identical_rails_toml(kinds) -> str:
    """Rails config with identical profiles: Eq. 8 gives alpha = 1/R, so the
    split is static (config 1's 50/50 with two rails)."""
    return "".join(f'[[rail]]\nprotocol = "{k}"\nt_setup_us = 20.0\nbandwidth_bps = 5.0e11\n' for k in kinds)


def cfg1_hbm_bytes(world: int, seg: int, kind: str) -> int:
    """Algorithmic HBM bytes of one rail op over a segment of `seg` bytes when
    all `world` ranks live on one GPU (loopback): SM two-shot —
    every rank reads its shard from every rank and writes the sum to every
    rank: 2 * world * seg; copy engine — per rank the gather reads and writes
    (N-1)/N seg, the reduce reads seg and writes seg/N, the scatter reads and
    writes (N-1)/N seg: world * seg * (5N - 3) / N."""
    if kind == "sm":
        return 2 * world * seg
    return world * seg * (5 * world - 3) // world


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
def cpu_baseline(world_sim: int = CFG1_RANKS, nbytes: int = CFG1_BYTES, budget_s: float = 20.0, min_ops: int = 3,
                 max_ops: int = 20):
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
    while len(times) < min_ops or (time.perf_counter() < t_end and len(times) < max_ops):
        _, us, _ = oracle.inmem_allreduce(inputs, oracle.F32, segs, 2, chunked=False, outputs=outs)
        times.append(us * 1e-6)
    t = statistics.mean(times)
    threads = world_sim * 2
    return {"value": round(ring_volume(world_sim, nbytes) / t / 1e9, 4), "unit": "GB/s", "cores": threads,
            "host_cpus": len(os.sched_getaffinity(0)), "kind": "port", "ms_per_op": round(t * 1e3, 3),
            "ops": len(times),
            "sample": f"config 1: {world_sim} simulated ranks x 2 rails (one thread per rank and rail), fp32 "
                      f"{nbytes >> 20} MiB per rank, static 50/50, Ring, 64 KiB frames, {len(times)} timed ops "
                      f"(mean {t * 1e3:.1f} ms/op); SPEC ring restated on the reference InMemoryFabric compiled "
                      f"from /root/reference/proj/src"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    world_sim = CFG1_RANKS if world == 1 else world  # the same ranks as our arm's headline
    nbytes = CFG1_BYTES
    res = cpu_baseline(world_sim, nbytes, budget_s=600.0, min_ops=max(1, args.steps), max_ops=max(1, args.steps))
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return 0
    v = res["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_op"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"config 1: {world_sim} ranks, 2 rails with identical profiles (static 50/50), "
                                   f"Ring, {nbytes >> 20} MiB fp32 per rank; CPU reference on host threads",
                       "bytes_per_rank": nbytes, "ranks": world_sim, "same_config": True},
            "cpu_baseline": res,
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------- N = 1: loopback ----
def run_loopback(args):
    """Config 1 with its 8 ranks as virtual ranks on the one B200."""
    import torch

    from paper_2405_17870_b200 import Engine, SymmetricBuffer, run_ranks
    from paper_2405_17870_b200._lib import BF16, F32
    from paper_2405_17870_b200.runtime import kernel_launch_count

    V, S = args.virtual_ranks, CFG1_BYTES
    kinds = ["sm", "ce"]
    toml = identical_rails_toml(kinds)
    torch.cuda.set_device(0)
    torch.cuda.init()
    steps, warm = args.steps, max(args.warmup, 3)
    bar = threading.Barrier(V)
    shared = {}
    clk = ClockSampler(0)
    fo_bytes = 256 << 20

    def body(comm):
        torch.cuda.set_device(0)
        r = comm.rank
        eng = Engine(comm, kinds=kinds, rails_toml=toml, algorithm=ALGO_RING, window=1 << 30, sync_overhead_us=0.0)
        bi, bo = SymmetricBuffer(comm, S), SymmetricBuffer(comm, S)
        g = torch.Generator(device="cuda").manual_seed(0x4E5A0000 + r)
        x = torch.rand(S // 4, device="cuda", generator=g) * 2 - 1
        bi.write(x.data_ptr(), S)
        stream = torch.cuda.Stream()
        torch.cuda.synchronize()
        for i in range(len(kinds)):
            eng.loop_timing(i, True)
        for _ in range(warm):
            eng.allreduce(bi, bo, S, F32, stream)
        eng.synchronize()
        plan = eng.last_plans()[0]["segs"]
        # ~0.4 s of the same load so the clock sampler sees the GPU busy.
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            eng.allreduce(bi, bo, S, F32, stream)
        e1.record(stream)
        e1.synchronize()
        t_est = max(max(json.loads(v_.decode()) for v_ in comm.allgather_bytes(
            json.dumps(e0.elapsed_time(e1) / 3e3).encode().ljust(32))), 1e-5)
        soak = min(4000, int(0.4 / t_est))  # the same count on every rank (collective)
        comm.barrier()
        if r == 0:
            clk.__enter__()
        comm.barrier()
        for _ in range(soak):
            eng.allreduce(bi, bo, S, F32, stream)
        eng.synchronize()
        for i in range(len(kinds)):
            eng.loop_time(i)  # reset the per-launch kernel timers
        comm.barrier()
        if r == 0:
            shared["launches0"] = kernel_launch_count()
        comm.barrier()
        e0.record(stream)
        for _ in range(steps):
            eng.allreduce(bi, bo, S, F32, stream)
        e1.record(stream)
        e1.synchronize()
        comm.barrier()
        if r == 0:
            shared["launches"] = kernel_launch_count() - shared["launches0"]
            clk.__exit__()
        eng.synchronize()
        t_step = e0.elapsed_time(e1) / 1e3 / steps
        comm.barrier()  # every rank's grids are in; one reader of the shared per-grid timers
        ktime = {kinds[i]: eng.loop_time(i) for i in range(len(kinds))} if r == 0 else None
        comm.barrier()
        for i in range(len(kinds)):
            eng.loop_timing(i, False)

        # e2e through the public host API: H2D of this rank's input, the
        # multi-rail allreduce, D2H of the result, every step.
        hin = torch.empty(S, dtype=torch.uint8).pin_memory()
        hout = torch.empty(S, dtype=torch.uint8).pin_memory()
        hin.copy_(x.view(torch.uint8).cpu())
        for _ in range(2):
            eng.allreduce_host(hin, hout, S, F32)
        ke = max(3, min(steps, 10))
        comm.barrier()
        bar.wait()
        t0 = time.perf_counter()
        for _ in range(ke):
            eng.allreduce_host(hin, hout, S, F32)
        bar.wait()
        te = (time.perf_counter() - t0) / ke
        eng.close()
        bi.free()
        bo.free()

        # Config 4 shape (bf16 256 MiB, RingChunked): the larger rail's link
        # dies on the last rank mid-op, unplanned; every rank detects it,
        # agrees on the orphan and reroutes it to the other rail.
        fo = None
        if not args.no_failover:
            try:
                fo = loop_failover(comm, g, stream)
            except Exception as e:  # reported, never fatal to the headline line
                fo = {"error": str(e)[:300]}
        return {"t_step": t_step, "ktime": ktime, "te": te, "plan": plan, "fo": fo}

    def loop_failover(comm, g, stream):
        eng2 = Engine(comm, kinds=kinds, rails_toml=toml, algorithm=ALGO_RING_CHUNKED, window=1 << 30,
                      sync_overhead_us=0.0)
        b2i, b2o = SymmetricBuffer(comm, fo_bytes), SymmetricBuffer(comm, fo_bytes)
        try:
            mon = eng2.state()["monitor"]  # the same on every rank (agreed at engine creation)
            if not mon["on"]:
                return {"error": "failure monitor off: " + mon.get("off_reason", "")}
            xb = (torch.rand(fo_bytes // 2, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
            b2i.write(xb.data_ptr(), fo_bytes)
            torch.cuda.synchronize()
            eng2.allreduce(b2i, b2o, fo_bytes, BF16, stream)
            eng2.synchronize()
            segs = eng2.last_plans()[0]["segs"]
            victim = max(segs, key=lambda s_: s_[2])
            nch = -(-victim[2] // victim[3])
            if comm.rank == V - 1:
                eng2.inject_failure(eng2.op_seq, victim[0], nch // 2)
            comm.barrier()
            eng2.allreduce(b2i, b2o, fo_bytes, BF16, stream)
            eng2.synchronize()
            fos = eng2.failovers()
            return fos[-1] if fos else None
        finally:
            eng2.close()
            b2i.free()
            b2o.free()

    res = run_ranks(V, body, timeout=1800)
    t_step = max(r_["t_step"] for r_ in res)
    busbw = ring_volume(V, S) / t_step / 1e9
    algbw = S / t_step / 1e9
    plan = res[0]["plan"]
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6538.3)
    # Dominant kernel: the SM rail's two-shot fold grid over the 8 virtual
    # ranks (fold_kernel_vr<F32,8,8>), timed by CUDA events on the stream it
    # runs on, every launch of the timed region.
    seg = {kinds[s_[0]]: s_[2] for s_ in plan}
    kt = res[0]["ktime"]["sm"]
    roofline = None
    if kt["launches"]:
        t_launch = kt["total_us"] / kt["launches"] * 1e-6
        per_launch = cfg1_hbm_bytes(V, seg.get("sm", 0), "sm")
        ach = per_launch / t_launch / 1e9
        roofline = {"bound": "hbm", "kernel": "fold_kernel_vr<F32,8,8> (SM rail two-shot, 8 virtual ranks)",
                    "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                    "traffic": ncu_traffic("fold_kernel_vr", per_launch), "per_launch_bytes": per_launch,
                    "launches": kt["launches"], "us_per_launch": round(t_launch * 1e6, 2),
                    "note": "achieved = algorithmic HBM bytes of one launch (every virtual rank reads its shard of the "
                            "32 MiB segment from all 8 ranks and writes the sum to all 8: 2*8*32 MiB) / the kernel's "
                            "mean duration (CUDA events around each launch on its stream, timed region); peak = "
                            "MEASURED_PEAKS.json hbm_gbs" + ("" if "hbm_gbs" in peaks else " (fallback)")}
    kce = res[0]["ktime"]["ce"]
    te = max(r_["te"] for r_ in res)
    clocks = clk.summary()
    out = {"metric": METRIC, "value": round(busbw, 2), "unit": "GB/s", "n_gpus": 1, "steps": steps,
           "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": f"config 1: {V} ranks as virtual ranks on one B200 (nz_comm_init_loopback), rails "
                                  f"sm + ce with identical profiles (static 50/50), Ring, {S >> 20} MiB fp32 per rank, "
                                  f"engine allreduce; value = busbw = ringVolume({V}, S) / t",
                      "bytes_per_rank": S, "ranks": V, "virtual_ranks": True, "same_config": True,
                      "l2": f"{V} x {S >> 20} MiB per buffer > 126 MB L2; no flush", "plan": plan,
                      "algbw_GBs": round(algbw, 2),
                      "parity": "bit-exact vs the reference ring golden hash: tests/test_gpu_vranks.py::"
                                "test_loopback_config1_hash (same engine call, oracle inputs)"},
           "roofline": roofline, "gpu_launches": res and shared.get("launches"), "clocks": clocks,
           "e2e": {"value": round(ring_volume(V, S) / te / 1e9, 3), "unit": "GB/s",
                   "h2d_bytes_per_step": V * S, "d2h_bytes_per_step": V * S, "ms_per_step": round(te * 1e3, 3),
                   "note": "nz_engine_allreduce_host on every virtual rank from pinned host memory (H2D, allreduce, "
                           "D2H each step), wall clock between thread barriers"},
           "kernels": {k: {"launches": v["launches"], "us_per_launch": round(v["total_us"] / max(1, v["launches"]), 2)}
                       for k, v in res[0]["ktime"].items()}}
    if kce["launches"]:
        t_ce = kce["total_us"] / kce["launches"] * 1e-6
        out["kernels"]["ce"]["note"] = "copy-engine rail barrier grids (its DMA and reduce run on rank streams)"
        del t_ce
    errs = [r_["fo"]["error"] for r_ in res if r_["fo"] and "error" in r_["fo"]]
    fos = [r_["fo"] for r_ in res if r_["fo"] and "error" not in r_["fo"]]
    if errs:
        out["failover_error"] = errs[0]
    if fos:
        out["failover"] = {"payload": "bf16 256 MiB, RingChunked, larger rail's link dies on the last rank at its "
                                      "middle chunk (unplanned)",
                           "failed_rail": kinds[fos[0]["failed_rail"]], "target_rail": kinds[fos[0]["target_rail"]],
                           "orphan_bytes": fos[0]["orphan_length"], "orphan_chunk": fos[0]["orphan_chunk"],
                           "detect_us_max": round(max(f["detect_us"] for f in fos), 2),
                           "resume_after_detect_us_max": round(max(f["resume_after_detect_us"] for f in fos), 2),
                           "done_us_max": round(max(f["done_us"] for f in fos), 2)}
        out["failover_ms"] = round(max(f["done_us"] for f in fos) / 1e3, 4)
    if not args.no_cpu:
        cb = cpu_baseline(V, S)
        if cb:
            out["cpu_baseline"] = cb
    print(json.dumps(out))
    return 0


# ------------------------------------------------------ N > 1: real GPUs ----
def multirail_ab(comm, bin_, bout, dt, cap, max_over_ranks):
    from paper_2405_17870_b200 import Rail
    from paper_2405_17870_b200._lib import RAIL_KINDS

    world = comm.world
    base = "nvls" if comm.multicast else "sm"
    others = [k for k in ("sm", "ce") if k != base]
    rails = {k: Rail(comm, RAIL_KINDS[k], 30 + i) for i, k in enumerate([base] + others)}
    rows = []
    try:
        for S_ in [s_ for s_ in (64 << 20, 256 << 20, GiB) if s_ <= cap]:
            iters = 20 if S_ <= (64 << 20) else (10 if S_ <= (256 << 20) else 5)
            row = {"bytes": S_}
            for other in [None] + others:
                for f in ((0.0,) if other is None else (0.1, 0.2, 0.3)):
                    split = (int(S_ * (1 - f)) >> 21) << 21  # 2 MiB multiples
                    parts = [(rails[base], 0, split)] + ([(rails[other], split, S_ - split)] if other else [])

                    def op():
                        for r_, off, ln in parts:
                            chunk = max(65536, ((ln // (2 * world)) + 3) & ~3)  # P10
                            r_.allreduce(bin_, bout, off, ln, chunk, dt)

                    for _ in range(2):
                        op()
                    for r_, _, _ in parts:
                        r_.synchronize()
                    comm.barrier()
                    t0 = time.perf_counter()
                    for _ in range(iters):
                        op()
                    for r_, _, _ in parts:
                        r_.synchronize()
                    t = max_over_ranks((time.perf_counter() - t0) / iters)
                    key = base if other is None else f"{base}+{other}@{f:.1f}"
                    row[key] = round(ring_volume(world, S_) / t / 1e9, 2)
            rows.append(row)
    except Exception as e:  # reported, never fatal to the headline line
        rows.append({"error": str(e)[:300]})
    finally:
        for r_ in rails.values():
            r_.close()
    return {"unit": "busbw GB/s", "base": base, "rows": rows,
            "note": "fixed shares f on the second rail, no planner; wall clock over K concurrent ops"}


def run_multi(args):
    import torch

    from paper_2405_17870_b200 import Comm, Engine, Rail, SymmetricBuffer
    from paper_2405_17870_b200._lib import DTYPES, RAIL_KINDS
    from paper_2405_17870_b200.runtime import kernel_launch_count

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    session = f"bench-{os.environ.get('MASTER_PORT', '0')}-{os.environ.get('TORCHELASTIC_RUN_ID', str(os.getppid()))}"
    comm = Comm(rank, world, local, session)
    dt = DTYPES[args.dtype]
    S = CFG1_BYTES

    def max_over_ranks(x: float) -> float:
        vals = comm.allgather_bytes(json.dumps(x).encode().ljust(32))
        return max(json.loads(v.decode().strip()) for v in vals)

    # Headline: config 1's shape at N ranks (static 50/50, Ring, 64 MiB fp32).
    kinds1 = ["nvls", "ce"] if comm.multicast else ["sm", "ce"]
    eng1 = Engine(comm, kinds=kinds1, rails_toml=identical_rails_toml(kinds1), algorithm=ALGO_RING,
                  window=1 << 30, sync_overhead_us=0.0)
    cap = max(S, args.sweep_max if not args.no_sweep else 0, 8192, 256 << 20)
    bin_, bout = SymmetricBuffer(comm, cap), SymmetricBuffer(comm, cap)
    g = torch.Generator(device="cuda").manual_seed(0x4E5A0000 + rank)
    x = torch.rand(cap // 4, device="cuda", generator=g) * 2 - 1
    bin_.write(x.data_ptr(), cap)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 3)):
        eng1.allreduce(bin_, bout, S, 0, stream)
    eng1.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        eng1.allreduce(bin_, bout, S, 0, stream)
    e1.record(stream)
    e1.synchronize()
    # The soak is a collective: every rank takes the count from the slowest rank's estimate.
    soak = max(1, min(4000, int(0.4 / max(1e-6, max_over_ranks(e0.elapsed_time(e1) / 3e3)))))
    comm.barrier()
    with ClockSampler(local) as clk:
        for _ in range(soak):  # same count on every rank (collective)
            eng1.allreduce(bin_, bout, S, 0, stream)
        eng1.synchronize()
        eng1.stats_reset()
        comm.barrier()
        torch.cuda.synchronize()
        launches0 = kernel_launch_count()
        e0.record(stream)
        for _ in range(args.steps):
            eng1.allreduce(bin_, bout, S, 0, stream)
        e1.record(stream)
        e1.synchronize()
    launches = kernel_launch_count() - launches0
    eng1.synchronize()
    t_step = max_over_ranks(e0.elapsed_time(e1) / 1e3 / args.steps)
    busbw = ring_volume(world, S) / t_step / 1e9
    plan1 = eng1.last_plans()[0]["segs"]
    # Dominant rail: largest segment; its per-op time on its own stream (Timer).
    dom = max(plan1, key=lambda s_: s_[2])
    st = eng1.rail_stats(dom[0])
    roofline = None
    if st["ops"]:
        t_rail = max_over_ranks(st["total_us"] / st["ops"] * 1e-6)
        rv = ring_volume(world, dom[2])
        ach = rv / t_rail / 1e9
        wire = (world + 1) * dom[2] // world if kinds1[dom[0]] == "nvls" else rv
        roofline = {"bound": "nvlink", "kernel": f"{kinds1[dom[0]]} rail", "achieved": round(ach, 1),
                    "peak": NVLINK_GBS, "unit": "GB/s", "frac": round(ach / NVLINK_GBS, 4), "traffic": None,
                    "per_launch_bytes": rv, "op_busbw_frac": round(busbw / NVLINK_GBS, 4),
                    "wire": {"bytes_per_op": wire, "GBs": round(wire / t_rail / 1e9, 1), "peak": NVLINK_COPY_GBS,
                             "frac": round(wire / t_rail / 1e9 / NVLINK_COPY_GBS, 4)},
                    "note": "achieved = ringVolume(N, segment) / the rail's time per op (CUDA events on the rail "
                            "stream), peak = NVLink 900 GB/s per direction (BASELINE.md); wire = bytes one GPU "
                            "actually sends (NVLS (N+1)/N*S) against the 770 GB/s measured peer copy"}
    out = {"metric": METRIC, "value": round(busbw, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": f"config 1 shape at {world} GPUs: rails {'+'.join(kinds1)} with identical "
                                  f"profiles (static 50/50), Ring, {S >> 20} MiB fp32 per rank; value = busbw",
                      "bytes_per_rank": S, "ranks": world, "same_config": True, "plan": plan1,
                      "l2": "inputs 64 MiB per rank x 2 buffers; each step rewrites the output (no flush)",
                      "algbw_GBs": round(S / t_step / 1e9, 2)},
           "roofline": roofline, "gpu_launches": launches, "clocks": clk.summary()}

    # e2e through the public host API (H2D + allreduce + D2H every step).
    if not args.no_e2e:
        hin = torch.empty(S, dtype=torch.uint8).pin_memory()
        hout = torch.empty(S, dtype=torch.uint8).pin_memory()
        hin.copy_(x.view(torch.uint8)[:S].cpu())
        for _ in range(2):
            eng1.allreduce_host(hin, hout, S, 0)
        k = max(3, min(args.steps, 10))
        comm.barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            eng1.allreduce_host(hin, hout, S, 0)
        te = max_over_ranks((time.perf_counter() - t0) / k)
        out["e2e"] = {"value": round(ring_volume(world, S) / te / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": S,
                      "d2h_bytes_per_step": S, "ms_per_step": round(te * 1e3, 3),
                      "note": "nz_engine_allreduce_host from pinned host memory, wall clock, max over ranks"}
    eng1.close()

    # Secondary: the state-machine engine over every rail, calibrated at startup.
    kinds = [k for k in args.rails.split(",") if k != "nvls" or comm.multicast] or ["sm"]
    eng = Engine(comm, kinds=kinds, window=5, eta=0.2, demote_after=1, calibrate_max_bytes=min(GiB, cap),
                 tune_budgets=1 if args.tune else 0)

    def timed(nbytes, iters, warm):
        for _ in range(warm):
            eng.allreduce(bin_, bout, nbytes, dt, stream)
        eng.synchronize()
        comm.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(iters):
            eng.allreduce(bin_, bout, nbytes, dt, stream)
        b.record(stream)
        b.synchronize()
        eng.synchronize()
        return max_over_ranks(a.elapsed_time(b) / 1e3 / iters)

    for _ in range(args.tune_ops):
        eng.allreduce(bin_, bout, min(GiB, cap), dt, stream)
    eng.synchronize()

    pg = None
    if not args.no_nccl:
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

    def nccl_time(nbytes, iters):
        t = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
        for _ in range(5):
            pg.all_reduce(t)
        torch.cuda.synchronize()
        pg.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            pg.all_reduce(t)
        b.record()
        b.synchronize()
        return max_over_ranks(a.elapsed_time(b) / 1e3 / iters)

    if pg is not None:
        out["nccl_busbw_GBs"] = round(ring_volume(world, S) / nccl_time(S, 20) / 1e9, 2)

    if not args.no_sweep:
        sweep = []
        s = 4096
        while s <= min(args.sweep_max, cap):
            it = 200 if s <= (1 << 20) else (40 if s <= (64 << 20) else 8)
            t = timed(s, it, warm=20 if s <= (64 << 20) else 12)
            row = {"bytes": s, "us": round(t * 1e6, 2), "busbw_GBs": round(ring_volume(world, s) / t / 1e9, 2),
                   "hot": bool(eng.last_plans()[0]["hot"]) if eng.last_plans() else None,
                   "rails": sorted({seg[0] for p in eng.last_plans() for seg in p["segs"]})}
            if pg is not None:
                tn = nccl_time(s, it)
                row["nccl_busbw_GBs"] = round(ring_volume(world, s) / tn / 1e9, 2)
                row["nccl_us"] = round(tn * 1e6, 2)
            sweep.append(row)
            s *= 2
        out["sweep"] = sweep

    # 8 KiB p50 latency over >= 10,000 ops, the SAME sync pattern for every
    # contender: issue, then torch.cuda.synchronize() (device-wide, so it
    # covers the rail's own stream too), from an agreed start instant.
    def p50_host(fn, n):
        import struct
        lat = []
        for _ in range(n):
            prop = time.perf_counter() + 1e-3
            start = max(struct.unpack("d", b_)[0] for b_ in comm.allgather_bytes(struct.pack("d", prop)))
            while time.perf_counter() < start:
                pass
            fn()
            torch.cuda.synchronize()
            lat.append(time.perf_counter() - start)
        mine = struct.pack(f"{n}d", *lat)
        per_op = sorted(max(v) for v in zip(*[struct.unpack(f"{n}d", b_) for b_ in comm.allgather_bytes(mine)]))
        return {"p50_us": round(per_op[len(per_op) // 2] * 1e6, 2), "p99_us": round(per_op[int(len(per_op) * 0.99)] * 1e6, 2)}

    n_lat = args.latency_ops
    lat = {"ops": n_lat, "engine": p50_host(lambda: eng.allreduce(bin_, bout, 8192, dt, stream), n_lat)}
    for k in ("nvls", "ce", "sm"):
        if k == "nvls" and not comm.multicast:
            continue
        r_ = Rail(comm, RAIL_KINDS[k], 10 + len(lat))
        lat[f"{k}_alone"] = p50_host(lambda: r_.allreduce(bin_, bout, 0, 8192, 65536, dt), n_lat)
        r_.close()
    if pg is not None:
        t8 = torch.empty(2048, dtype=torch.float32, device="cuda")
        lat["nccl"] = p50_host(lambda: pg.all_reduce(t8), n_lat)
    out["latency_8k"] = lat

    # Multi-rail worth on one NVSwitch: the base rail (NVLS, or
    # SM without multicast) alone against the base plus a FIXED share f of
    # the payload on a second rail, the two rails' launches concurrent on
    # their own streams; wall clock over K ops, max over ranks.
    if not args.no_sweep:
        out["multirail_ab"] = multirail_ab(comm, bin_, bout, dt, cap, max_over_ranks)

    # Failover: config 4 shape (bf16 256 MiB, largest-alpha rail's link dies
    # on the last rank at its middle chunk, unplanned).
    def agreed_error(err):
        """Every rank's outcome of a section; the first error, or None."""
        blobs = comm.allgather_bytes(json.dumps(err).encode()[:480].ljust(512))
        errs = [json.loads(b_.decode().strip() or "null") for b_ in blobs]
        return next((e_ for e_ in errs if e_), None)

    eng_ok = True
    if not args.no_failover and len(kinds) > 1:
        err, fo, victim = None, None, None
        try:
            mon = eng.state()["monitor"]  # the same on every rank
            if not mon["on"]:
                raise RuntimeError("failure monitor off: " + mon.get("off_reason", ""))
            fs = 256 << 20
            eng.allreduce(bin_, bout, fs, DTYPES["bf16"], stream)
            eng.synchronize()
            segs = eng.last_plans()[0]["segs"]
            victim = max(segs, key=lambda s_: s_[2])
            nch = -(-victim[2] // victim[3])
            if rank == world - 1:
                eng.inject_failure(eng.op_seq, victim[0], nch // 2)
            comm.barrier()
            eng.allreduce(bin_, bout, fs, DTYPES["bf16"], stream)
            eng.synchronize()
            fo = eng.last_failover()
            if not fo:
                raise RuntimeError("no failover recorded")
        except Exception as e:  # reported, never fatal to the headline line
            err = str(e)[:300]
        # Agreed before any further collective: a rank that raised must not
        # leave its peers inside a collective it skipped.
        err = agreed_error(err)
        if err:
            out["failover_error"] = err
            eng_ok = False  # the engine's collectives may be out of step: no more sections on it
        else:
            out["failover"] = {"failed_rail": kinds[fo["failed_rail"]], "target_rail": kinds[fo["target_rail"]],
                               "orphan_bytes": fo["orphan_length"], "orphan_chunk": fo["orphan_chunk"],
                               "detect_us": round(max_over_ranks(fo["detect_us"]), 2),
                               "resume_after_detect_us": round(max_over_ranks(fo["resume_after_detect_us"]), 2),
                               "done_us": round(max_over_ranks(fo["done_us"]), 2), "payload": "bf16 256 MiB"}
            out["failover_ms"] = round(out["failover"]["done_us"] / 1e3, 4)
            try:
                eng.readmit(victim[0])
                err = None
            except Exception as e:
                err = str(e)[:300]
            err = agreed_error(err)
            if err:
                out["readmit_error"] = err
                eng_ok = False

    # Config 3: mixed 8 KiB - 4 MiB stream through the state machine.
    if not args.no_sweep and eng_ok:
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
        out["config3_mixed_stream"] = {"ops": n_ops, "sizes": "log-uniform 8 KiB-4 MiB, seed 7",
                                       "mean_us_per_op": round(tm / n_ops * 1e6, 2),
                                       "hot_buckets": [e["bucket"] for e in table["buckets"]
                                                       if e["hot"] and 13 <= e["bucket"] <= 22],
                                       "threshold": table["threshold"]}

        # Config 5: DDP gradient-bucket traces (torch 2.11 bucketing, tests/golden).
        traces = json.load(open(os.path.join(ROOT, "tests", "golden", "ddp_buckets.json")))
        c5 = {}
        for name, buckets in traces.items():
            if max(buckets) > cap:
                continue
            for _ in range(3):
                for nb in buckets:
                    eng.allreduce(bin_, bout, nb, dt, stream)
            eng.synchronize()
            comm.barrier()
            a.record(stream)
            for _ in range(5):
                for nb in buckets:
                    eng.allreduce(bin_, bout, nb, dt, stream)
            b.record(stream)
            b.synchronize()
            eng.synchronize()
            t_it = max_over_ranks(a.elapsed_time(b) / 1e3 / 5)
            c5[name] = {"buckets": len(buckets), "bytes": sum(buckets), "ms_per_iter": round(t_it * 1e3, 3)}
        out["config5_ddp_buckets"] = c5

    eng.close()
    bin_.free()
    bout.free()
    comm.close()
    if pg is not None:
        pg.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--virtual-ranks", type=int, default=CFG1_RANKS, help="N = 1: ranks of config 1 on the one GPU")
    ap.add_argument("--rails", default="nvls,ce,sm", help="N > 1 secondary engine rails")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16", "i32"])
    ap.add_argument("--tune-ops", type=int, default=200, help="N > 1: balancer convergence ops before the sweep")
    ap.add_argument("--latency-ops", type=int, default=10000)
    ap.add_argument("--sweep-max", type=int, default=GiB)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-failover", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tune", action="store_true",
                    help="N > 1: the engine measures its CTA budgets and LL crossover at startup (tune_budgets=1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    _, world, _ = env_rank()
    if world == 1:
        return run_loopback(args)
    return run_multi(args)


if __name__ == "__main__":
    sys.exit(main())
