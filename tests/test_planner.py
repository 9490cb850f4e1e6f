"""Planner parity: the product's balancer + faults decisions (C++, reached
through nz_planner_run_trace in libnezha_b200.so) must equal the oracle's
independent restatement (oracle/planner.py) byte for byte on the same
injected per-rail latency / failure traces; plus the SPEC's known answers.
CPU only."""
import math

import pytest

from oracle import planner as P

lib_missing = False
try:
    from paper_2405_17870_b200 import run_trace
    from paper_2405_17870_b200 import lib as _lib

    _lib()
except Exception:  # pragma: no cover
    lib_missing = True

needs_lib = pytest.mark.skipif(lib_missing, reason="libnezha_b200.so not built")


# ------------------------------------------------------------ SPEC known answers
def test_cold_latency_example():
    # (10 us, 10 GB/s) and (1000 us, 12.5 GB/s), S = 1e6 -> 110 us on rail 0
    rails = [P.Rail(0, 10, 10e9), P.Rail(1, 1000, 12.5e9)]
    t, best = P.cold(rails, 1_000_000)
    assert best == 0 and t == pytest.approx(110.0)
    # identical rails -> rail 0 by tie-break
    assert P.cold([P.Rail(0, 5, 1e9), P.Rail(1, 5, 1e9)], 4096)[1] == 0


def test_hot_latency_examples():
    # (100 us, 1 GB/s), (300 us, 1 GB/s), alpha (0.75, 0.25), S = 1e6 -> 850 us
    rails = [P.Rail(0, 100, 1e9), P.Rail(1, 300, 1e9)]
    assert P.hot(rails, [0.75, 0.25], 1_000_000, 0.0) == pytest.approx(850.0)
    # unit vector -> that rail + sync
    assert P.hot(rails, [0.0, 1.0], 1_000_000, 7.0) == pytest.approx(300 + 1000 + 7.0)
    # symmetric halves
    sym = [P.Rail(0, 10, 1e9), P.Rail(1, 10, 1e9)]
    assert P.hot(sym, [0.5, 0.5], 2_000_000, 0.0) == pytest.approx(10 + 1000)
    with pytest.raises(ValueError):
        P.hot(rails, [0.7, 0.7], 1000, 0.0)


def test_init_coefficients_examples():
    # SPEC.md:291-293
    assert P.eq8([100.0, 300.0]) == [0.75, 0.25]
    a = P.eq8([1.0, 1.0, 2.0])
    assert a == pytest.approx([3 / 8, 3 / 8, 2 / 8]) and sum(a) == pytest.approx(1.0)
    assert P.eq8([5.0] * 4) == pytest.approx([0.25] * 4)
    with pytest.raises(ValueError):
        P.eq8([1.0, 0.0])


def test_update_coefficients_properties():
    # fixed point, direction, simplex, |a'-a|_1 <= eta
    a, conv = P.eq7([0.5, 0.5], [100.0, 100.0], 0.05, 0.01)
    assert conv and a == [0.5, 0.5]
    a, conv = P.eq7([0.5, 0.5], [120.0, 100.0], 0.05, 0.01)
    assert not conv and a[0] < 0.5 < a[1] and sum(a) == pytest.approx(1.0)
    a3, _ = P.eq7([0.2, 0.3, 0.5], [50.0, 80.0, 200.0], 0.05, 0.01)
    assert sum(abs(x - y) for x, y in zip(a3, [0.2, 0.3, 0.5])) <= 0.05 + 1e-12


def test_convergence_to_equal_finish_time():
    # t_setup 100/300 us, equal B, S = 1 MB -> alpha* = (T2-T1+S/B2)/(S/B1+S/B2)
    rails = [P.Rail(0, 100, 1e9), P.Rail(1, 300, 1e9)]
    S = 1_000_000
    want = (300 - 100 + 1000) / (1000 + 1000)
    a = [0.5, 0.5]
    for _ in range(2000):
        lens = P.split(a, S)
        T = [rails[i].latency(lens[i]) for i in range(2)]
        a, conv = P.eq7(a, T, 0.05, 0.0005)
        if conv:
            break
    assert abs(a[0] - want) <= 0.05


def test_threshold_identical_rails():
    # identical rails with sync T_sync -> threshold = 2 B T_sync
    B, Ts = 1e9, 50.0
    rails = [P.Rail(0, 10, B), P.Rail(1, 10, B)]
    f = lambda S: P.hot(rails, [0.5, 0.5], S, Ts) - P.cold(rails, S)[0]
    thr = P.threshold(f, 4096, 1 << 30)
    assert thr == pytest.approx(2 * B * Ts * 1e-6, rel=1e-3)
    # sync = 0 -> hot wins everywhere probed
    f0 = lambda S: P.hot(rails, [0.5, 0.5], S, 0.0) - P.cold(rails, S)[0]
    assert P.threshold(f0, 4096, 1 << 30) == 4095
    # hot never wins -> +inf
    slow = [P.Rail(0, 1, 1e12), P.Rail(1, 10_000, 1e6)]
    fs = lambda S: P.hot(slow, [0.5, 0.5], S, 0.0) - P.cold(slow, S)[0]
    assert P.threshold(fs, 4096, 1 << 30) is None


def test_rho_gate_examples():
    # identical rails, equal split -> 1
    assert P.rho([P.Rail(0, 5, 1e9), P.Rail(1, 5, 1e9)], [0.5, 0.5], 1 << 20) == 1.0
    # SHARP 0.73 GB/s vs TCP 0.06 GB/s at 32 KB -> ~12.2 > 5
    S = 32 * 1024
    sharp = P.Rail(0, 0.0, 0.73e9)
    tcp = P.Rail(1, 0.0, 0.06e9)
    assert P.rho([sharp, tcp], [0.5, 0.5], S) == pytest.approx(0.73 / 0.06, rel=1e-6)


def test_split_examples():
    # S = 8 MB, alpha (0.5, 0.5) -> two 4 MB segments
    assert P.split([0.5, 0.5], 8 << 20) == [4 << 20, 4 << 20]
    # round4 down, remainder to the last participant
    assert P.split([1 / 3, 1 / 3, 1 / 3], 1000) == [332, 332, 336]
    assert P.split([0.0, 1.0, 0.0], 1000) == [0, 1000, 0]


# ------------------------------------------------------- product vs oracle traces
TWO_HOMOG = """
world 8
config sync_us 20 window 10 max_iters 100
rail 0 tcp 30 1.25e9
rail 1 tcp 30 1.25e9
truth 0 30 1.25e9 0.05
truth 1 30 1.25e9 0.05
truth_sync 20
seed 3
ops 40 8192
ops 60 262144
ops 80 8388608
ops 40 67108864
"""

THREE_HETERO = """
world 8
config sync_us 6 window 20 eta 0.1
rail 0 nvls 12 7.0e11
rail 1 ce 45 5.0e11
rail 2 sm 15 4.5e11
truth 0 14 6.2e11 0.04
truth 1 40 3.8e11 0.04
truth 2 16 3.0e11 0.04
truth_sync 5
seed 7
ops_loguniform 3000 8192 4194304
ops 300 268435456
"""

FAILOVER = """
world 8
config sync_us 6 window 10
rail 0 nvls 12 7.0e11
rail 1 ce 45 5.0e11
rail 2 sm 15 4.5e11 cal 4096:15 65536:16 1048576:18.5 67108864:170 1073741824:2400
truth 0 14 6.2e11 0.02
truth 1 40 3.8e11 0.02
truth 2 16 3.0e11 0.02
seed 11
ops 50 268435456
fail 20 0 7
ops 30 268435456
readmit 70 0
ops 40 1048576
fail 90 2 0
ops 20 4096
"""

GATED = """
world 4
config sync_us 1 window 5
rail 0 sharp 0 0.73e9
rail 1 tcp 0 0.06e9
truth 0 1 0.73e9 0
truth 1 1 0.06e9 0
seed 1
ops 30 32768
ops 30 67108864
fail 40 1 0
fail 45 0 0
ops 10 65536
"""

RING_ALGO = """
world 4
algorithm ring
config sync_us 3 window 8 demote_after 2
rail 0 nvls 10 6e11
rail 1 ce 30 5.5e11
truth 0 10 3e11 0.1
truth 1 30 2.5e11 0.1
seed 5
ops 100 134217728
fail 60 1 0
"""


SHARED_LINKS = """
world 8
config sync_us 4 window 6 demote_after 2
rail 0 nvls 12 8.0e11 cal 4096:12 1048576:14 67108864:95 1073741824:1400
rail 1 ce 40 6.5e11 cal 4096:40 1048576:42 67108864:140 1073741824:1750
concurrent 0 nvls 12 5.0e11 cal 4096:13 1048576:16 33554432:80 536870912:1150
concurrent 1 ce 40 3.0e11 cal 4096:41 1048576:45 33554432:150 536870912:1900
truth 0 13 4.6e11 0.03
truth 1 41 2.8e11 0.03
seed 9
ops 40 1073741824
ops 40 8388608
"""


CASCADE = """
world 4
config sync_us 1 window 3
rail 0 nvls 5 6e11
rail 1 ce 20 5e11
rail 2 sm 6 5e11
truth 0 5 6e11 0.01
truth 1 20 5e11 0.01
truth 2 6 5e11 0.01
seed 21
ops 12 536870912
fail 3 2 1
fail 6 0 5
ops 3 4096
fail 9 1 0
ops 4 1048576
readmit 14 2
ops 4 1048576
"""


# Unplanned failures: one rank's link dies mid-op; the
# orphan starts at the last wave boundary every rank completed, the ops the
# issuing thread planned before the agreement landed (lag) lose the rail at
# entry and are rerouted whole, the planner drops the rail at the agreed op.
UNPLANNED = """
world 8
config sync_us 6 window 10
rail 0 nvls 12 7.0e11
rail 1 ce 45 5.0e11
rail 2 sm 15 4.5e11
truth 0 14 6.2e11 0.02
truth 1 40 3.8e11 0.02
truth 2 16 3.0e11 0.02
seed 11
wave_bytes 33554432
ops 40 1073741824
stall 20 0 11 3
ops 30 268435456
readmit 60 0
ops 20 268435456
stall 80 2 0 0
stall 85 2 3 1
ops 10 4096
"""


@needs_lib
@pytest.mark.parametrize("name,scenario", [("two_homog", TWO_HOMOG), ("three_hetero", THREE_HETERO),
                                           ("failover", FAILOVER), ("gated", GATED), ("ring", RING_ALGO),
                                           ("shared_links", SHARED_LINKS), ("cascade", CASCADE),
                                           ("unplanned", UNPLANNED)])
def test_trace_parity_byte_exact(name, scenario):
    got = run_trace(scenario)
    want = P.run(scenario)
    g, w = got.splitlines(), want.splitlines()
    for i, (a, b) in enumerate(zip(g, w)):
        assert a == b, f"{name}: first difference at line {i}:\nproduct: {a}\noracle:  {b}"
    assert len(g) == len(w)


@needs_lib
def test_trace_behaviour_three_rails():
    """Config 3 shape: cold for small payloads, hot (split) for large ones, flushes happen."""
    import json

    lines = [json.loads(l) for l in run_trace(THREE_HETERO).splitlines()]
    ops = [l for l in lines if "op" in l and "segs" in l]
    small = [o for o in ops if o["S"] < 64 * 1024]
    big = [o for o in ops if o["S"] >= 256 << 20]
    assert all(len(o["segs"]) == 1 for o in small)
    assert all(len(o["segs"]) == 3 for o in big)
    assert any("flush" in l for l in lines)


@needs_lib
def test_trace_unplanned_failure():
    """Orphan = last wave boundary at or before the dead chunk; lagged ops lose
    the rail whole; the planner drops it at op + 1 + lag; P9 target."""
    import json

    lines = [json.loads(l) for l in run_trace(UNPLANNED).splitlines()]
    st = [l for l in lines if l.get("stall", {}).get("op") == 20][0]
    assert st["fired"] and st["activation"] == 24
    op20 = [l for l in lines if l.get("op") == 20 and "segs" in l][0]
    seg0 = [s_ for s_ in op20["segs"] if s_[0] == 0][0]
    C = P.chunk_bytes(seg0[2], 8)
    waves = P.wave_ranges(C, 0, -(-seg0[2] // C), 32 << 20)
    k = [w[0] for w in waves if w[0] <= 11 < w[1]][0]
    assert st["orphan_chunk"] == k and st["ticket"]["offset"] == seg0[1] + k * C
    lost = [l for l in lines if "lost" in l]
    assert [l["lost"]["op"] for l in lost if l["lost"]["rail"] == 0] == [21, 22, 23]
    assert all(l["ticket"]["offset"] == [s_ for s_ in p["segs"] if s_[0] == 0][0][1]
               for l in lost if l["lost"]["rail"] == 0
               for p in [x for x in lines if x.get("op") == l["lost"]["op"] and "segs" in x])
    assert any(l.get("dropped") == 0 and l["op"] == 24 for l in lines)
    for l in lines:
        if "segs" in l and 24 <= l["op"] < 60:
            assert all(s_[0] != 0 for s_ in l["segs"])


@needs_lib
def test_trace_failover_tickets():
    import json

    lines = [json.loads(l) for l in run_trace(FAILOVER).splitlines()]
    fails = [l for l in lines if "fail" in l]
    first = fails[0]
    assert first["ticket"]["source"] == 0
    # target = surviving rail with the largest data_length in that op (P9)
    op = [l for l in lines if l.get("op") == 20 and "segs" in l][0]
    lens = {s[0]: s[2] for s in op["segs"] if s[0] != 0}
    assert first["ticket"]["target"] == max(sorted(lens), key=lambda r: lens[r])
    seg0 = [s for s in op["segs"] if s[0] == 0][0]
    C = P.chunk_bytes(seg0[2], 8)
    assert first["ticket"]["offset"] == seg0[1] + 7 * C
    assert first["ticket"]["length"] == seg0[2] - 7 * C
    # after the failure rail 0 never appears until readmitted at op 70
    for l in lines:
        if "segs" in l and 20 < l["op"] < 70:
            assert all(s[0] != 0 for s in l["segs"])


@needs_lib
def test_acceptance_balancer_convergence():
    """SPEC.md:537 (acceptance 3): 20 random 2-3 rail profile sets with rho <= 5;
    the table converges to within 5% of the 0.001-grid optimum of T_hot in <= 100
    flushes (one flush per op here: window 1)."""
    import json
    import random

    rnd = random.Random(2405)
    done = 0
    while done < 20:
        R = rnd.choice([2, 3])
        rails = [(rnd.uniform(5, 60), rnd.uniform(1e11, 6e11)) for _ in range(R)]
        S = 256 << 20
        thr = sorted(S / (t + S / b * 1e6) for t, b in rails)
        if thr[-1] / thr[0] > 5:
            continue
        done += 1
        lines = ["world 8", "config sync_us 0 window 1 eta 0.2 eps 0.001 max_iters 100"]
        for i, (t, b) in enumerate(rails):
            lines += [f"rail {i} tcp {t} {b}", f"truth {i} {t} {b} 0"]
        lines += ["seed 1", f"ops 101 {S}"]
        out = [json.loads(l) for l in run_trace("\n".join(lines)).splitlines()]
        final = [l for l in out if "segs" in l][-1]
        T = max(t + n / b * 1e6 for (t, b), (_, _, n) in zip([rails[s[0]] for s in final["segs"]], final["segs"]))
        profs = [P.Rail(i, t, b) for i, (t, b) in enumerate(rails)]
        best = float("inf")
        if R == 2:
            for k in range(1, 1000):
                a = k / 1000
                best = min(best, P.hot(profs, [a, 1 - a], S, 0.0))
        else:
            for k in range(1, 200):
                for m in range(1, 200 - k):
                    a = [k / 200, m / 200, 1 - (k + m) / 200]
                    best = min(best, P.hot(profs, a, S, 0.0))
        assert T <= 1.05 * best, (rails, T, best)


@needs_lib
def test_acceptance_rho_gate():
    """SPEC.md:538 (acceptance 4): throughput ratio > 5 -> single rail; <= 5 -> split."""
    import json

    def plan(bw1):
        sc = "\n".join(["world 4", "config sync_us 0 window 50",
                        "rail 0 tcp 0 5e9", f"rail 1 tcp 0 {bw1}", "truth 0 0 5e9 0", f"truth 1 0 {bw1} 0",
                        "seed 1", "ops 1 67108864"])
        return [json.loads(l) for l in run_trace(sc).splitlines() if '"segs"' in l][0]

    assert len(plan(0.9e9)["segs"]) == 1  # ratio ~5.6 at the model split
    assert len(plan(2.5e9)["segs"]) == 2  # ratio ~2


def test_acceptance_8_cold_start_threshold_shrinks_with_nodes():
    """SPEC.md:541 (acceptance 8): under the SPEC's ring-step model
    (2(N-1) steps of t_setup + (S/N)/B) the Eq. 6 threshold
    strictly decreases when the node count doubles, and below it the plan is
    a single rail, i.e. dual-rail latency = the best single rail's."""
    from paper_2405_17870_b200.runtime import Planner

    def toml(n):
        t_step, b = 5.0, 25e9
        rail = f"t_setup_us = {2 * (n - 1) * t_step}\nbandwidth_bps = {b * n / (2 * (n - 1))}\n"
        return f'[[rail]]\nprotocol = "tcp"\n{rail}[[rail]]\nprotocol = "glex"\n{rail}'

    thr = {}
    for n in (2, 4, 8, 16):
        p = Planner(toml(n), sync_overhead_us=50.0)
        thr[n] = p.table()["threshold"]
        below = p.allocate(max(4096, thr[n] // 2))
        assert len(below["segs"]) == 1 and not below["hot"]
        above = p.allocate(min(1 << 30, thr[n] * 4))
        assert above["hot"] and len(above["segs"]) == 2
        p.close()
    assert thr[2] > thr[4] > thr[8] > thr[16], thr


# ------------------------------------------------------------ randomized parity
def random_scenario(seed):
    """A random planner scenario: 2-8 ranks, Ring or RingChunked, 2-3 rails of
    any protocol with parametric or calibrated profiles, optional concurrent
    profiles, jittered truth, fixed and log-uniform op blocks, failures and
    readmissions at random ops / chunks."""
    import random as _random

    return _gen(_random.Random(seed))


def _gen(R):
    world = R.choice([2, 4, 8])
    lines = [f"world {world}"]
    if R.random() < 0.3:
        lines.append("algorithm ring")
    cfg = f"config sync_us {R.choice([0, 1, 3, 6, 20])} window {R.randint(2, 15)}"
    if R.random() < 0.5: cfg += f" eta {R.choice([0.05, 0.1, 0.2, 0.3])}"
    if R.random() < 0.4: cfg += f" demote_after {R.randint(1, 3)}"
    if R.random() < 0.3: cfg += f" tau {R.choice([2, 5, 10])}"
    lines.append(cfg)
    nr = R.choice([2, 3])
    protos = ["nvls", "ce", "sm", "tcp", "sharp", "glex"]
    for r in range(nr):
        t = R.choice([0, 1, 5, 12, 30, 45, 200])
        b = R.choice([0.06e9, 1e9, 1.25e9, 3e11, 5e11, 7e11])
        l = f"rail {r} {R.choice(protos)} {t} {b:.6g}"
        if R.random() < 0.3:
            base = t + 1
            l += f" cal 4096:{base} 1048576:{base + 2 + R.random() * 5:.3f} 67108864:{base + 100 + R.random() * 50:.3f}"
        lines.append(l)
    if R.random() < 0.3:
        for r in range(nr):
            lines.append(f"concurrent {r} {R.choice(protos)} {R.choice([5, 15, 40])} {R.choice([2e11, 4e11]):.6g}")
    for r in range(nr):
        lines.append(f"truth {r} {R.choice([1, 5, 14, 40])} {R.choice([1e9, 3e11, 6e11]):.6g} {R.choice([0, 0.02, 0.1])}")
    lines.append(f"truth_sync {R.choice([0, 2, 5])}")
    lines.append(f"seed {R.randint(0, 1000)}")
    total = 0
    for _ in range(R.randint(1, 4)):
        n = R.randint(5, 120)
        if R.random() < 0.3:
            lines.append(f"ops_loguniform {n} 8192 {R.choice([1 << 20, 1 << 24, 1 << 30])}")
        else:
            lines.append(f"ops {n} {R.choice([4096, 8192, 65536, 1 << 20, 8 << 20, 64 << 20, 256 << 20, 1 << 30, 3 << 29])}")
        total += n
    fails = []
    for _ in range(R.randint(0, 3)):
        op = R.randint(0, max(0, total - 1)); rail = R.randrange(nr)
        fails.append((op, rail))
        lines.append(f"fail {op} {rail} {R.randint(0, 7)}")
    for op, rail in fails:
        if R.random() < 0.5 and op + 2 < total:
            lines.append(f"readmit {R.randint(op + 1, total - 1)} {rail}")
    if R.random() < 0.4:
        lines.append(f"wave_bytes {R.choice([1 << 20, 8 << 20, 64 << 20])}")
    for _ in range(R.randint(0, 2)):
        op = R.randint(0, max(0, total - 1)); rail = R.randrange(nr)
        lines.append(f"stall {op} {rail} {R.randint(0, 9)} {R.randint(0, 4)}")
        if R.random() < 0.5 and op + 2 < total:
            lines.append(f"readmit {R.randint(op + 1, total - 1)} {rail}")
    return "\n".join(lines) + "\n"



@needs_lib
def test_trace_parity_randomized():
    """200 random scenarios: product and oracle decision logs identical byte for
    byte (or both reject the scenario)."""
    for seed in range(200):
        sc = random_scenario(seed)
        try:
            want, werr = P.run(sc), None
        except Exception as e:  # noqa: BLE001
            want, werr = None, e
        try:
            got, gerr = run_trace(sc), None
        except Exception as e:  # noqa: BLE001
            got, gerr = None, e
        assert (werr is None) == (gerr is None), (seed, werr, gerr, sc)
        assert got == want, (seed, sc)
