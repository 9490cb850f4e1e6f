"""Oracle restatement of the balancer and fault decisions — TEST INFRASTRUCTURE ONLY.

Independent Python restatement of SPEC.md's balancer and
faults modules with the DESIGN.md pins, over the
reference's core cost model (proj/src/core/types.cpp:54-77,
proj/src/core/math.cpp:26-35). It consumes the same scenario text as
nz_planner_run_trace and must print a byte-identical decision log.

Parity pinning: the reference ships no balancer code or tests
(proj/tests/CMakeLists.txt:14-16 commented out), so this restatement is pinned
by the SPEC's own known-answer examples (tests/test_planner_oracle.py, which
checks every example in SPEC.md:264-328 and :395-411 against this file) —
"parity pinned to SPEC examples", not to reference outputs.
"""
from __future__ import annotations

import math

KMIN, KMAX = 0, 40
NO_THRESHOLD = None
PROTO = {"tcp": 0, "sharp": 1, "glex": 2, "custom": 3, "nvls": 1, "ce": 2, "sm": 0}


def fmt(v: float) -> str:
    return "%.17g" % v


class Rail:
    """RailProfile (proj/include/nezha/core/types.hpp:26-44)."""

    def __init__(self, rail_id, t_setup_us, bandwidth_bps, points=()):
        self.rail_id = rail_id
        self.t = float(t_setup_us)
        self.bw = float(bandwidth_bps)
        self.points = [(int(s), float(l)) for s, l in points]

    def latency(self, size: int) -> float:
        """messageLatency (types.cpp:54-77)."""
        pts = self.points
        if not pts:
            return self.t + float(size) / self.bw * 1e6
        if len(pts) == 1 or size <= pts[0][0]:
            return pts[0][1]
        hi = 1
        while hi + 1 < len(pts) and pts[hi][0] < size:
            hi += 1
        x0, y0 = pts[hi - 1]
        x1, y1 = pts[hi]
        frac = (float(size) - float(x0)) / (float(x1) - float(x0))
        return y0 + frac * (y1 - y0)

    def throughput(self, size: int) -> float:
        """realTimeThroughput (math.cpp:26-35)."""
        if size == 0:
            return 0.0
        t = self.latency(size)
        if t <= 0:
            return 0.0
        return float(size) / (t * 1e-6)


def split(alpha, S):
    """P8: round4down shares in rail order, remainder to the last participant."""
    part = [i for i, a in enumerate(alpha) if a > 0]
    if not part:
        raise ValueError("no participant")
    out = [0] * len(alpha)
    used = 0
    for i in part[:-1]:
        n = int(alpha[i] * float(S)) & ~3
        if n > S - used:
            n = (S - used) & ~3
        out[i] = n
        used += n
    out[part[-1]] = S - used
    return out


def rho(rails, alpha, S):
    """Eq. 3 (P3)."""
    lens = split(alpha, S)
    thr = sorted((r.throughput(n) for r, n in zip(rails, lens) if n > 0), reverse=True)
    if len(thr) < 2:
        return 1.0
    if not thr[1] > 0:
        raise ArithmeticError("degenerate profile")
    return thr[0] / thr[1]


def cold(rails, S):
    """Eq. 4: (latency, index), ties to the lowest index."""
    best, t = 0, rails[0].latency(S)
    for i in range(1, len(rails)):
        ti = rails[i].latency(S)
        if ti < t:
            best, t = i, ti
    return t, best


def hot(rails, alpha, S, sync):
    """Eq. 5 over participating rails."""
    if any(a < 0 for a in alpha):
        raise ValueError("off simplex")
    tot = 0.0
    for a in alpha:
        tot += a
    if abs(tot - 1.0) > 1e-9:
        raise ValueError("off simplex")
    worst = 0.0
    for r, n in zip(rails, split(alpha, S)):
        if n > 0:
            worst = max(worst, r.latency(n))
    return worst + sync


def eq8(T):
    """init_coefficients with N = number of rails."""
    if any(not t > 0 for t in T):
        raise ValueError("invalid telemetry")
    R = len(T)
    if R == 1:
        return [1.0]
    tot = 0.0
    for t in T:
        tot += t
    return [(tot - t) / (tot * float(R - 1)) for t in T]


def eq7(alpha, T, eta, eps):
    """update_coefficients (P4). Returns (alpha', converged)."""
    part = [i for i, a in enumerate(alpha) if a > 0]
    if len(part) < 2:
        return list(alpha), True
    m = part[0]
    tmax = tmin = T[m]
    tsum = 0.0
    for i in part:
        if T[i] > tmax:
            tmax, m = T[i], i
        tmin = min(tmin, T[i])
        tsum += T[i]
    if tmax - tmin <= eps * tmax:
        return list(alpha), True
    tbar = tsum / float(len(part))
    step = 0.5 * eta * ((tmax - tbar) / tmax)
    slack = 0.0
    for i in part:
        if i != m:
            slack += tmax - T[i]
    nxt = list(alpha)
    nxt[m] = alpha[m] - step
    for i in part:
        if i != m:
            nxt[i] = alpha[i] + step * ((tmax - T[i]) / slack)
    tot = 0.0
    for i in range(len(nxt)):
        if nxt[i] < 0:
            nxt[i] = 0.0
        tot += nxt[i]
    return [a / tot for a in nxt], False


def threshold(f, lo, hi):
    """Eq. 6 bisection in log2 space (P5)."""
    if f(hi) >= 0:
        return NO_THRESHOLD
    if f(lo) < 0:
        return lo - 1
    a, b = lo, hi
    while b - a > 1:
        m = int(math.floor(math.exp2(0.5 * (math.log2(float(a)) + math.log2(float(b)))) + 0.5))
        m = max(m, a + 1)
        m = min(m, b - 1)
        if f(m) >= 0:
            a = m
        else:
            b = m
    return a


def calibrate(samples):
    """SPEC.md:434-446 calibrate(samples) with DESIGN.md P15's pins: relative
    least squares of t + c*S; kept if t >= 0, c > 0 and every residual <= 10 %,
    else the samples become an interpolation table. Returns
    (t_setup_us, bandwidth_bps, interpolated, max_rel_residual)."""
    pts = sorted(samples)
    if len(pts) < 2 or any(y <= 0 for _, y in pts) or len({x for x, _ in pts}) != len(pts):
        raise ValueError("bad samples")
    # Minimise sum(((t + c x - y) / y)^2): the 2x2 weighted normal equations,
    # w = 1/y^2, accumulated in sample order with the product's operation
    # order so the doubles agree bit for bit.
    a11 = a12 = a22 = b1 = b2 = 0.0
    for x, y in pts:
        x = float(x)
        w = 1.0 / (y * y)
        a11 += w
        a12 += w * x
        a22 += w * x * x
        b1 += w * y
        b2 += w * x * y
    det = a11 * a22 - a12 * a12
    t, c = (-1.0, -1.0) if det <= 0 else ((a22 * b1 - a12 * b2) / det, (a11 * b2 - a12 * b1) / det)
    worst = max(abs(t + c * x - y) / y for x, y in pts)
    if t >= 0 and c > 0 and worst <= 0.10:
        return t, 1e6 / c, False, worst
    if any(pts[i][1] <= pts[i - 1][1] for i in range(1, len(pts))):
        raise ValueError("interpolation table not increasing")
    dx, dy = pts[-1][0] - pts[0][0], pts[-1][1] - pts[0][1]
    return pts[0][1], dx / (dy * 1e-6), True, 0.0


def chunk_bytes(seg_len, world, chunked=True):
    """P10."""
    if not chunked:
        return max(seg_len, 4)
    return max(65536, (seg_len // (2 * world)) & ~3)


class Table:
    """AllocationTable + balancer control worker."""

    def __init__(self, rails, cfg):
        self.rails = sorted(rails, key=lambda r: r.rail_id)
        self.cfg = cfg
        self.ok = [True] * len(self.rails)
        self.b = {}
        self.thr = NO_THRESHOLD
        self.epoch = 0
        self.saved = {}
        self.win = {}  # bucket -> {index: [samples]}
        self.conc = []
        self.pver = 0  # profile version (model alpha cache key)
        self._mcache, self._mkey = {}, None
        self._rebuild()

    @property
    def hot_rails(self):
        """P13: the hot side (Eqs. 3, 5, 6, 8) uses the concurrent profiles when given."""
        return self.conc if self.conc else self.rails

    def set_concurrent(self, rails):
        self.conc = sorted(rails, key=lambda r: r.rail_id)
        self.pver += 1
        self._rebuild()

    # -- helpers
    def idx(self, rail_id):
        for i, r in enumerate(self.rails):
            if r.rail_id == rail_id:
                return i
        raise ValueError(rail_id)

    def healthy(self):
        return [i for i in range(len(self.rails)) if self.ok[i]]

    def restrict(self, a):
        a = list(a) + [0.0] * (len(self.rails) - len(a))
        tot = 0.0
        for i in range(len(a)):
            if not self.ok[i] or a[i] < 0:
                a[i] = 0.0
            tot += a[i]
        if tot > 0:
            return [x / tot for x in a]
        h = sum(self.ok)
        return [1.0 / h if self.ok[i] else 0.0 for i in range(len(a))]

    def model_alpha(self, k):
        """P11: Eq. 8 on the model's uniform-split latencies, then up to
        max_iters Eq. 7 steps on the model's own latencies (cached)."""
        key = (tuple(self.ok), self.pver)
        if key != self._mkey:
            self._mcache, self._mkey = {}, key
        if k in self._mcache:
            return list(self._mcache[k])
        H = self.healthy()
        hp = [self.hot_rails[i] for i in H]
        S = 1 << k
        share = max(S // len(H), 1)
        ah = eq8([r.latency(share) for r in hp])
        if len(hp) > 1:
            for _ in range(self.cfg["max_iters"]):
                lens = split(ah, S)
                t = [hp[j].latency(lens[j]) if lens[j] > 0 else 0.0 for j in range(len(hp))]
                ah, conv = eq7(ah, t, self.cfg["eta"], self.cfg["eps"])
                if conv:
                    break
        a = [0.0] * len(self.rails)
        for j, i in enumerate(H):
            a[i] = ah[j]
        self._mcache[k] = list(a)
        return a

    @staticmethod
    def clamp(S):
        return min(max(S.bit_length() - 1, KMIN), KMAX)

    def f(self, S):
        H = self.healthy()
        hp = [self.hot_rails[i] for i in H]
        a = [self.b[self.clamp(S)]["alpha"][i] for i in H]
        return hot(hp, a, S, self.cfg["sync_us"]) - cold([self.rails[i] for i in H], S)[0]

    def _rebuild(self):
        H = self.healthy()
        if not H:
            self.thr = NO_THRESHOLD
            for e in self.b.values():
                e["hot"] = False
            self.epoch += 1
            return
        before = {k: (e["hot"], e["best"], [x > 0 for x in e["alpha"]]) for k, e in self.b.items()}
        measured = [k for k in sorted(self.b) if self.b[k]["measured"]]
        for k in range(KMIN, KMAX + 1):
            e = self.b.setdefault(k, {"hot": False, "best": 0, "alpha": [], "measured": False, "iters": 0,
                                      "converged": False, "demoted": False})
            if e["measured"]:
                e["alpha"] = self.restrict(e["alpha"])
            elif measured:
                near = measured[0]
                for m in measured:
                    if abs(m - k) < abs(near - k):
                        near = m
                e["alpha"] = self.restrict(self.b[near]["alpha"])
            else:
                e["alpha"] = self.model_alpha(k)
        self.thr = threshold(self.f, self.cfg["probe_lo"], self.cfg["probe_hi"]) if len(H) >= 2 else NO_THRESHOLD
        hp = [self.rails[i] for i in H]
        for k in range(KMIN, KMAX + 1):
            e = self.b[k]
            e["best"] = H[cold(hp, 1 << k)[1]]
            e["hot"] = len(H) >= 2 and not e["demoted"] and self.thr is not None and (1 << k) > self.thr
            part = [x > 0 for x in e["alpha"]]
            old = before.get(k)
            if old is None or old[0] != e["hot"] or old[1] != e["best"] or (e["hot"] and old[2] != part):
                self.win.pop(k, None)
        self.epoch += 1

    # -- SPEC operations
    def allocate(self, S):
        k = self.clamp(S)
        if not self.healthy():
            return None
        e = self.b[k]
        plan = {"bucket": k, "hot": False, "rho": 1.0, "gated": False, "segs": []}
        if e["hot"]:
            H = self.healthy()
            plan["rho"] = rho([self.hot_rails[i] for i in H], [e["alpha"][i] for i in H], S)
            if plan["rho"] > self.cfg["tau"]:
                plan["gated"] = True
            else:
                plan["hot"] = True
                off = 0
                for i, n in enumerate(split(e["alpha"], S)):
                    if n:
                        plan["segs"].append((self.rails[i].rail_id, off, n))
                        off += n
                return plan
        plan["segs"].append((self.rails[e["best"]].rail_id, 0, S))
        return plan

    def record(self, plan, lat):
        """record_latency for each rail of one op; returns the flush or None."""
        if plan["gated"]:
            return None
        w = self.win.setdefault(plan["bucket"], {i: [] for i in range(len(self.rails))})
        full = False
        for rail_id, us in lat:
            s = w[self.idx(rail_id)]
            s.append(us)
            if len(s) >= self.cfg["window"]:
                full = True
        if not full:
            return None
        means = []
        for i in range(len(self.rails)):
            s = w[i]
            if s:
                acc = 0.0
                for x in s:
                    acc += x
                means.append((self.rails[i].rail_id, acc / float(len(s))))
        self.win.pop(plan["bucket"], None)
        self._flush(plan["bucket"], means)
        return means

    def _flush(self, k, means):
        e = self.b[k]
        worst = 0.0
        for _, m in means:
            worst = max(worst, m)
        if e["hot"]:
            T = [0.0] * len(self.rails)
            for rid, m in means:
                T[self.idx(rid)] = m
            if e["iters"] < self.cfg["max_iters"]:
                part = [0.0 if T[i] <= 0 else a for i, a in enumerate(e["alpha"])]
                a, conv = eq7(self.restrict(part), T, self.cfg["eta"], self.cfg["eps"])
                e["alpha"] = self.restrict(a)
                e["converged"] = conv
                e["iters"] += 1
            e["measured"] = True
            if self.cfg["demote_after"] > 0 and e["iters"] >= self.cfg["demote_after"]:
                hp = [self.rails[i] for i in self.healthy()]
                if worst >= cold(hp, 1 << k)[0]:
                    e["demoted"] = True
        self._rebuild()

    def fail(self, rail_id):
        i = self.idx(rail_id)
        if not self.ok[i]:
            return
        self.saved = {k: list(e["alpha"]) for k, e in self.b.items()}
        self.ok[i] = False
        self.win.clear()
        self._rebuild()

    def readmit(self, rail_id):
        i = self.idx(rail_id)
        if self.ok[i]:
            raise ValueError("not failed")
        self.ok[i] = True
        for k, a in self.saved.items():
            if k in self.b and self.b[k]["measured"]:
                self.b[k]["alpha"] = a
        self.saved = {}
        self.win.clear()
        self._rebuild()

    def json(self):
        parts = []
        for k in sorted(self.b):
            e = self.b[k]
            parts.append('{"bucket":%d,"hot":%s,"best":%d,"alpha":[%s],"measured":%s,"iters":%d,"converged":%s,'
                         '"demoted":%s}' % (k, _b(e["hot"]), self.rails[e["best"]].rail_id,
                                            ",".join(fmt(x) for x in e["alpha"]), _b(e["measured"]), e["iters"],
                                            _b(e["converged"]), _b(e["demoted"])))
        healthy = ",".join(str(self.rails[i].rail_id) for i in self.healthy())
        thr = "null" if self.thr is None else str(self.thr)
        return '{"epoch":%d,"threshold":%s,"healthy":[%s],"buckets":[%s]}' % (self.epoch, thr, healthy,
                                                                              ",".join(parts))


def _b(x):
    return "true" if x else "false"


M64 = (1 << 64) - 1


def splitmix(state):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def unit(x):
    return float(x >> 11) * (1.0 / 9007199254740992.0)


def parse(text):
    sc = {"world": 8, "chunked": True, "rails": [], "truth": {}, "truth_sync": 0.0, "seed": 0, "sizes": [],
          "faults": [], "readmits": [], "concurrent": [], "stalls": [], "wave_bytes": 64 << 20,
          "cfg": {"tau": 5.0, "eta": 0.05, "eps": 0.01, "sync_us": 0.0, "window": 100, "max_iters": 100,
                  "demote_after": 0, "probe_lo": 4096, "probe_hi": 1 << 30}}
    keys = {"tau": "tau", "eta": "eta", "eps": "eps", "sync_us": "sync_us", "window": "window",
            "max_iters": "max_iters", "demote_after": "demote_after"}
    for line in text.splitlines():
        line = line.split("#", 1)[0].split()
        if not line:
            continue
        k, a = line[0], line[1:]
        if k == "world":
            sc["world"] = int(a[0])
        elif k == "algorithm":
            sc["chunked"] = a[0] == "ring_chunked"
        elif k == "config":
            for name, val in zip(a[::2], a[1::2]):
                v = float(val)
                sc["cfg"][keys[name]] = int(v) if name in ("window", "max_iters", "demote_after") else v
        elif k in ("rail", "concurrent"):
            # Protocol names of the reference (types.cpp protocolKindFromString) + the B200 aliases.
            if a[1] not in ("tcp", "sharp", "glex", "custom", "nvls", "ce", "sm"):
                raise ValueError(f"unknown protocol kind: {a[1]}")
            pts = []
            if len(a) > 4:
                assert a[4] == "cal"
                for p in a[5:]:
                    s, l = p.split(":")
                    pts.append((int(s), float(l)))
            sc["rails" if k == "rail" else "concurrent"].append(Rail(int(a[0]), float(a[2]), float(a[3]), pts))
        elif k == "truth":
            sc["truth"][int(a[0])] = (float(a[1]), float(a[2]), float(a[3]))
        elif k == "truth_sync":
            sc["truth_sync"] = float(a[0])
        elif k == "seed":
            sc["seed"] = int(a[0])
        elif k == "ops":
            sc["sizes"] += [int(a[1])] * int(a[0])
        elif k == "ops_loguniform":
            n, lo, hi = int(a[0]), int(a[1]), int(a[2])
            st = sc["seed"]
            l0, l1 = math.log2(float(lo)), math.log2(float(hi))
            for _ in range(n):
                st, z = splitmix(st)
                s = int(math.floor(math.exp2(l0 + unit(z) * (l1 - l0)))) & ~3
                sc["sizes"].append(max(s, 4))
        elif k == "fail":
            sc["faults"].append((int(a[0]), int(a[1]), int(a[2])))
        elif k == "readmit":
            sc["readmits"].append((int(a[0]), int(a[1])))
        elif k == "stall":
            sc["stalls"].append((int(a[0]), int(a[1]), int(a[2]), int(a[3])))
        elif k == "wave_bytes":
            sc["wave_bytes"] = int(a[0])
            if sc["wave_bytes"] <= 0:
                raise ValueError("wave_bytes")
        else:
            raise ValueError(k)
    return sc


def truth(sc, op, rail_id, n, multi):
    a, b, jit = sc["truth"][rail_id]
    st = (sc["seed"] ^ ((op * 0x9E3779B97F4A7C15) & M64) ^ (((rail_id + 1) * 0xBF58476D1CE4E5B9) & M64)) & M64
    _, z = splitmix(st)
    u = 2.0 * unit(z) - 1.0
    us = a + float(n) / b * 1e6
    us = us * (1.0 + jit * u)
    if multi:
        us = us + sc["truth_sync"]
    return us


MAX_WAVES = 4  # nezha::kMaxWaves


def wave_ranges(C, cb, ce, wave_bytes):
    """Waves of a rail call over chunks [cb, ce): groups of
    max(ceil(wave_bytes / C), ceil((ce - cb) / MAX_WAVES)) chunks; a last group
    shorter than half a group joins the one before."""
    if ce <= cb or C == 0:
        return []
    per = max(1, -(-max(wave_bytes, 1) // C), -(-(ce - cb) // MAX_WAVES))
    w = [[c0, min(ce, c0 + per)] for c0 in range(cb, ce, per)]
    if len(w) > 1 and (w[-1][1] - w[-1][0]) * 2 < per:
        w[-2][1] = w[-1][1]
        w.pop()
    return w


def completed_before_stall(C, cb, ce, stall, wave_bytes):
    """Chunks complete on every rank when one rank's link dies at `stall`:
    the start of the wave that holds it (ce when none does) — SPEC.md:414's
    minimum over ranks of the chunks each completed, at wave granularity."""
    for c0, c1 in wave_ranges(C, cb, ce, wave_bytes):
        if c0 <= stall < c1:
            return c0
    return ce


def _ticket(plan, op, rid, off, n, C, k, healthy):
    """P9 / P10 ticket JSON (or "null") and whether no survivor existed."""
    if k * C >= n:
        return "null", False
    cands = sorted(r for r in healthy if r != rid)
    if not cands:
        return "null", True
    lens = {r: sum(s[2] for s in plan["segs"] if s[0] == r) for r in cands}
    tgt = cands[0]
    for r in cands:
        if lens[r] > lens[tgt]:
            tgt = r
    return '{"op_seq":%d,"offset":%d,"length":%d,"source":%d,"target":%d}' % (op, off + k * C, n - k * C, rid, tgt), False


def run(text: str) -> str:
    """Decision log for a scenario; must equal nz_planner_run_trace byte for byte."""
    sc = parse(text)
    t = Table(sc["rails"], sc["cfg"])
    if sc["concurrent"]:
        t.set_concurrent(sc["concurrent"])
    healthy = sorted(r.rail_id for r in t.rails)  # not failed by agreement (P9's survivors)
    activations = []  # [op, rail]: the planner drops the rail before planning op
    dead = []  # links dead on some rank: launches on them fail at entry
    out = []
    for op, S in enumerate(sc["sizes"]):
        for (rop, rid) in sc["readmits"]:
            if rop == op:
                if not any(a[1] == rid for a in activations):
                    t.readmit(rid)
                activations = [a for a in activations if a[1] != rid]
                if rid not in healthy:
                    healthy.append(rid)
                healthy = sorted(healthy)
                dead = [r for r in dead if r != rid]
                out.append('{"readmit":%d,"op":%d}' % (rid, op))
        keep = []
        for a in activations:
            if a[0] > op:
                keep.append(a)
                continue
            if t.ok[t.idx(a[1])]:
                t.fail(a[1])
            out.append('{"dropped":%d,"op":%d}' % (a[1], op))
        activations = keep
        plan = t.allocate(S)
        if plan is None:
            out.append('{"op":%d,"S":%d,"unrecoverable":true}' % (op, S))
            continue
        segs = ",".join("[%d,%d,%d]" % s for s in plan["segs"])
        out.append('{"op":%d,"S":%d,"bucket":%d,"hot":%s,"rho":%s,"gated":%s,"segs":[%s]}' % (
            op, S, plan["bucket"], _b(plan["hot"]), fmt(plan["rho"]), _b(plan["gated"]), segs))
        failed = False
        for (fop, rid, k) in sc["faults"]:
            if fop != op:
                continue
            failed = True
            seg = [s for s in plan["segs"] if s[0] == rid]
            ticket, unrec = "null", False
            if seg:
                _, off, n = seg[-1]
                C = chunk_bytes(n, sc["world"], sc["chunked"])
                ticket, unrec = _ticket(plan, op, rid, off, n, C, k, healthy)
            out.append('{"fail":{"op":%d,"rail":%d,"chunk":%d},"ticket":%s%s}' % (
                op, rid, k, ticket, ',"unrecoverable":true' if unrec else ""))
            healthy = [r for r in healthy if r != rid]
            t.fail(rid)
        for (rid, off, n) in plan["segs"]:
            if rid not in dead:
                continue
            failed = True
            C = chunk_bytes(n, sc["world"], sc["chunked"])
            ticket, unrec = _ticket(plan, op, rid, off, n, C, 0, healthy)
            out.append('{"lost":{"op":%d,"rail":%d},"ticket":%s%s}' % (
                op, rid, ticket, ',"unrecoverable":true' if unrec else ""))
        for (sop, rid, k, lag) in sc["stalls"]:
            if sop != op:
                continue
            seg = [s for s in plan["segs"] if s[0] == rid]
            head = '{"stall":{"op":%d,"rail":%d,"chunk":%d}' % (op, rid, k)
            if not seg or rid in dead:
                out.append(head + ',"fired":false}')
                continue
            _, off, n = seg[-1]
            C = chunk_bytes(n, sc["world"], sc["chunked"])
            nch = -(-n // C)
            kk = completed_before_stall(C, 0, nch, k, sc["wave_bytes"])
            if kk >= nch:
                out.append(head + ',"fired":false}')
                continue
            failed = True
            healthy = [r for r in healthy if r != rid]
            dead.append(rid)
            activations.append([op + 1 + lag, rid])
            ticket, unrec = _ticket(plan, op, rid, off, n, C, kk, healthy)
            out.append(head + ',"fired":true,"orphan_chunk":%d,"activation":%d,"ticket":%s%s}' % (
                kk, op + 1 + lag, ticket, ',"unrecoverable":true' if unrec else ""))
        if failed:
            continue
        multi = len(plan["segs"]) > 1
        lat = [(s[0], truth(sc, op, s[0], s[2], multi)) for s in plan["segs"]]
        means = t.record(plan, lat)
        if means is not None:
            e = t.b[plan["bucket"]]
            out.append('{"flush":%d,"op":%d,"means":[%s],"epoch":%d,"threshold":%s,"alpha":[%s],"hot":%s,'
                       '"iters":%d,"converged":%s,"demoted":%s}' % (
                           plan["bucket"], op, ",".join("[%d,%s]" % (r, fmt(m)) for r, m in means), t.epoch,
                           "null" if t.thr is None else str(t.thr), ",".join(fmt(x) for x in e["alpha"]),
                           _b(e["hot"]), e["iters"], _b(e["converged"]), _b(e["demoted"])))
    out.append(t.json())
    return "\n".join(out) + "\n"
