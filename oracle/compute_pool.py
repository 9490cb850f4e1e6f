"""ComputePool oracle — TEST INFRASTRUCTURE ONLY (never imported by the product).

Independent restatement of SPEC.md:252-255 (ComputePool type) and :329-337
(acquire_phase_tokens / release_phase_tokens), with the accounting the SPEC
leaves open pinned as DESIGN.md P14:
  * io / communication: grant 1, immediate, not counted against the total;
  * computation: grant min(demand, total), FIFO among waiters, granted when
    nothing waits ahead and outstanding + grant <= total; demand 0 -> 0;
  * one grant outstanding per rail; violations raise ValueError (the
    product's std::invalid_argument / NZ_ERR_INVALID).
Blocking is modelled as an event log: a request that cannot be granted joins
the queue and is granted later, inside the release() that frees room.

plan_grants restates the engine's stream-order arbitration of one op
(include/nezha/compute_pool.hpp planComputeGrants).
"""
from __future__ import annotations

from collections import deque

IO, COMMUNICATION, COMPUTATION = 0, 1, 2


class Pool:
    def __init__(self, total: int):
        if total < 1:
            raise ValueError("total_tokens must be >= 1")
        self.total = total
        self.demand: dict[int, tuple[int, int, int]] = {}
        self.held: dict[int, tuple[int, int]] = {}  # rail -> (phase, grant)
        self.out = 0
        self.peak = 0
        self.queue: deque[tuple[int, int]] = deque()  # (rail, grant) of blocked computation requests

    def _grant_for(self, rail: int, phase: int) -> int:
        if rail not in self.demand:
            raise ValueError(f"rail {rail} not declared")
        if phase not in (IO, COMMUNICATION, COMPUTATION):
            raise ValueError("bad phase")
        return 1 if phase != COMPUTATION else min(self.demand[rail][2], self.total)

    def declare(self, rail: int, io: int, comm: int, comp: int) -> None:
        if min(io, comm, comp) < 0:
            raise ValueError("negative demand")
        if rail in self.held or any(r == rail for r, _ in self.queue):
            raise ValueError("redeclare while holding")
        self.demand[rail] = (io, comm, comp)

    def _take(self, rail: int, phase: int, g: int) -> None:
        self.held[rail] = (phase, g)
        if phase == COMPUTATION:
            self.out += g
            self.peak = max(self.peak, self.out)

    def try_acquire(self, rail: int, phase: int) -> int | None:
        g = self._grant_for(rail, phase)
        if rail in self.held:
            raise ValueError("already holds a grant")
        if phase == COMPUTATION and g > 0 and (self.queue or self.out + g > self.total):
            return None
        self._take(rail, phase, g)
        return g

    def acquire(self, rail: int, phase: int) -> int | None:
        """Blocking acquire as an event: the grant, or None when the rail now waits."""
        g = self._grant_for(rail, phase)
        if rail in self.held or any(r == rail for r, _ in self.queue):
            raise ValueError("already holds a grant")
        if phase == COMPUTATION and g > 0 and (self.queue or self.out + g > self.total):
            self.queue.append((rail, g))
            return None
        self._take(rail, phase, g)
        return g

    def release(self, rail: int, phase: int) -> list[tuple[int, int]]:
        """Phase exit; returns the blocked requests granted as a consequence, in order."""
        if rail not in self.held or self.held[rail][0] != phase:
            raise ValueError("does not hold that grant")
        _, g = self.held.pop(rail)
        if phase == COMPUTATION:
            self.out -= g
        woke = []
        while self.queue and self.out + self.queue[0][1] <= self.total:
            r, g2 = self.queue.popleft()
            self._take(r, COMPUTATION, g2)
            woke.append((r, g2))
        return woke


OFF, BLOCK, SHRINK = 0, 1, 2


def plan_grants(total: int, mode: int, demands: list[tuple[int, int]]) -> list[dict]:
    """Per rail in order: {"rail", "demand", "grant", "waits"} (rails whose
    computation-phase exit it waits for). Stream-order rule: a request that
    does not fit waits for the oldest holders, one at a time, until it fits."""
    res = []
    holders: deque[tuple[int, int]] = deque()
    free = total
    for rail, demand in demands:
        waits: list[int] = []
        if mode == OFF:
            res.append({"rail": rail, "demand": demand, "grant": demand, "waits": waits})
            continue
        want = min(demand, total)
        if mode == SHRINK and want > 0:
            while free <= 0:
                r, g = holders.popleft()
                free += g
                waits.append(r)
            want = min(want, free)
        while want > free:
            r, g = holders.popleft()
            free += g
            waits.append(r)
        free -= want
        if want > 0:
            holders.append((rail, want))
        res.append({"rail": rail, "demand": demand, "grant": want, "waits": waits})
    return res
