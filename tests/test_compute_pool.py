"""ComputePool (P14): the product
(nz_pool_* through the C ABI) against oracle/compute_pool.py. CPU only."""
import threading
import time

import numpy as np
import pytest

from oracle import compute_pool as ocp
from paper_2405_17870_b200 import NezhaError
from paper_2405_17870_b200.runtime import ComputePool, plan_compute_grants

IO, COMM, COMP = ComputePool.IO, ComputePool.COMMUNICATION, ComputePool.COMPUTATION


def test_spec_examples():
    # total=8, two rails each demanding 8 for computation -> serialized
    p = ComputePool(8)
    p.declare(0, 8)
    p.declare(1, 8)
    assert p.try_acquire(0, COMP) == 8
    assert p.try_acquire(1, COMP) is None
    # io phase -> always immediate grant of 1
    assert p.try_acquire(1, IO) == 1
    p.release(1, IO)
    p.release(0, COMP)
    assert p.try_acquire(1, COMP) == 8
    p.release(1, COMP)
    # three rails, total=6, demand 3 each -> at most two compute concurrently
    q = ComputePool(6)
    for r in range(3):
        q.declare(r, 3)
    assert q.try_acquire(0, COMP) == 3 and q.try_acquire(1, COMP) == 3
    assert q.try_acquire(2, COMP) is None
    assert q.outstanding == 6
    # demand > total_tokens -> capped
    q.declare(5, 100)
    q.release(0, COMP)
    q.release(1, COMP)
    assert q.try_acquire(5, COMP) == 6


def test_contract_violations_raise():
    p = ComputePool(4)
    with pytest.raises(NezhaError):
        p.try_acquire(0, IO)  # undeclared
    p.declare(0, 2)
    p.try_acquire(0, IO)
    with pytest.raises(NezhaError):
        p.try_acquire(0, COMP)  # single grant outstanding per rail
    with pytest.raises(NezhaError):
        p.release(0, COMP)  # not held
    with pytest.raises(NezhaError):
        p.declare(0, 1)  # redeclare while holding
    with pytest.raises(NezhaError):
        ComputePool(0)


def test_blocking_acquire_wakes_fifo():
    p = ComputePool(4)
    for r in range(3):
        p.declare(r, 4 if r != 2 else 1)
    assert p.acquire(0, COMP) == 4
    order = []

    def worker(r):
        g = p.acquire(r, COMP)
        order.append((r, g))
        time.sleep(0.02)
        p.release(r, COMP)

    t1 = threading.Thread(target=worker, args=(1,))
    t1.start()
    while p.waiting < 1:
        time.sleep(0.001)
    t2 = threading.Thread(target=worker, args=(2,))  # fits by size but queues behind rail 1 (FIFO)
    t2.start()
    while p.waiting < 2:
        time.sleep(0.001)
    assert order == []
    p.release(0, COMP)
    t1.join(5)
    t2.join(5)
    assert order == [(1, 4), (2, 1)]
    assert p.outstanding == 0


@pytest.mark.parametrize("seed", range(6))
def test_random_traces_match_oracle(seed):
    rng = np.random.default_rng(seed)
    total = int(rng.integers(1, 20))
    prod, orc = ComputePool(total), ocp.Pool(total)
    rails = list(range(int(rng.integers(1, 5))))
    for r in rails:
        d = int(rng.integers(0, 2 * total))
        prod.declare(r, d)
        orc.declare(r, 1, 1, d)
    for _ in range(400):
        r = int(rng.choice(rails))
        phase = int(rng.integers(0, 3))
        act = rng.integers(0, 3)
        if act == 0:
            d = int(rng.integers(0, 2 * total))
            try:
                orc.declare(r, 1, 1, d)
                want = None
            except ValueError as e:
                want = e
            if want is None:
                prod.declare(r, d)
            else:
                with pytest.raises(NezhaError):
                    prod.declare(r, d)
        elif act == 1:
            try:
                want = orc.try_acquire(r, phase)
            except ValueError:
                with pytest.raises(NezhaError):
                    prod.try_acquire(r, phase)
                continue
            assert prod.try_acquire(r, phase) == want
        else:
            try:
                orc.release(r, phase)
            except ValueError:
                with pytest.raises(NezhaError):
                    prod.release(r, phase)
                continue
            prod.release(r, phase)
        assert prod.outstanding == orc.out <= total


@pytest.mark.parametrize("mode", [ocp.OFF, ocp.BLOCK, ocp.SHRINK])
def test_plan_grants_match_oracle(mode):
    rng = np.random.default_rng(100 + mode)
    for _ in range(300):
        total = int(rng.integers(1, 300))
        n = int(rng.integers(0, 5))
        ids = sorted(rng.choice(8, size=n, replace=False).tolist())
        demands = [(int(r), int(rng.integers(0, 2 * total))) for r in ids]
        assert plan_compute_grants(total, mode, demands) == ocp.plan_grants(total, mode, demands)


def test_plan_grants_b200_defaults():
    # NVLS 32 CTAs, CE fold all 148 SMs, SM rail 64 (rails.cu gridFor defaults).
    d = [(0, 32), (1, 148), (2, 64)]
    blk = plan_compute_grants(148, ocp.BLOCK, d)
    assert [x["waits"] for x in blk] == [[], [0], [1]]
    shr = plan_compute_grants(148, ocp.SHRINK, d)
    assert [x["grant"] for x in shr] == [32, 116, 32] and shr[2]["waits"] == [0]
