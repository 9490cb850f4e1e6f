"""calibrate(samples) -> CalibratedProfile (P15):
product (nz_core_calibrate) vs oracle/planner.py, with the SPEC's Table 1
examples. CPU only."""
import numpy as np
import pytest

from oracle.planner import calibrate as oracle_calibrate
from paper_2405_17870_b200 import NezhaError
from paper_2405_17870_b200.runtime import calibrate

KB, MB = 1024, 1 << 20
TABLE1 = {  # SPEC.md:440-441 (Table 1, 4 nodes)
    "sharp": [(1 * KB, 9.0), (8 * MB, 22140.0), (64 * MB, 181484.0)],
    "tcp": [(1 * KB, 982.0), (8 * MB, 37137.0), (64 * MB, 316323.0)],
}


def model(c, x):
    return c["t_setup_us"] + x / c["bandwidth_bps"] * 1e6


@pytest.mark.parametrize("name", sorted(TABLE1))
def test_table1_reproduced_within_10_percent(name):
    c = calibrate(TABLE1[name])
    if not c["interpolated"]:
        for x, y in TABLE1[name]:
            assert abs(model(c, x) - y) <= 0.10 * y
    assert c["max_rel_residual"] <= 0.10


def test_noiseless_linear_recovered_exactly():
    t, b = 12.5, 4.0e11
    c = calibrate([(x, t + x / b * 1e6) for x in (4096, 1 << 20, 1 << 26)])
    assert not c["interpolated"]
    assert c["t_setup_us"] == pytest.approx(t, rel=1e-9)
    assert c["bandwidth_bps"] == pytest.approx(b, rel=1e-9)


def test_inconsistent_samples_fall_back_to_interpolation():
    # Concave samples: the line through them needs a negative t_setup / misses by > 10 %.
    c = calibrate([(1 << 10, 1.0), (1 << 20, 1000.0), (1 << 21, 1001.0), (1 << 30, 1002.0)])
    assert c["interpolated"]


def test_bad_samples_raise():
    for s in ([(4096, 1.0)], [(4096, 1.0), (4096, 2.0)], [(4096, 0.0), (8192, 1.0)]):
        with pytest.raises(NezhaError):
            calibrate(s)


@pytest.mark.parametrize("seed", range(4))
def test_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    for _ in range(200):
        n = int(rng.integers(2, 8))
        xs = sorted({int(4096 * 2 ** rng.uniform(0, 18)) for _ in range(n)})
        if len(xs) < 2:
            continue
        t, b = rng.uniform(0.5, 2000), 10 ** rng.uniform(8, 12)
        ys = [(t + x / b * 1e6) * rng.uniform(0.8, 1.25) for x in xs]
        ys = list(np.maximum.accumulate(ys) + np.arange(len(ys)) * 1e-3)
        got = calibrate(list(zip(xs, ys)))
        want = oracle_calibrate(list(zip(xs, ys)))
        # Same operation order on both sides: bit-identical doubles.
        assert (got["t_setup_us"], got["bandwidth_bps"], got["interpolated"], got["max_rel_residual"]) == want
