"""Host-side loop pieces of the product vs the oracle (CPU only)."""
import numpy as np
import pytest

import oracle
from paper_2604_26555_b200 import hostref


def test_rng_matches_reference_streams(oracle_port):
    for seed, stream in [(7, 2), (2604, 4), (0, 3)]:
        r = hostref.Rng(seed, stream)
        a = [r.next() for _ in range(700)]
        b, _ = oracle_port.rng_draws(seed, stream, 700)
        assert a == [int(v) for v in b]


def test_mt19937_64_standard_value():
    r = hostref.Rng(5489)
    x = 0
    for _ in range(10000):
        x = r.next()
    assert x == 9981545732273789042


@pytest.mark.parametrize("n,p,seed", [(500, 16, 3), (5000, 100, 2601), (20, 30, 1)])
def test_init_sample_draw_matches_oracle(oracle_port, n, p, seed):
    x = oracle_port.synth_uniform(n, 3, seed)
    w = hostref.init_sample_draw(x, p, seed)
    ref = np.empty((p, 3), np.float32)
    oracle_port.lib.orc_init_sample_draw(x, n, 3, p, seed, ref)
    assert (w == ref).all()


@pytest.mark.parametrize("kind", ["rect", "hex"])
def test_lattice_dist_matches_oracle(oracle_port, kind):
    assert (hostref.lattice_dist(kind, 7, 5) == oracle_port.lattice_dist(kind, 7, 5)).all()


def test_schedule_values(oracle_port):
    for kind in ("linear", "exponential"):
        for t in range(10):
            assert hostref.schedule_value(0.5, kind, t, 10, 1e-4) == \
                oracle_port.schedule_value(0.5, kind, t, 10, 1e-4)
    assert hostref.schedule_value(0.001, "linear", 99, 100, 1e-4) == 1e-4
    assert hostref.resolved_sigma0("hex", 32, 32) == 16.0
    assert hostref.resolved_sigma0("mst", 0, 0) == 3.0


def test_refresh_schedule_matches_reference():
    # test_topology.cpp:351-367: growth 2, warmup 10 -> 0..9, 10, 12, 16, 24
    st = hostref.RefreshState(10, 2.0, 25)
    got = []
    for it in range(30):
        if st.should_refresh(it):
            st.mark(it)
            got.append(it)
    assert got == [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 16, 24]
    assert st.post_warmup_refreshes == 4
    # test_topology.cpp:369-383: saturation at max_interval
    st = hostref.RefreshState(1, 10.0, 5)
    got = []
    for it in range(25):
        if st.should_refresh(it):
            st.mark(it)
            got.append(it)
    assert got == [0, 1, 6, 11, 16, 21]
