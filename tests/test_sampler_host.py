"""Host-side pieces of the device samplers (no GPU): the MT19937-64 jump-ahead
that seeds the device generators, and the reference sampler through the oracle."""
import numpy as np
import pytest


@pytest.mark.parametrize("seed,jump", [(1, 1), (5489, 311), (5489, 312), (2604 + 4, 19937),
                                       (7, 1_000_003), (123456789, 987_654_321)])
def test_mt19937_64_jump_ahead_equals_sequential(seed, jump):
    from paper_2604_26555_b200 import _lib
    assert _lib.mt_selftest(seed, jump) == 0


def test_port_rng_matches_reference_stream(oracle_port, oracle_ref):
    # the device sampler reproduces Rng(seed, SeedStream::sampler) (stream 3)
    a, _ = oracle_port.rng_draws(2607, 3, 2000)
    b, _ = oracle_ref.rng_draws(2607, 3, 2000)
    assert (np.asarray(a) == np.asarray(b)).all()


@pytest.mark.parametrize("kind", ["random", "adaptive"])
def test_reference_sampler_is_sorted_distinct(oracle_ref, kind):
    sels = oracle_ref.sampler_run(kind, 5000, 9, 4, rho=0.2,
                                  dist_by_row=np.random.default_rng(0).random(5000))
    for s in sels:
        assert len(s) == 1000
        assert (np.diff(s.astype(np.int64)) > 0).all()
