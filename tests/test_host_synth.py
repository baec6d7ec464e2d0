"""The product's host generator of the SURVEY.md §8(d) rows (tsom_synth_gmm_host,
host_synth.cpp: every thread jumps the reference's mt19937_64 stream to its
first row) against the reference generator itself (oracle/_ref: Rng(seed,
synth) in sequence) and the oracle's restatement: bit-identical for even and
odd d (odd d carries a cached Box-Muller value across rows) and any thread
count.  CPU only."""
import numpy as np
import pytest

from paper_2604_26555_b200 import _lib


@pytest.mark.parametrize("n,d,seed,n_comp,threads", [
    (1000, 50, 2604, 16, 1), (200_003, 50, 2606, 16, 16), (199_999, 7, 11, 3, 16),
    (150_001, 1, 5, 1, 5), (300_001, 3, 9, 5, 7), (393_221, 51, 1, 16, 3), (0, 50, 1, 16, 4),
])
def test_host_synth_matches_reference_generator(oracle_port, n, d, seed, n_comp, threads):
    import oracle
    got = _lib.synth_gmm_host(n, d, seed, n_comp, threads)
    want = (oracle.ref if oracle.ref.available else oracle_port).synth_gmm(n, d, seed, n_comp)
    assert got.shape == (n, d)
    assert np.array_equal(got.view(np.uint32), np.asarray(want, np.float32).view(np.uint32))


@pytest.mark.parametrize("d", [50, 7])
def test_host_synth_row_slices(oracle_port, d):
    """A rank's slice [row0, row0 + n) equals the same rows of the whole set."""
    whole = _lib.synth_gmm_host(300_000, d, 77, 16, 8)
    for row0, n in [(0, 1000), (123_457, 100_000), (299_999, 1), (150_000, 150_000)]:
        part = _lib.synth_gmm_host(n, d, 77, 16, 8, row0=row0)
        assert np.array_equal(part, whole[row0:row0 + n])


def test_host_synth_rejects_bad_arguments():
    with pytest.raises(_lib.InvalidArgument):
        _lib.synth_gmm_host(10, 0)
