"""Edge cases of the GPU path against the oracle: tiny and ragged shapes, one
node, one feature, features beyond the tensor-core layout (SIMT path), many
codebook groups, empty and single-row selections."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


SHAPES = [  # (rows, nodes, dims)
    (1, 1, 1), (1, 5, 3), (127, 7, 2), (129, 33, 5), (300, 1, 50), (1000, 2, 1),
    (777, 40, 54), (500, 64, 100), (3000, 4096, 8), (257, 300, 17),
]


@pytest.mark.parametrize("n,p,d", SHAPES)
def test_shapes_bmu(pkg, oracle_port, n, p, d):
    rng = np.random.default_rng(n * 7 + p)
    x = rng.standard_normal((n, d)).astype(np.float32) * 2
    w = rng.standard_normal((p, d)).astype(np.float32) * 2
    e = pkg.Engine(p, d)
    e.set_codebook(w)
    b, dist = e.bmu(x)
    bo, do = oracle_port.find_bmus(x, w)
    assert (b == bo).all()
    np.testing.assert_allclose(dist, do, rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("n,p,d", SHAPES)
def test_shapes_accumulators(pkg, oracle_port, n, p, d):
    rng = np.random.default_rng(n * 11 + p)
    x = rng.standard_normal((n, d)).astype(np.float32) * 2
    w = rng.standard_normal((p, d)).astype(np.float32) * 2
    infl = np.exp(-rng.random((p, p)) * 3)
    e = pkg.Engine(p, d)
    e.bind(x)
    e.set_codebook(w)
    e.set_influence(infl)
    sel = np.arange(n, dtype=np.uint32)
    u, h, dist = e.epoch(0.3, sel, want_dist=True)
    uo, ho, _, _, do = oracle_port.run_iteration(x, sel, w, infl, 0.3, 1, 1)
    assert np.max(np.abs(u - uo)) <= 1e-9 * max(np.max(np.abs(uo)), 1e-30)
    np.testing.assert_allclose(h, ho, rtol=1e-9)
    np.testing.assert_allclose(dist, do, rtol=1e-12)
    if n > 2:  # single-row and strided selections
        for s in (np.array([n // 2], np.uint32), np.arange(0, n, 3, dtype=np.uint32)):
            u1, h1, d1 = e.epoch(0.3, s, want_dist=True)
            u2, h2, _, _, d2 = oracle_port.run_iteration(x, s, w, infl, 0.3, 1, 1)
            assert np.max(np.abs(u1 - u2)) <= 1e-9 * max(np.max(np.abs(u2)), 1e-30)
            np.testing.assert_allclose(d1, d2, rtol=1e-12)


def test_epoch_requires_influence(pkg):
    e = pkg.Engine(4, 2)
    e.bind(np.zeros((8, 2), np.float32))
    e.set_codebook(np.zeros((4, 2), np.float32))
    with pytest.raises(ValueError, match="influence not set"):
        e.epoch(0.1)


def test_simt_and_tc_agree_on_many_groups(pkg, oracle_port):
    from paper_2604_26555_b200 import _lib
    x = oracle_port.synth_gmm(5000, 50, 2660)
    w = oracle_port.synth_gmm(2304, 50, 2661)  # 9 groups of 256
    outs = []
    for kern in (1, 2):
        e = pkg.Engine(2304, 50)
        e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kern)
        e.set_codebook(w)
        outs.append(e.bmu(x)[0])
    bo, _ = oracle_port.find_bmus(x, w)
    assert (outs[0] == bo).all() and (outs[1] == bo).all()


@pytest.mark.parametrize("dup_every", [2, 16])
def test_near_tie_passes_and_overflow(pkg, oracle_port, dup_every):
    """More rows than one near-tie pass holds (n > 2^20: the enumerate scratch
    is n / 16 rows, 4 passes): with every node duplicated, every row is an
    exact tie, so the 4 passes fill and the remaining 75 % of the rows take
    the full exact re-scan.  Every BMU must still be the reference's
    (ties to the lowest index, trainer.hpp:293-304), and U / H match."""
    n, p, d = 1_200_000, 64, 50
    x = oracle_port.synth_gmm(n, d, 2730)
    base = x[np.linspace(0, n - 1, p // dup_every).astype(int)]
    w = np.repeat(base, dup_every, axis=0).copy()
    e = pkg.Engine(p, d)
    e.bind(x)
    e.set_codebook(w)
    b, dist = e.bmu_bound(None, want_dist=True)
    assert e.last_recheck_count > n // 2
    bo, do = oracle_port.find_bmus(x, w)
    assert (b == bo).all()
    np.testing.assert_allclose(dist, do, rtol=1e-12)
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 8, 8), 2.0)
    e.set_influence(infl)
    u, h, _ = e.epoch(0.3)
    sel = np.arange(n, dtype=np.uint32)
    uo, ho, _, _, _ = oracle_port.run_iteration(x, sel, w, infl, 0.3, 1, 8)
    assert np.max(np.abs(u - uo)) <= 1e-9 * np.max(np.abs(uo))
    np.testing.assert_allclose(h, ho, rtol=1e-9)
