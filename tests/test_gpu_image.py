"""Selections through the split image (K1 kGather: TMA tile::gather4 of the
selected rows from the row-major 3xFP16 image, multicast over the cluster of
the codebook-group CTAs, 128-B-swizzled A operand; diagnostics option 95 = 1,
off by default because it measured slower).

The same selections must give the same results as the per-pass split into
tiles (the default, option 95 = 0) and as the CPU oracle: BMUs and
per-row distances bit-identical, U / H identical (the accumulation is the same
code on the same BMUs) — for sorted, unsorted and repeated selections, for
codebooks that make every row a near-tie (the enumerate pass gathers too), and
for a sampled device-resident run.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


@pytest.fixture(scope="module")
def data(oracle_port):
    x = oracle_port.synth_gmm(50_000, 50, 2608)
    rng = np.random.default_rng(8)
    w = x[rng.choice(len(x), 1024, replace=False)].copy()
    wdup = w.copy()
    wdup[512:] = wdup[:512]  # nodes j and j + 512 identical: every row an exact tie
    return x, w, wdup


def engines(pkg, x, w, infl):
    out = []
    for mode in (1, 0):
        e = pkg.Engine(w.shape[0], w.shape[1])
        e.set_option(95, mode)
        e.bind(x)
        e.set_codebook(w)
        e.set_influence(infl)
        out.append(e)
    return out


@pytest.mark.parametrize("which", ["plain", "duplicates"])
def test_selection_passes_match(pkg, data, oracle_port, which):
    from paper_2604_26555_b200.hostref import lattice_dist
    x, w, wdup = data
    w = w if which == "plain" else wdup
    infl = oracle_port.influence_from_dist(lattice_dist("hex", 32, 32), 5.0)
    a, b = engines(pkg, x, w, infl)
    try:
        rng = np.random.default_rng(3)
        for sel in (np.sort(rng.choice(len(x), 15_000, replace=False)),
                    rng.integers(0, len(x), 9_000),
                    np.arange(len(x) - 1, 100, -3)):
            sel = sel.astype(np.uint32)
            ba, da = a.bmu_bound(sel)
            bb, db = b.bmu_bound(sel)
            assert np.array_equal(ba, bb) and np.array_equal(da, db)
            bo, do = oracle_port.find_bmus(x[sel], w)
            assert np.array_equal(ba, bo), f"{(ba != bo).sum()} BMUs differ from the oracle"
            np.testing.assert_allclose(da, do, rtol=1e-12)
            ua, ha, _ = a.epoch(0.4, sel)
            ub, hb, _ = b.epoch(0.4, sel)
            assert np.array_equal(ua, ub) and np.array_equal(ha, hb)
        if which == "duplicates":
            assert a.last_recheck_count > 0
    finally:
        a.close()
        b.close()


def test_sampled_run_matches(pkg, data):
    from paper_2604_26555_b200.hostref import lattice_dist
    x, w, _ = data
    es = []
    try:
        for mode in (1, 0):
            e = pkg.Engine(1024, 50)
            e.set_option(95, mode)
            e.bind(x)
            e.set_codebook(w)
            e.set_topology_distance(lattice_dist("hex", 32, 32))
            e.sampler_init("adaptive", len(x) // 10, 2608, 1.0, 2.0)
            es.append(e)
        for e in es:
            e.train_epochs([0.5, 0.4, 0.3, 0.2], [8.0, 6.0, 4.0, 2.0], sampled=True)
        assert np.array_equal(es[0].get_codebook(), es[1].get_codebook())
        assert np.array_equal(es[0].sampler_select(), es[1].sampler_select())
    finally:
        for e in es:
            e.close()
