"""BMU-ordered residency (TSOM_OPT_ROW_ORDER, csrc/k_order.cu).

After a full pass the engine re-lays its resident rows out in that pass's BMU
order (K1's epilogue then skips column chunks, K2 gathers runs of rows in one
copy).  Row ids never change for the caller: every result must equal the
engine that keeps the bind order —

  * BMUs and per-row distances of full passes and of selections (sorted,
    unsorted, repeated ids) bit-identical, returned in caller order;
  * U / H of an epoch to 1e-12 (only the FP64 grouping of the sums differs),
    and bit-identical in exact mode (TSOM_OPT_DETERMINISTIC);
  * tsom_get_rows returns the caller's rows;
  * whole device-resident runs (lattice, random / adaptive device sampler,
    periodic re-layout) to 1e-6 relative max-norm;
  * and the re-laid-out engine still equals the CPU oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


def rel_maxnorm(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-300))


def make_pair(pkg, x, w, dist, order=2, exact=False, kernel=0):
    from paper_2604_26555_b200 import _lib
    es = []
    for ro in (0, order):
        e = pkg.Engine(w.shape[0], w.shape[1])
        if kernel:
            e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kernel)
        e.set_option(_lib.TSOM_OPT_ROW_ORDER, ro)
        e.set_option(93, 0)  # re-lay out even these 60k rows (default: >= 2^18 rows)
        if exact:
            e.set_option(_lib.TSOM_OPT_DETERMINISTIC, 1)
        e.bind(x)
        e.set_codebook(w)
        e.set_topology_distance(dist)
        es.append(e)
    return es


@pytest.fixture(scope="module")
def data(oracle_port):
    from paper_2604_26555_b200.hostref import lattice_dist
    x = oracle_port.synth_gmm(60_000, 50, 2604)
    rng = np.random.default_rng(5)
    w = x[rng.choice(len(x), 1024, replace=False)].copy()
    return x, w, lattice_dist("hex", 32, 32)


def influence(oracle_port, dist, sigma):
    return oracle_port.influence_from_dist(dist, sigma)


@pytest.mark.parametrize("kernel", [3, 2, 1], ids=["3xFP16", "3xTF32", "SIMT"])
def test_epoch_outputs_match_bind_order(pkg, data, oracle_port, kernel):
    x, w, dist = data
    a, b = make_pair(pkg, x, w, dist, kernel=kernel)
    try:
        infl = influence(oracle_port, dist, 6.0)
        for e in (a, b):
            e.set_influence(infl)
        # pass 1 leaves the BMU order, pass 2 runs on the re-laid-out rows
        for _ in range(2):
            ua, ha, da = a.epoch(0.5, None, want_dist=True)
            ub, hb, db = b.epoch(0.5, None, want_dist=True)
            assert np.array_equal(da, db), "per-row distances differ"
            assert np.max(np.abs(ub - ua)) <= 1e-12 * np.max(np.abs(ua))
            assert np.allclose(hb, ha, rtol=1e-12, atol=0)
        ba, dba = a.bmu_bound(None)
        bb, dbb = b.bmu_bound(None)
        assert np.array_equal(ba, bb) and np.array_equal(dba, dbb)
        assert np.array_equal(b.get_rows(), x), "get_rows must return the caller's rows"
        assert np.array_equal(b.get_rows(1234, 777), x[1234:2011])
        rng = np.random.default_rng(1)
        for sel in (np.sort(rng.choice(len(x), 5000, replace=False)),
                    rng.integers(0, len(x), 7000),          # unsorted, repeats
                    np.arange(len(x))[::-1].copy()):        # every row, reversed
            sel = sel.astype(np.uint32)
            ua, ha, da = a.epoch(0.5, sel, want_dist=True)
            ub, hb, db = b.epoch(0.5, sel, want_dist=True)
            assert np.array_equal(da, db)
            assert np.max(np.abs(ub - ua)) <= 1e-12 * np.max(np.abs(ua))
            assert np.allclose(hb, ha, rtol=1e-12, atol=0)
            assert np.array_equal(a.bmu_bound(sel)[0], b.bmu_bound(sel)[0])
        sa, ca = a.qe()
        sb, cb = b.qe()
        assert ca == cb and abs(sa - sb) <= 1e-12 * sa
        # and against the CPU oracle on the re-laid-out engine
        bo, do = oracle_port.find_bmus(x, w)
        assert np.array_equal(bb, bo)
    finally:
        a.close()
        b.close()


def test_exact_mode_bit_identical(pkg, data, oracle_port):
    x, w, dist = data
    a, b = make_pair(pkg, x, w, dist, exact=True)
    try:
        infl = influence(oracle_port, dist, 4.0)
        for e in (a, b):
            e.set_influence(infl)
        for _ in range(3):
            ua, ha, da = a.epoch(0.3, None, want_dist=True)
            ub, hb, db = b.epoch(0.3, None, want_dist=True)
            assert np.array_equal(ua, ub) and np.array_equal(ha, hb) and np.array_equal(da, db)
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("order", [1, 2, 3])
def test_training_runs_match(pkg, data, order):
    """1 = auto (re-laid out in a call with >= 20 epochs left: here at the
    second of 24), 2 = once, 3 = every 3 full passes."""
    from paper_2604_26555_b200.hostref import resolved_sigma0, schedule_value
    x, w, dist = data
    s0 = resolved_sigma0("hex", 32, 32)
    etas = [schedule_value(0.5, "linear", t % 12, 12, 1e-4) for t in range(24)]
    sigmas = [schedule_value(s0, "linear", t % 12, 12, 0.3) for t in range(24)]
    a, b = make_pair(pkg, x, w, dist, order=order)
    try:
        a.train_epochs(etas, sigmas)
        b.train_epochs(etas, sigmas)
        if order == 1:
            from paper_2604_26555_b200 import _lib
            import ctypes as C
            L = _lib.load()
            L.tsom_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
            L.tsom_debug_read.restype = C.c_int64
            perm = np.empty(len(x), np.uint32)
            assert L.tsom_debug_read(b.h, 11, perm.ctypes.data, perm.nbytes) == perm.nbytes, \
                "auto mode did not re-lay out in a 24-epoch call"
            assert not np.array_equal(perm, np.arange(len(x), dtype=np.uint32))
        assert rel_maxnorm(b.get_codebook(), a.get_codebook()) <= 1e-6
        assert np.array_equal(a.bmu_bound(None)[0], b.bmu_bound(None)[0])
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("kind", ["random", "adaptive"])
def test_device_sampler_after_relayout(pkg, data, kind):
    x, w, dist = data
    a, b = make_pair(pkg, x, w, dist)
    try:
        # two full epochs: b is re-laid out before its sampler starts
        for e in (a, b):
            e.train_epochs([0.5, 0.4], [6.0, 5.0])
            e.sampler_init(kind, len(x) // 10, 2608, 1.0, 2.0)
        assert rel_maxnorm(b.get_codebook(), a.get_codebook()) <= 1e-6
        for t in range(4):
            a.train_epoch(0.3, 3.0, sampled=True)
            b.train_epoch(0.3, 3.0, sampled=True)
        assert rel_maxnorm(b.get_codebook(), a.get_codebook()) <= 1e-6
        assert np.array_equal(a.sampler_select(), b.sampler_select())
        if kind == "adaptive":
            ea, aa = a.sampler_state()
            eb, ab = b.sampler_state()
            assert np.array_equal(aa, ab)
            assert np.allclose(ea, eb, rtol=1e-12, atol=0)
    finally:
        a.close()
        b.close()


def test_rebind_drops_order(pkg, data, oracle_port):
    x, w, dist = data
    _, b = make_pair(pkg, x, w, dist)
    try:
        b.set_influence(influence(oracle_port, dist, 6.0))
        b.epoch(0.5)
        b.epoch(0.5)  # re-laid out
        y = x[:20_000][::-1].copy()
        b.bind(y)
        assert np.array_equal(b.get_rows(), y)
        bb, _ = b.bmu_bound(None)
        assert np.array_equal(bb, oracle_port.find_bmus(y, w)[0])
    finally:
        b.close()


def test_row_order_option_validation(pkg):
    from paper_2604_26555_b200 import _lib
    e = pkg.Engine(16, 4)
    try:
        for v in (0, 1, 2, 3, 100):
            e.set_option(_lib.TSOM_OPT_ROW_ORDER, v)
        with pytest.raises(ValueError):
            e.set_option(_lib.TSOM_OPT_ROW_ORDER, -1)
    finally:
        e.close()


def test_short_runs_keep_the_bind_order(pkg, data):
    """Auto mode (the default) re-lays out only in a tsom_train_epochs call
    with >= 20 epochs left: a 10-epoch call and single-epoch calls leave the
    rows in bind order."""
    import ctypes as C
    from paper_2604_26555_b200 import _lib
    x, w, dist = data
    e = pkg.Engine(w.shape[0], w.shape[1])
    try:
        e.set_option(93, 0)
        e.bind(x)
        e.set_codebook(w)
        e.set_topology_distance(dist)
        e.train_epochs([0.5] * 10, [4.0] * 10)
        for _ in range(3):
            e.train_epoch(0.3, 3.0)
        L = _lib.load()
        L.tsom_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
        L.tsom_debug_read.restype = C.c_int64
        buf = np.empty(len(x), np.uint32)
        assert L.tsom_debug_read(e.h, 11, buf.ctypes.data, buf.nbytes) == 0  # no permutation
    finally:
        e.close()
