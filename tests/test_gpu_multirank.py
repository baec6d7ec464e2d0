"""The engine's own multi-rank epoch, on one GPU.

Ranks are engines joined by an in-process rank group (tsom_group_*, the same
reduce hook NCCL uses: one ordered f64 reduce of [S | c | sum dist | rows] per
epoch), each driven from its own thread and owning a
contiguous slice of the rows (assign_shards, parallel.hpp:28-41).  The
reference pins worker-count invariance (test_parallel.cpp:144-162: G in
{1, 2, 4} give identical accumulators); here G ranks must give the
single-engine result:

  * one epoch: U / H to 1e-12 of max|U| / rtol 1e-12 (only the FP64 grouping
    of the per-rank sums differs), per-row distances and BMUs bit-identical;
  * whole device-resident runs (tsom_train_epochs, sharded device sampler,
    device topology refresh): codebooks to 1e-6 relative max-norm (in practice
    identical) and the reference's golden runs to the single-engine bars;
  * the C++ drop-ins with several engines (CudaExecutor as a ThreadedExecutor
    of engines, train_device) against the reference's runs;
  * the barrier deadline: a rank that never arrives is named
    ("reduce barrier timed out after X s waiting for worker g",
    collect_with_barrier parallel.hpp:67-86), and a NCCL communicator whose
    peers never join is aborted instead of hanging.
"""
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


def assign_shards(n, g):
    """parallel.hpp:28-41: the first n mod G slices get one extra item."""
    base, extra = divmod(n, g)
    out, b = [], 0
    for r in range(g):
        c = base + (1 if r < extra else 0)
        out.append((b, b + c))
        b += c
    return out


def rel_maxnorm(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-300))


def run_ranks(world, fn):
    """fn(rank) on `world` threads; re-raise the first failure in rank order."""
    out, err = [None] * world, [None] * world

    def main(r):
        try:
            out[r] = fn(r)
        except BaseException as ex:  # noqa: BLE001 - reported below
            err[r] = ex

    th = [threading.Thread(target=main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    # the first failure in rank order; a peer's "aborted" follows a timeout
    for e in err:
        if e is not None and "reduce barrier aborted" not in str(e):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out


def make_ranks(pkg, x, p, world, configure):
    """world engines, rank r bound to slice r of x, joined by one group."""
    g = pkg.RankGroup(world)
    sl = assign_shards(len(x), world)
    engines = []
    for r, (a, b) in enumerate(sl):
        e = pkg.Engine(p, x.shape[1])
        e.bind(x[a:b])
        e.join_group(g, r)
        configure(e)
        engines.append(e)
    return g, engines, sl


# --- one epoch ---------------------------------------------------------------

@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("sampling", ["full", "random"])
def test_epoch_ranks_equal_single_engine(pkg, oracle_port, world, sampling):
    n, p = 30011, 256
    x = oracle_port.synth_gmm(n, 50, 2700 + world)
    w = x[np.linspace(0, n - 1, p).astype(int)].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("hex", 16, 16), 4.0)
    sel = None
    if sampling == "random":
        sel = np.sort(np.random.default_rng(world).choice(n, n // 3, replace=False)).astype(np.uint32)

    def configure(e):
        e.set_codebook(w)
        e.set_influence(infl)

    single = pkg.Engine(p, 50)
    single.bind(x)
    configure(single)
    u1, h1, d1 = single.epoch(0.45, sel, want_dist=True)
    b1, _ = single.bmu_bound(sel, want_dist=False)

    g, engines, sl = make_ranks(pkg, x, p, world, configure)

    def local_sel(r):
        if sel is None:
            return None
        a, b = sl[r]
        s = sel[(sel >= a) & (sel < b)]
        return (s - a).astype(np.uint32)

    res = run_ranks(world, lambda r: engines[r].epoch(0.45, local_sel(r), want_dist=True))
    for r in range(world):  # every rank holds the reduced sums
        u, h, _ = res[r]
        assert np.max(np.abs(u - u1)) <= 1e-12 * np.max(np.abs(u1)), f"rank {r} U"
        np.testing.assert_allclose(h, h1, rtol=1e-12, atol=0)
    d = np.concatenate([res[r][2] for r in range(world)])
    assert (d == d1).all(), "per-row distances (exact FP64) differ"
    bm = run_ranks(world, lambda r: engines[r].bmu_bound(local_sel(r), want_dist=False)[0])
    assert (np.concatenate(bm) == b1).all()
    # and the reference with G workers (its result is G-invariant)
    ids = np.arange(n, dtype=np.uint32) if sel is None else sel
    uo, ho, _, _, _ = oracle_port.run_iteration(x, ids, w, infl, 0.45, 1, world)
    assert np.max(np.abs(res[0][0] - uo)) <= 1e-9 * np.max(np.abs(uo))
    # QE over the ranks: one reduce of the distance sums
    qe = run_ranks(world, lambda r: engines[r].qe(local_sel(r)))
    s1, c1 = single.qe(sel)
    assert all(c == c1 for _, c in qe)
    assert all(abs(s - s1) <= 1e-12 * s1 for s, _ in qe)
    assert engines[0].barrier_wait_s > 0.0
    for e in engines:
        e.close()
    g.close()


def test_epoch_rank_with_no_rows(pkg, oracle_port):
    """A rank whose slice holds no selected row still joins the reduce (an
    empty slice, assign_shards with G > n, parallel.hpp:26-27)."""
    n, p = 5000, 64
    x = oracle_port.synth_gmm(n, 50, 2711)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 8, 8), 2.0)

    def configure(e):
        e.set_codebook(w)
        e.set_influence(infl)

    single = pkg.Engine(p, 50)
    single.bind(x)
    configure(single)
    sel = np.arange(100, 900, dtype=np.uint32)  # all in rank 0's slice
    u1, h1, d1 = single.epoch(0.3, sel, want_dist=True)
    g, engines, sl = make_ranks(pkg, x, p, 3, configure)
    sels = [sel - sl[0][0], np.array([], np.uint32), np.array([], np.uint32)]
    res = run_ranks(3, lambda r: engines[r].epoch(0.3, sels[r], want_dist=True))
    for r in range(3):
        assert np.max(np.abs(res[r][0] - u1)) <= 1e-12 * np.max(np.abs(u1))
        np.testing.assert_allclose(res[r][1], h1, rtol=1e-12)
    assert (res[0][2] == d1).all()
    g.close()


# --- whole device-resident runs ----------------------------------------------

def _schedules(n_iters, sigma0, sigma_min=0.3):
    from paper_2604_26555_b200.hostref import schedule_value
    etas = [schedule_value(0.5, "linear", t, n_iters, 1e-4) for t in range(n_iters)]
    sigmas = [schedule_value(sigma0, "linear", t, n_iters, sigma_min) for t in range(n_iters)]
    return etas, sigmas


@pytest.mark.parametrize("world", [2, 3, 4])
def test_train_epochs_ranks_equal_single_engine(pkg, oracle_port, world):
    """tsom_train_epochs (c2 shape on 40k rows: 32x32 hex, 10 epochs) split over
    `world` ranks: every rank ends with the single engine's codebook."""
    from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist, resolved_sigma0
    n, p = 40000, 1024
    x = oracle_port.synth_gmm(n, 50, 2606)
    w0 = init_sample_draw(x, p, 2606)
    dist = lattice_dist("hex", 32, 32)
    etas, sigmas = _schedules(10, resolved_sigma0("hex", 32, 32))

    def configure(e):
        e.set_codebook(w0)
        e.set_topology_distance(dist)

    single = pkg.Engine(p, 50)
    single.bind(x)
    configure(single)
    single.train_epochs(etas, sigmas)
    w1 = single.get_codebook()
    g, engines, _ = make_ranks(pkg, x, p, world, configure)
    run_ranks(world, lambda r: engines[r].train_epochs(etas, sigmas))
    for r in range(world):
        assert rel_maxnorm(engines[r].get_codebook(), w1) <= 1e-6, f"rank {r}"
    q = run_ranks(world, lambda r: engines[r].qe())
    s1, c1 = single.qe()
    assert q[0][1] == c1 and abs(q[0][0] - s1) <= 1e-9 * s1
    g.close()


@pytest.mark.parametrize("world,kind", [(2, "adaptive"), (3, "adaptive"), (3, "random")])
def test_sampled_rng_run_ranks_equal_single_engine(pkg, oracle_port, world, kind):
    """The c4 shape in small (RNG graph refreshed on the device, device sampler
    rho = 0.2, 8 epochs) with the rows split over ranks: one sharded sampler
    picks the reference Sampler's rows, one reduce per epoch; every rank ends
    with the single engine's codebook."""
    from paper_2604_26555_b200.hostref import RefreshState, init_sample_draw, resolved_sigma0
    n, p, iters = 24000, 128, 8
    x = oracle_port.synth_gmm(n, 50, 2608 + world)
    w0 = init_sample_draw(x, p, 2608)
    m = int(n * 0.2)
    etas, sigmas = _schedules(iters, resolved_sigma0("rng", 0, 0, 0.0))

    def train(e):
        e.sampler_init(kind, m, 2608)
        refresh = RefreshState(max(1, iters // 10), 1.5, 25)
        for t in range(iters):
            if refresh.should_refresh(t):
                e.refresh_topology("rng")
                refresh.mark(t)
            e.train_epoch(etas[t], sigmas[t], sampled=True)
        return e.get_codebook()

    single = pkg.Engine(p, 50)
    single.bind(x)
    single.set_codebook(w0)
    w1 = train(single)
    g, engines, _ = make_ranks(pkg, x, p, world, lambda e: e.set_codebook(w0))
    ws = run_ranks(world, lambda r: train(engines[r]))
    for r in range(world):
        assert rel_maxnorm(ws[r], w1) <= 1e-6, f"rank {r}"
    g.close()


# --- the C++ drop-ins with several engines -----------------------------------

DROPIN_CONFIGS = [
    dict(topology="hex", grid_w=4, grid_h=4, n_iters=8, seed=17),
    dict(topology="mst", nodes=16, n_iters=8, seed=17),
    dict(topology="rng", nodes=12, n_iters=6, seed=4, sampling="adaptive", rho=0.3),
    dict(topology="rect", grid_w=5, grid_h=3, n_iters=6, seed=23, sampling="random", rho=0.5,
         use_momentum=True, momentum=0.4),
]


@pytest.mark.parametrize("engines", [2, 3])
@pytest.mark.parametrize("kw", DROPIN_CONFIGS, ids=lambda k: f"{k['topology']}")
def test_dropin_executor_engines_vs_golden(pkg, kw, engines):
    """train_with_executor + a CudaExecutor of `engines` engines (the
    ThreadedExecutor shape) vs the reference's run and the one-engine run."""
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "train_runs.npz"))
    i = DROPIN_CONFIGS.index(kw)
    cfg = dropin.TrainConfig(**kw)
    w1, qe1, _, _ = dropin.train_cuda(cfg, g["x"], log_qe=True)
    w, qe, _, _ = dropin.train_cuda(cfg, g["x"], log_qe=True, engines=engines)
    assert rel_maxnorm(w, g[f"w{i}"]) <= 1e-4
    np.testing.assert_allclose(qe, g[f"qe{i}"], rtol=1e-5)
    assert rel_maxnorm(w, w1) <= 1e-6
    np.testing.assert_allclose(qe, qe1, rtol=1e-12)


@pytest.mark.parametrize("engines", [2, 4])
@pytest.mark.parametrize("kw", DROPIN_CONFIGS, ids=lambda k: f"{k['topology']}")
def test_dropin_train_device_engines(pkg, kw, engines):
    """toposom_b200::train_device with the rows split over `engines` engines."""
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "train_runs.npz"))
    i = DROPIN_CONFIGS.index(kw)
    cfg = dropin.TrainConfig(**kw)
    w1, qe1, r1, _ = dropin.train_device(cfg, g["x"], log_qe=True)
    w, qe, r, _ = dropin.train_device(cfg, g["x"], log_qe=True, engines=engines)
    assert rel_maxnorm(w, w1) <= 1e-6
    np.testing.assert_allclose(qe, qe1, rtol=1e-12)
    assert (r == r1).all()
    assert rel_maxnorm(w, g[f"w{i}"]) <= 1e-4
    np.testing.assert_allclose(qe, g[f"qe{i}"], rtol=1e-5)


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_config_shape_runs_on_three_engines(pkg, oracle_port, name):
    """The BASELINE shapes (K = 1024, 1e5 rows, 10 epochs) through
    train_device with the rows on 3 engines vs the reference's runs (the
    bars of tests/test_gpu_configs.py) and the 1-engine run."""
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    path = os.path.join(GOLDEN, "config_shapes_1e5.npz")
    if not os.path.exists(path):
        pytest.skip("golden runs not generated")
    gold = np.load(path)
    seed, n = int(gold[f"{name}_seed"]), int(gold["n"])
    x = oracle_port.synth_gmm(n, 50, seed)
    kw = {"c2": dict(topology="hex", grid_w=32, grid_h=32),
          "c3": dict(topology="mst", nodes=1024),
          "c4": dict(topology="rng", nodes=1024, sampling="adaptive", rho=0.1)}[name]
    cfg = dropin.TrainConfig(n_iters=10, seed=seed, **kw)
    w1, qe1, _, _ = dropin.train_device(cfg, x, log_qe=True)
    w, qe, ref, _ = dropin.train_device(cfg, x, log_qe=True, engines=3)
    assert rel_maxnorm(w, w1) <= 1e-6
    ref_w = gold[f"{name}_w"]
    dev = np.max(np.abs(w.astype(np.float64) - ref_w), axis=1) / np.max(np.abs(ref_w))
    hits = np.bincount(oracle_port.find_bmus(x, ref_w)[0], minlength=1024)
    need = 20 if name == "c4" else 1
    assert dev[hits >= need].max() <= 1e-4
    assert dev.max() <= 1e-3
    np.testing.assert_allclose(qe, gold[f"{name}_qe"], rtol=1e-5)
    assert (ref == gold[f"{name}_refresh"]).all()


# --- the barrier deadline -------------------------------------------------------

def test_reduce_barrier_names_the_missing_rank(pkg, oracle_port):
    """Rank 1 never reaches the reduce: rank 0 fails after the deadline with the
    reference's message (collect_with_barrier, parallel.hpp:67-86) instead of
    hanging, and its engine keeps working on its own afterwards."""
    from paper_2604_26555_b200 import _lib
    n, p = 4000, 64
    x = oracle_port.synth_gmm(n, 50, 2720)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 8, 8), 2.0)
    g = pkg.RankGroup(2)
    e0 = pkg.Engine(p, 50)
    e0.bind(x[:2000])
    e0.join_group(g, 0)
    e0.set_option(_lib.TSOM_OPT_BARRIER_TIMEOUT_MS, 300)
    e0.set_codebook(w)
    e0.set_influence(infl)
    with pytest.raises(pkg.BarrierTimeout,
                       match=r"^reduce barrier timed out after 0\.300000 s waiting for worker 1$"):
        e0.epoch(0.5)
    assert isinstance(pkg.BarrierTimeout(6, ""), RuntimeError)  # std::runtime_error
    g.close()


def test_barrier_timeout_in_the_drop_in_is_a_runtime_error(pkg, oracle_port):
    """A 3-rank group where rank 2 arrives late: ranks 0 and 1 time out, and
    the executor's collection names worker 2."""
    from paper_2604_26555_b200 import _lib
    n, p = 3000, 16
    x = oracle_port.synth_gmm(n, 50, 2721)
    w = x[:p].copy()
    infl = np.eye(p)

    def configure(e):
        e.set_option(_lib.TSOM_OPT_BARRIER_TIMEOUT_MS, 250)
        e.set_codebook(w)
        e.set_influence(infl)

    g, engines, _ = make_ranks(pkg, x, p, 3, configure)

    def rank(r):
        if r == 2:
            return None  # never arrives
        return engines[r].epoch(0.5)

    with pytest.raises(pkg.BarrierTimeout, match="waiting for worker 2"):
        run_ranks(3, rank)
    g.close()


def test_nccl_comm_init_times_out_without_peers(pkg):
    """A non-blocking NCCL communicator of world 2 whose rank 1 never joins:
    initialisation is aborted at the deadline (ncclCommAbort) instead of
    blocking, and the engine stays usable on its own."""
    from paper_2604_26555_b200 import _lib
    e = pkg.Engine(16, 4)
    e.set_option(_lib.TSOM_OPT_BARRIER_TIMEOUT_MS, 1500)
    uid = e.comm_unique_id()
    with pytest.raises(pkg.BarrierTimeout, match="comm init timed out"):
        e.comm_init(uid, 0, 2)
    x = np.random.default_rng(0).standard_normal((500, 4)).astype(np.float32)
    e.bind(x)
    e.set_codebook(x[:16])
    e.set_influence(np.eye(16))
    u, h, _ = e.epoch(0.5)
    assert h.sum() == 500.0


def test_selection_validation(pkg, oracle_port):
    """fetch_rows (dataset.hpp:393-416) gathers any list of in-range ids: an
    unsorted list with repeats is a valid gather (same sums as the sorted
    multiset), an id past the data anywhere in the list is out_of_range, and an
    N-long list spanning [0, N-1] that is not the identity is not treated as
    one."""
    n, p = 3000, 32
    x = oracle_port.synth_gmm(n, 50, 2722)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 8, 4), 2.0)
    e = pkg.Engine(p, 50)
    e.bind(x)
    e.set_codebook(w)
    e.set_influence(infl)
    rng = np.random.default_rng(3)
    sel = rng.integers(0, n, 2000).astype(np.uint32)  # unsorted, with repeats
    u, h, d = e.epoch(0.5, sel, want_dist=True)
    uo, ho, _, _, do = oracle_port.run_iteration(x, sel, w, infl, 0.5, 1, 1)
    assert np.max(np.abs(u - uo)) <= 1e-9 * np.max(np.abs(uo))
    np.testing.assert_allclose(h, ho, rtol=1e-9)
    np.testing.assert_allclose(d, do, rtol=1e-12)
    bad = np.arange(n, dtype=np.uint32)
    bad[1500] = n + 7  # out of range in the middle, endpoints look fine
    with pytest.raises(IndexError, match="fetch_rows: row index beyond data size"):
        e.epoch(0.5, bad)
    dup = np.arange(n, dtype=np.uint32)
    dup[1] = 0  # N ids spanning [0, N-1], not the identity
    u2, h2, _ = e.epoch(0.5, dup)
    uo2, ho2, _, _, _ = oracle_port.run_iteration(x, dup, w, infl, 0.5, 1, 1)
    np.testing.assert_allclose(h2, ho2, rtol=1e-9)
    assert np.max(np.abs(u2 - uo2)) <= 1e-9 * np.max(np.abs(uo2))


# --- exact mode: bit-identical for any rank count ------------------------------
#
# TSOM_OPT_DETERMINISTIC puts every feature value and distance on a fixed-point
# grid set by the data's global bounds and sums them in int64 limbs, reduced as
# integers: the reference's guarantee (accum.hpp:12-20, parallel.hpp:17-21 —
# "any G produces bit-identical final weights"; test_parallel.cpp:144-162).

def exact_engine(pkg, rows, p, configure):
    from paper_2604_26555_b200 import _lib
    e = pkg.Engine(p, rows.shape[1])
    e.set_option(_lib.TSOM_OPT_DETERMINISTIC, 1)
    e.bind(rows)
    configure(e)
    return e


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exact_epoch_bit_identical_across_ranks(pkg, oracle_port, world):
    from paper_2604_26555_b200 import _lib
    n, p = 30011, 256
    x = oracle_port.synth_gmm(n, 50, 2750 + world)
    w = x[np.linspace(0, n - 1, p).astype(int)].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("hex", 16, 16), 4.0)

    def configure(e):
        e.set_codebook(w)
        e.set_influence(infl)

    single = exact_engine(pkg, x, p, configure)
    u1, h1, d1 = single.epoch(0.45, want_dist=True)
    s1, c1 = single.qe()
    plain = pkg.Engine(p, 50)
    plain.bind(x)
    configure(plain)
    u0, h0, _ = plain.epoch(0.45)
    assert np.max(np.abs(u1 - u0)) <= 1e-12 * np.max(np.abs(u0))  # the grid costs nothing
    assert np.array_equal(h1, h0)
    g = pkg.RankGroup(world)
    sl = assign_shards(n, world)
    engines = []
    for r, (a, b) in enumerate(sl):
        e = exact_engine(pkg, x[a:b], p, configure)
        e.join_group(g, r)
        engines.append(e)
    res = run_ranks(world, lambda r: engines[r].epoch(0.45, want_dist=True))
    for r in range(world):
        assert np.array_equal(res[r][0], u1), f"rank {r}: U not bit-identical"
        assert np.array_equal(res[r][1], h1)
    assert np.array_equal(np.concatenate([res[r][2] for r in range(world)]), d1)
    q = run_ranks(world, lambda r: engines[r].qe())
    assert all(s == s1 and c == c1 for s, c in q)
    g.close()


def test_exact_sums_ignore_selection_order(pkg, oracle_port):
    """The same multiset of rows in any order gives bit-identical sums."""
    n, p = 20000, 128
    x = oracle_port.synth_gmm(n, 50, 2760)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 16, 8), 3.0)

    def configure(e):
        e.set_codebook(w)
        e.set_influence(infl)

    e = exact_engine(pkg, x, p, configure)
    sel = np.sort(np.random.default_rng(4).choice(n, 9000, replace=False)).astype(np.uint32)
    u1, h1, _ = e.epoch(0.5, sel)
    u2, h2, _ = e.epoch(0.5, np.random.default_rng(5).permutation(sel))
    assert np.array_equal(u1, u2) and np.array_equal(h1, h2)


@pytest.mark.parametrize("world", [2, 4])
def test_exact_training_bit_identical_across_ranks(pkg, oracle_port, world):
    """tsom_train_epochs at the c2 shape: every rank's final codebook equals the
    single engine's bit for bit."""
    from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist, resolved_sigma0
    n, p = 40000, 1024
    x = oracle_port.synth_gmm(n, 50, 2606)
    w0 = init_sample_draw(x, p, 2606)
    dist = lattice_dist("hex", 32, 32)
    etas, sigmas = _schedules(10, resolved_sigma0("hex", 32, 32))

    def configure(e):
        e.set_codebook(w0)
        e.set_topology_distance(dist)

    single = exact_engine(pkg, x, p, configure)
    single.train_epochs(etas, sigmas)
    w1 = single.get_codebook()
    g = pkg.RankGroup(world)
    engines = []
    for r, (a, b) in enumerate(assign_shards(n, world)):
        e = exact_engine(pkg, x[a:b], p, configure)
        e.join_group(g, r)
        engines.append(e)
    run_ranks(world, lambda r: engines[r].train_epochs(etas, sigmas))
    for r in range(world):
        assert np.array_equal(engines[r].get_codebook(), w1), f"rank {r}"
    g.close()


@pytest.mark.parametrize("kw", [dict(topology="rng", nodes=12, n_iters=6, seed=4,
                                     sampling="adaptive", rho=0.3),
                                dict(topology="hex", grid_w=4, grid_h=4, n_iters=8, seed=17)],
                         ids=["rng-adaptive", "hex"])
def test_exact_dropin_bit_identical_across_engines(pkg, kw):
    """The C++ drop-ins with CudaOptions::exact: 1, 2 and 3 engines give the same
    weights bit for bit (the reference's train_parallel guarantee)."""
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "train_runs.npz"))
    cfg = dropin.TrainConfig(**kw)
    ws = [dropin.train_device(cfg, g["x"], engines=k, exact=True)[0] for k in (1, 2, 3)]
    assert np.array_equal(ws[0], ws[1]) and np.array_equal(ws[0], ws[2])
    wc = [dropin.train_cuda(cfg, g["x"], engines=k, exact=True)[0] for k in (1, 3)]
    assert np.array_equal(wc[0], wc[1])


@pytest.mark.parametrize("world", [1, 3])
def test_exact_training_with_bmu_ordered_shards(pkg, oracle_port, world):
    """Every rank re-lays its shard out in BMU order (TSOM_OPT_ROW_ORDER, forced
    at this size) while the single reference engine keeps the bind order: in
    exact mode the sums do not depend on the row order, so the codebooks are
    identical bit for bit, and the per-row BMUs come back in caller order."""
    from paper_2604_26555_b200 import _lib
    from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist, resolved_sigma0
    n, p = 40000, 1024
    x = oracle_port.synth_gmm(n, 50, 2606)
    w0 = init_sample_draw(x, p, 2606)
    dist = lattice_dist("hex", 32, 32)
    etas, sigmas = _schedules(10, resolved_sigma0("hex", 32, 32))

    def configure(e):
        e.set_codebook(w0)
        e.set_topology_distance(dist)

    single = exact_engine(pkg, x, p, configure)
    single.set_option(_lib.TSOM_OPT_ROW_ORDER, 0)
    single.train_epochs(etas, sigmas)
    w1 = single.get_codebook()
    b1, _ = single.bmu_bound(None, want_dist=False)
    g = pkg.RankGroup(world)
    engines = []
    sl = assign_shards(n, world)
    for r, (a, b) in enumerate(sl):
        e = pkg.Engine(p, 50)
        e.set_option(_lib.TSOM_OPT_DETERMINISTIC, 1)
        e.set_option(_lib.TSOM_OPT_ROW_ORDER, 2)  # once, at the second full pass
        e.set_option(93, 0)  # even for these shards
        e.bind(x[a:b])
        configure(e)
        e.join_group(g, r)
        engines.append(e)
    run_ranks(world, lambda r: engines[r].train_epochs(etas, sigmas))
    for r in range(world):
        assert np.array_equal(engines[r].get_codebook(), w1), f"rank {r}"
    bm = run_ranks(world, lambda r: engines[r].bmu_bound(None, want_dist=False)[0])
    assert (np.concatenate(bm) == b1).all()
    for r, (a, b) in enumerate(sl):
        assert np.array_equal(engines[r].get_rows(), x[a:b])
    g.close()
