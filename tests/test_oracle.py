"""Pin the CPU oracle before trusting it (CPU only).

Two anchors, as the reference's own tests hold them (paths relative to
/root/reference/proj/tests):
  1. the reference's known-answer tests re-expressed here;
  2. bit-for-bit agreement of the C restatement (oracle.port) with the
     reference headers themselves (oracle.ref, built from /root/reference by
     oracle/Makefile) and with the committed golden vectors (tests/golden/).
"""
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CHECKERS = ["port", "ref"]


@pytest.fixture(params=CHECKERS)
def chk(request):
    c = getattr(oracle, request.param)
    if not c.available:
        pytest.skip(f"oracle.{request.param} not built")
    return c


# --- test_rng.cpp -----------------------------------------------------------

def test_mt19937_64_reference_value(oracle_port):
    # test_rng.cpp:23-29: the standard fixes the 10000th output of a default-seeded mt19937_64
    assert oracle_port.mt19937_64_default(10000) == 9981545732273789042


def test_seed_streams_match_reference(oracle_port, oracle_ref):
    for seed, stream in [(7, 1), (7, 2), (2605, 4), (0, 3)]:
        a, ga = oracle_port.rng_draws(seed, stream, 64)
        b, gb = oracle_ref.rng_draws(seed, stream, 64)
        assert (a == b).all() and (ga == gb).all()


# --- test_trainer.cpp: BMU --------------------------------------------------

def test_find_bmus_kat(chk):
    # test_trainer.cpp:213-222
    w = np.array([[0, 0], [5, 0], [0, 5]], np.float32)
    x = np.array([[1, 1], [4.5, 0.5]], np.float32)
    b, d = chk.find_bmus(x, w)
    assert b.tolist() == [0, 1]
    assert d[0] == pytest.approx(math.sqrt(2.0)) and d[1] == pytest.approx(math.sqrt(0.5))


def test_bmu_tie_lowest_index(chk):
    # test_trainer.cpp:224-232
    b, d = chk.find_bmus(np.array([[7.0]], np.float32), np.array([[2.0], [2.0], [2.0]], np.float32))
    assert b[0] == 0 and d[0] == pytest.approx(5.0)


def test_map_samples_kat(chk):
    # test_trainer.cpp:453-462
    b, d = chk.find_bmus(np.array([[1.0], [9.0], [4.0]], np.float32),
                         np.array([[0.0], [10.0]], np.float32))
    assert b.tolist() == [0, 1, 0] and d[2] == pytest.approx(4.0)


# --- test_trainer.cpp: accumulate + update ----------------------------------

def test_hand_computed_batch_step(chk):
    # test_trainer.cpp:246-277
    w = np.array([[0.0], [10.0]], np.float32)
    x = np.array([[1.0], [9.0]], np.float32)
    infl = np.array([[1.0, 0.5], [0.5, 1.0]])
    u, h, ur, hr, _ = chk.run_iteration(x, np.arange(2, dtype=np.uint32), w, infl, 0.2)
    assert u[0, 0] == pytest.approx(1.1) and h[0] == pytest.approx(1.5)
    assert u[1, 0] == pytest.approx(-1.1) and h[1] == pytest.approx(1.5)
    w2, prev = oracle.port.apply_update(w, np.zeros_like(w), u, h)
    assert w2[0, 0] == pytest.approx(1.1 / 1.5) and w2[1, 0] == pytest.approx(10.0 - 1.1 / 1.5)
    assert prev[0, 0] == 0.0


def test_momentum_and_safeguard(oracle_port):
    # test_trainer.cpp:279-295 (delta = 3/1 + 0.5*2 = 4)
    w, prev = oracle_port.apply_update(np.array([[0.0]], np.float32), np.array([[2.0]], np.float32),
                                       np.array([[3.0]]), np.array([1.0]), True, 0.5)
    assert w[0, 0] == pytest.approx(4.0) and prev[0, 0] == pytest.approx(4.0)
    # test_trainer.cpp:297-313 (H_1 = 0 < 1e-12: node frozen, memory cleared)
    w, prev = oracle_port.apply_update(np.array([[1.0], [5.0]], np.float32),
                                       np.array([[0.25], [0.75]], np.float32),
                                       np.array([[0.5], [0.0]]), np.array([1.0, 0.0]), True, 0.5)
    assert w[0, 0] == pytest.approx(1.0 + 0.5 + 0.5 * 0.25) and w[1, 0] == 5.0 and prev[1, 0] == 0.0


def test_chunk_count_invariance(chk):
    # test_trainer.cpp:315-333 (bit-exact across chunk counts)
    x = chk.synth_uniform(200, 4, 5)
    w = x[[3, 17, 42, 77, 91, 120, 150, 180, 199]].copy()
    infl = oracle.port.influence_from_dist(oracle.port.lattice_dist("rect", 3, 3), 1.5)
    sel = np.arange(200, dtype=np.uint32)
    base = chk.run_iteration(x, sel, w, infl, 0.3, 1)
    for chunks in (3, 7, 200):
        r = chk.run_iteration(x, sel, w, infl, 0.3, chunks)
        assert (r[2] == base[2]).all() and (r[3] == base[3]).all() and (r[4] == base[4]).all()


# --- test_parallel.cpp ------------------------------------------------------

def test_quantization_grid(oracle_port):
    # test_parallel.cpp:41-56
    assert oracle_port.quantize_term(1.0) == 1099511627776
    assert oracle_port.quantize_term(-0.5) == -549755813888
    assert oracle_port.quantize_term(0.0) == 0
    assert oracle_port.quantize_term(4194303.0) == 4194303 * 1099511627776
    for bad in (4194304.0, -1e30):
        with pytest.raises(oracle.OracleError, match="numerical fault"):
            oracle_port.quantize_term(bad)


@pytest.mark.parametrize("workers", [2, 3, 5])
def test_worker_split_equals_serial(chk, workers):
    # test_parallel.cpp:100-138
    x = chk.synth_uniform(120, 3, 1)
    w = x[:9].copy()
    infl = oracle.port.influence_from_dist(oracle.port.lattice_dist("rect", 3, 3), 1.2)
    sel = np.arange(120, dtype=np.uint32)
    a = chk.run_iteration(x, sel, w, infl, 0.4, 2, 1)
    b = chk.run_iteration(x, sel, w, infl, 0.4, 2, workers)
    assert (a[2] == b[2]).all() and (a[3] == b[3]).all() and (a[4] == b[4]).all()


# --- test_metrics.cpp -------------------------------------------------------

def test_qe_kat(chk):
    # test_metrics.cpp:11-17: distances 1, 1, 1, 2 -> 1.25
    qe = chk.mean_bmu_distance(np.array([[1.0], [-1.0], [9.0], [12.0]], np.float32),
                               np.array([[0.0], [10.0]], np.float32))
    assert qe == pytest.approx(1.25)


# --- test_topology.cpp ------------------------------------------------------

def test_influence_kats(chk):
    # test_topology.cpp:314-328
    h = chk.influence_from_dist(np.array([0.0, 1.0, 2.0]), 1.0)
    assert h[0] == 1.0 and h[1] == pytest.approx(math.exp(-0.5)) and h[2] == pytest.approx(math.exp(-2.0))
    g = chk.influence_from_hops(np.array([0, 3], np.uint16), 2.0)
    assert g[0] == 1.0 and g[1] == pytest.approx(math.exp(-9.0 / 8.0))


def test_hops_path_graph(chk):
    # test_topology.cpp:412-420: a path 0-1-2 built by MST
    sq = chk.pairwise_sq_dists(np.array([[0.0], [1.0], [2.0]], np.float32))
    e = chk.build_graph("mst", sq)
    hops = chk.hop_distances(e, 3)
    assert hops[0, 1] == 1 and hops[0, 2] == 2 and hops[0, 0] == 0


def test_refresh_schedule(oracle_port):
    # test_topology.cpp:351-367 via the training loop's refresh log: growth 2, warmup 10
    x = oracle_port.synth_uniform(60, 2, 28)
    cfg = oracle.SomConfig(topology="mst", nodes=6, n_iters=30, refresh_warmup=10,
                           refresh_growth=2.0, refresh_max_interval=25, seed=1)
    _, _, ref = oracle_port.train(cfg, x)
    assert np.flatnonzero(ref).tolist() == [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 16, 24]


# --- whole runs --------------------------------------------------------------

def test_two_blobs_converge(chk):
    # test_trainer.cpp:398-412
    x = np.zeros((120, 2), np.float32)
    rng = np.random.default_rng(13)
    x[:60] = 0.0 + 0.01 * rng.standard_normal((60, 2))
    x[60:] = 8.0 + 0.01 * rng.standard_normal((60, 2))
    cfg = oracle.SomConfig(topology="rect", grid_w=2, grid_h=1, n_iters=60, eta0=0.8,
                           sigma_min=0.05, seed=5)
    w, _, _ = chk.train(cfg, x)
    xs = sorted(w[:, 0].tolist())
    assert xs[0] == pytest.approx(0.0, abs=0.05) and xs[1] == pytest.approx(8.0, abs=0.05)


CONFIGS = [
    oracle.SomConfig(topology="hex", grid_w=4, grid_h=4, n_iters=8, seed=17),
    oracle.SomConfig(topology="mst", nodes=16, n_iters=8, seed=17, n_threads=2),
    oracle.SomConfig(topology="rng", nodes=12, n_iters=6, seed=4, sampling="adaptive", rho=0.3),
    oracle.SomConfig(topology="rect", grid_w=5, grid_h=3, n_iters=6, seed=23, sampling="random",
                     rho=0.5, use_momentum=True, momentum=0.4),
]


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"{c.topology}-{c.sampling}")
def test_port_train_equals_reference(oracle_port, oracle_ref, cfg):
    x = oracle_port.synth_gmm(300, 8, 2610)
    a = oracle_port.train(cfg, x, log_qe=True)
    b = oracle_ref.train(cfg, x, log_qe=True)
    assert (a[0] == b[0]).all(), "final weights must be bit-identical"
    assert (a[1] == b[1]).all() and (a[2] == b[2]).all()


def test_port_hot_path_equals_reference(oracle_port, oracle_ref):
    x = oracle_port.synth_gmm(3000, 50, 2605)
    assert (x == oracle_ref.synth_gmm(3000, 50, 2605)).all()
    w = x[:100] + np.float32(0.25)
    bp, dp = oracle_port.find_bmus(x, w)
    br, dr = oracle_ref.find_bmus(x, w)
    assert (bp == br).all() and (dp == dr).all()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 10, 10), 2.5)
    sel = np.arange(0, 3000, 3, dtype=np.uint32)
    a = oracle_port.run_iteration(x, sel, w, infl, 0.37, 1, 4)
    b = oracle_ref.run_iteration(x, sel, w, infl, 0.37, 1, 1)
    assert all((p == q).all() for p, q in zip(a, b))


# --- golden fixtures (generated by tests/golden/make_golden.py from oracle.ref) --

def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} missing")
    return np.load(path)


def test_golden_hot_path(oracle_port):
    g = _golden("hot_path.npz")
    b, d = oracle_port.find_bmus(g["x"], g["w"])
    assert (b == g["bmu"]).all() and (d == g["dist"]).all()
    r = oracle_port.run_iteration(g["x"], g["sel"], g["w"], g["infl"], float(g["eta"]), 1, 1)
    assert (r[2] == g["u_raw"]).all() and (r[3] == g["h_raw"]).all()


def test_golden_training_runs(oracle_port):
    g = _golden("train_runs.npz")
    for i, cfg in enumerate(CONFIGS):
        w, qe, _ = oracle_port.train(cfg, g["x"], log_qe=True)
        assert (w == g[f"w{i}"]).all() and (qe == g[f"qe{i}"]).all()
