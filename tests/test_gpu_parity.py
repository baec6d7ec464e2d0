"""GPU parity: the B200 engine (through the C-ABI) against the CPU oracle.

Bars:
  * BMU indices: bit-exact for every row (near-ties are re-checked in exact FP64);
  * per-row distances: rtol 1e-12 (FP64, summation order differs);
  * U, H accumulators of one epoch: rtol 1e-9 of max|U| (FP64 smoothing of
    FP32-per-CTA residual sums flushed to FP64);
  * whole runs: codebook relative max-norm <= 1e-4, QE relative <= 1e-5.
"""
import math
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KERNELS = [1, 2, 3]  # SIMT, tcgen05 3xTF32, tcgen05 3xFP16


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


def engine(pkg, p, d, kernel=0):
    e = pkg.Engine(p, d)
    if kernel in (2, 3):
        from paper_2604_26555_b200 import _lib
        try:
            e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kernel)
        except pkg.InvalidArgument:
            pytest.skip("tcgen05 kernel unsupported for this shape")
    elif kernel == 1:
        from paper_2604_26555_b200 import _lib
        e.set_option(_lib.TSOM_OPT_BMU_KERNEL, 1)
    return e


def rel_maxnorm(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(b)), 1e-300))


# --- reference KATs through the engine -------------------------------------

@pytest.mark.parametrize("kernel", KERNELS)
def test_find_bmus_kat(pkg, kernel):
    # test_trainer.cpp:213-222
    e = engine(pkg, 3, 2, kernel)
    e.set_codebook(np.array([[0, 0], [5, 0], [0, 5]], np.float32))
    b, d = e.bmu(np.array([[1, 1], [4.5, 0.5]], np.float32))
    assert b.tolist() == [0, 1]
    assert d[0] == pytest.approx(math.sqrt(2.0), rel=1e-14)
    assert d[1] == pytest.approx(math.sqrt(0.5), rel=1e-14)


@pytest.mark.parametrize("kernel", KERNELS)
def test_bmu_ties_lowest_index(pkg, kernel):
    # test_trainer.cpp:224-232: equidistant nodes -> node 0, distance 5
    e = engine(pkg, 3, 1, kernel)
    e.set_codebook(np.array([[2.0], [2.0], [2.0]], np.float32))
    b, d = e.bmu(np.array([[7.0]], np.float32))
    assert b[0] == 0 and d[0] == pytest.approx(5.0)


def test_map_samples_and_qe_kats(pkg):
    # test_trainer.cpp:453-462 and test_metrics.cpp:11-17
    w = np.array([[0.0], [10.0]], np.float32)
    b, d = pkg.map_samples(w, np.array([[1.0], [9.0], [4.0]], np.float32))
    assert b.tolist() == [0, 1, 0] and d[2] == pytest.approx(4.0)
    assert pkg.quantization_error(np.array([[1.0], [-1.0], [9.0], [12.0]], np.float32), w) == \
        pytest.approx(1.25)
    with pytest.raises(ValueError, match="dimension mismatch"):
        pkg.find_bmus(np.zeros((1, 2), np.float32), np.zeros((2, 3), np.float32))


def test_hand_computed_batch_step(pkg):
    # test_trainer.cpp:246-277: U0 = 1.1, H0 = 1.5, U1 = -1.1, H1 = 1.5
    e = pkg.Engine(2, 1)
    e.bind(np.array([[1.0], [9.0]], np.float32))
    e.set_codebook(np.array([[0.0], [10.0]], np.float32))
    e.set_influence(np.array([[1.0, 0.5], [0.5, 1.0]]))
    u, h, _ = e.epoch(0.2)
    assert u[0, 0] == pytest.approx(1.1, rel=1e-12) and h[0] == pytest.approx(1.5, rel=1e-12)
    assert u[1, 0] == pytest.approx(-1.1, rel=1e-12) and h[1] == pytest.approx(1.5, rel=1e-12)


def test_device_update_hand_step_and_safeguard(pkg):
    # same step through the device-resident update (apply_update on the GPU):
    # influence exp(-d^2/2) = 0.5 at d = sqrt(2 ln 2)
    e = pkg.Engine(2, 1)
    e.bind(np.array([[1.0], [9.0]], np.float32))
    e.set_codebook(np.array([[0.0], [10.0]], np.float32))
    dd = math.sqrt(2 * math.log(2.0))
    e.set_topology_distance(np.array([[0.0, dd], [dd, 0.0]]))
    e.train_epoch(0.2, 1.0)
    w = e.get_codebook()
    assert w[0, 0] == pytest.approx(1.1 / 1.5, rel=1e-6)
    assert w[1, 0] == pytest.approx(10.0 - 1.1 / 1.5, rel=1e-6)
    # H floor (trainer.hpp:349-353): a node with no support does not move
    e2 = pkg.Engine(2, 1)
    e2.bind(np.array([[1.0]], np.float32))
    e2.set_codebook(np.array([[0.0], [100.0]], np.float32))
    e2.set_topology_distance(np.array([[0.0, 100.0], [100.0, 0.0]]))
    e2.train_epoch(0.5, 1.0)
    w2 = e2.get_codebook()
    # node 0: H = 1, U = 0.5 * (1 - 0) -> moves halfway; node 1: h = exp(-5000) cut to 0
    assert w2[1, 0] == 100.0 and w2[0, 0] == pytest.approx(0.5)


# --- BMU bit-exactness at scale ----------------------------------------------

@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("p,n", [(100, 20000), (1024, 20000), (300, 7777)])
def test_bmu_bit_exact_vs_oracle(pkg, oracle_port, kernel, p, n):
    x = oracle_port.synth_gmm(n, 50, 2600 + p)
    w = x[np.linspace(0, n - 1, p).astype(int)] * np.float32(0.9) + np.float32(0.05)
    e = engine(pkg, p, 50, kernel)
    e.set_codebook(w)
    b, d = e.bmu(x)
    bo, do = oracle_port.find_bmus(x, w)
    assert (b == bo).all(), f"{int((b != bo).sum())} BMU mismatches"
    np.testing.assert_allclose(d, do, rtol=1e-12, atol=0)


@pytest.mark.parametrize("kernel", KERNELS)
def test_bmu_exact_ties_and_duplicates(pkg, oracle_port, kernel):
    """Duplicated codebook rows create exact FP64 ties: lowest index must win."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal((64, 50)).astype(np.float32)
    w = np.concatenate([base, base, base[::-1]], 0)  # every node has an exact twin
    x = np.concatenate([base + rng.standard_normal((64, 50)).astype(np.float32) * 0.1,
                        rng.standard_normal((4000, 50)).astype(np.float32)], 0)
    e = engine(pkg, w.shape[0], 50, kernel)
    e.set_codebook(w)
    b, _ = e.bmu(x)
    bo, _ = oracle_port.find_bmus(x, w)
    assert (b == bo).all()
    assert e.last_recheck_count >= x.shape[0]  # every row had an exact tie


@pytest.mark.parametrize("kernel", KERNELS)
def test_bmu_many_way_ties_full_rescan(pkg, oracle_port, kernel):
    """Eight identical nodes per cluster (> 4 candidates in one group) force the
    full exact re-scan path; indices must still match the reference."""
    rng = np.random.default_rng(9)
    centres = rng.standard_normal((40, 50)).astype(np.float32) * 3
    w = np.repeat(centres, 8, axis=0)  # 320 nodes: groups of 8 exact twins
    x = (centres[rng.integers(0, 40, 3000)] +
         0.2 * rng.standard_normal((3000, 50))).astype(np.float32)
    e = engine(pkg, w.shape[0], 50, kernel)
    e.set_codebook(w)
    b, d = e.bmu(x)
    bo, do = oracle_port.find_bmus(x, w)
    assert (b == bo).all()
    np.testing.assert_allclose(d, do, rtol=1e-12)


def test_golden_hot_path(pkg):
    """Reference outputs (tests/golden/hot_path.npz, made from oracle/_ref)."""
    g = np.load(os.path.join(GOLDEN, "hot_path.npz"))
    e = pkg.Engine(100, 50)
    e.set_codebook(g["w"])
    b, d = e.bmu(g["x"])
    assert (b == g["bmu"]).all()
    np.testing.assert_allclose(d, g["dist"], rtol=1e-12)
    e.bind(g["x"])
    e.set_influence(g["infl"])
    u, h, dist = e.epoch(float(g["eta"]), g["sel"], want_dist=True)
    scale = np.max(np.abs(g["u"]))
    assert np.max(np.abs(u - g["u"])) <= 1e-9 * scale
    np.testing.assert_allclose(h, g["h"], rtol=1e-9)
    np.testing.assert_allclose(dist, g["sel_dist"], rtol=1e-12)


# --- one epoch: accumulators ------------------------------------------------

@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("sampling", ["full", "random"])
def test_epoch_accumulators_vs_oracle(pkg, oracle_port, kernel, sampling):
    n, p = 30000, 256
    x = oracle_port.synth_gmm(n, 50, 2611)
    w = x[np.linspace(0, n - 1, p).astype(int)].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("hex", 16, 16), 4.0)
    if sampling == "full":
        sel = np.arange(n, dtype=np.uint32)
    else:
        sel = np.sort(np.random.default_rng(1).choice(n, n // 3, replace=False)).astype(np.uint32)
    e = engine(pkg, p, 50, kernel)
    e.bind(x)
    e.set_codebook(w)
    e.set_influence(infl)
    u, h, dist = e.epoch(0.45, sel, want_dist=True)
    uo, ho, _, _, do = oracle_port.run_iteration(x, sel, w, infl, 0.45, 1, 8)
    assert np.max(np.abs(u - uo)) <= 1e-9 * np.max(np.abs(uo))
    np.testing.assert_allclose(h, ho, rtol=1e-9)
    np.testing.assert_allclose(dist, do, rtol=1e-12)


@pytest.mark.parametrize("d", [50, 13])
@pytest.mark.parametrize("sampling", ["full", "random"])
def test_epoch_accumulators_multi_chunk(pkg, oracle_port, d, sampling):
    # K2 sorts rows by (chunk of 131072 rows, BMU): several chunks and a
    # ragged last one, async (even d) and generic (odd d) gathers
    n, p = 400_000 + 77, 256
    x = oracle_port.synth_gmm(n, d, 2612)
    w = x[np.linspace(0, n - 1, p).astype(int)].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("hex", 16, 16), 4.0)
    if sampling == "full":
        sel = np.arange(n, dtype=np.uint32)
    else:
        sel = np.sort(np.random.default_rng(2).choice(n, 300_001, replace=False)).astype(np.uint32)
    e = engine(pkg, p, d, 0)
    e.bind(x)
    e.set_codebook(w)
    e.set_influence(infl)
    u, h, dist = e.epoch(0.45, sel, want_dist=True)
    uo, ho, _, _, do = oracle_port.run_iteration(x, sel, w, infl, 0.45, 1, 8)
    assert np.max(np.abs(u - uo)) <= 1e-9 * np.max(np.abs(uo))
    np.testing.assert_allclose(h, ho, rtol=1e-9)
    np.testing.assert_allclose(dist, do, rtol=1e-12)
    qs, qc = e.qe(sel)
    assert qc == len(sel)
    assert qs == pytest.approx(float(np.sum(do)), rel=1e-12)


def test_streamed_equals_resident(pkg, oracle_port):
    n, p = 50000, 128
    x = oracle_port.synth_gmm(n, 50, 2612)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 16, 8), 3.0)
    out = []
    for streamed in (False, True):
        e = pkg.Engine(p, 50)
        from paper_2604_26555_b200 import _lib
        e.set_option(_lib.TSOM_OPT_STREAM_CHUNK, 7000)  # ragged chunks
        e.bind(x, streamed=streamed)
        e.set_codebook(w)
        e.set_influence(infl)
        sel = np.arange(1, n, 3, dtype=np.uint32)
        out.append(e.epoch(0.3, sel, want_dist=True))
    (u0, h0, d0), (u1, h1, d1) = out
    # same rows, same BMUs; only the grouping of the FP32 per-CTA partial sums differs
    assert np.max(np.abs(u0 - u1)) <= 1e-9 * np.max(np.abs(u0))
    np.testing.assert_allclose(h0, h1, rtol=1e-12)
    np.testing.assert_allclose(d0, d1, rtol=1e-14)


# --- error behaviour (the reference's exception types / messages) ----------

def test_errors(pkg):
    e = pkg.Engine(4, 2)
    e.bind(np.zeros((10, 2), np.float32))
    e.set_codebook(np.zeros((4, 2), np.float32))
    e.set_influence(np.eye(4))
    with pytest.raises(IndexError, match="fetch_rows: row index beyond data size"):
        e.epoch(0.1, np.array([3, 10], np.uint32))
    with pytest.raises(pkg.NumericalFault, match="numerical fault"):
        e.bind(np.full((10, 2), 3e6, np.float32))
        e.epoch(2.0)
    u, h, _ = e.epoch(0.1, np.array([], np.uint32))  # empty selection: zero accumulators
    assert not u.any() and not h.any()


# --- whole runs --------------------------------------------------------------

def test_resident_training_config1_shape(pkg, oracle_port):
    """Config-1 shape (10x10 rect, D=50, 10 epochs) on 20k rows vs the reference run."""
    g = np.load(os.path.join(GOLDEN, "config1_20k.npz"))
    x = oracle_port.synth_gmm(int(g["n"]), 50, int(g["seed"]))
    cfg = pkg.ResidentConfig(topology="rect", grid_w=10, grid_h=10, n_iters=10,
                             seed=int(g["seed"]))
    e = pkg.Engine(100, 50)
    e.bind(x)
    w0 = pkg.api.init_sample_draw(x, 100, cfg.seed)
    log = pkg.train_resident(cfg, e, w0, log_qe=True)
    w = e.get_codebook()
    assert rel_maxnorm(w, g["w"]) <= 1e-4
    qe = np.array([r["qe_train"] for r in log])
    np.testing.assert_allclose(qe, g["qe"], rtol=1e-5)


def gpu_qe(pkg, x, w):
    """quantization_error (metrics.hpp:28-30) of codebook w on rows x, on the GPU."""
    e = pkg.Engine(w.shape[0], w.shape[1])
    e.bind(x)
    e.set_codebook(w)
    s, c = e.qe()
    e.close()
    return s / c


DROPIN_CONFIGS = [
    dict(topology="hex", grid_w=4, grid_h=4, n_iters=8, seed=17),
    dict(topology="mst", nodes=16, n_iters=8, seed=17),
    dict(topology="rng", nodes=12, n_iters=6, seed=4, sampling="adaptive", rho=0.3),
    dict(topology="rect", grid_w=5, grid_h=3, n_iters=6, seed=23, sampling="random", rho=0.5,
         use_momentum=True, momentum=0.4),
]


@pytest.mark.parametrize("kw", DROPIN_CONFIGS, ids=lambda k: f"{k['topology']}")
def test_dropin_train_vs_golden(pkg, kw):
    """The reference loop + CudaExecutor vs the reference loop + SerialExecutor."""
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "train_runs.npz"))
    i = DROPIN_CONFIGS.index(kw)
    cfg = dropin.TrainConfig(**kw)
    w, qe, _, _ = dropin.train_cuda(cfg, g["x"], log_qe=True)
    assert rel_maxnorm(w, g[f"w{i}"]) <= 1e-4
    # the per-epoch QE above is the reference loop's own (host) mean_bmu_distance
    # (trainer.hpp:518); the trained codebook's QE on the GPU (tsom_qe):
    np.testing.assert_allclose(qe, g[f"qe{i}"], rtol=1e-5)
    np.testing.assert_allclose(gpu_qe(pkg, g["x"], w), g[f"qe{i}"][-1], rtol=1e-5)


def test_dropin_config1_run(pkg, oracle_port):
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "config1_20k.npz"))
    x = oracle_port.synth_gmm(int(g["n"]), 50, int(g["seed"]))
    cfg = dropin.TrainConfig(topology="rect", grid_w=10, grid_h=10, n_iters=10,
                             seed=int(g["seed"]))
    w, qe, _, _ = dropin.train_cuda(cfg, x, log_qe=True)
    assert rel_maxnorm(w, g["w"]) <= 1e-4
    np.testing.assert_allclose(qe, g["qe"], rtol=1e-5)
    np.testing.assert_allclose(gpu_qe(pkg, x, w), g["qe"][-1], rtol=1e-5)


# --- BASELINE-size properties (1e7 x 50, K = 1024) --------------------------

@pytest.mark.slow
def test_full_size_properties(pkg, oracle_port):
    n, p = 10_000_000, 1024
    e = pkg.Engine(p, 50)
    e.bind_synthetic_gmm(n, 2602)
    # codebook: 1024 rows of a host GMM sample (same centres)
    w = oracle_port.synth_gmm(p, 50, 2602) + np.float32(0.01)
    e.set_codebook(w)
    dist = pkg.api.lattice_dist("hex", 32, 32)
    infl = oracle_port.influence_from_dist(dist, 16.0)
    e.set_influence(infl)
    u, h, _ = e.epoch(0.5)
    assert np.isfinite(u).all() and np.isfinite(h).all()
    s, c = e.qe()
    assert c == n
    # checksum of checksums: sum_j H_j = sum_b c_b * sum_j h[b][j]
    b, _ = e.bmu_bound(None, want_dist=False)
    counts = np.bincount(b, minlength=p).astype(np.float64)
    assert counts.sum() == n
    np.testing.assert_allclose(h, infl.T @ counts, rtol=1e-9)
    np.testing.assert_allclose(h.sum(), (infl.sum(1) * counts).sum(), rtol=1e-9)
    # and H is the reference's quantised sum exactly: every term h[b][j] on the
    # 2^-40 grid (accum.hpp:34-42), c_b copies of it, summed in integers
    q = np.rint(infl * 2.0**40).astype(np.int64).astype(object)
    cb = counts.astype(np.int64).astype(object)
    hq = np.array([float(sum(cb[i] * q[i, j] for i in range(p) if cb[i])) for j in range(p)])
    assert np.array_equal(h, hq / 2.0**40)


def test_nccl_world1_allreduce_path(pkg, oracle_port):
    """The multi-GPU code path (dlopen NCCL, unique id, ncclCommInitRank, one
    allreduce per epoch) on a world-size-1 communicator: results must equal the
    communicator-free epoch."""
    n, p = 20000, 256
    x = oracle_port.synth_gmm(n, 50, 2670)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("hex", 16, 16), 3.0)
    out = []
    for comm in (False, True):
        e = pkg.Engine(p, 50)
        e.bind(x)
        if comm:
            e.comm_init(e.comm_unique_id(), 0, 1)
        e.set_codebook(w)
        e.set_influence(infl)
        out.append(e.epoch(0.4))
        e.set_topology_distance(oracle_port.lattice_dist("hex", 16, 16))
        e.train_epoch(0.4, 3.0)
        out.append((e.get_codebook(),))
    assert (out[0][0] == out[2][0]).all() and (out[0][1] == out[2][1]).all()
    assert (out[1][0] == out[3][0]).all()


# --- operand range: the FP16 encoding rescales by a power of two ------------

@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("scale", [1e-30, 1e-4, 1.0, 3e3, 1e18])
def test_bmu_exact_across_magnitudes(pkg, oracle_port, kernel, scale):
    rng = np.random.default_rng(int(abs(np.log10(scale))) + 17)
    x = (rng.standard_normal((3000, 50)) * scale).astype(np.float32)
    w = x[rng.choice(3000, 300, replace=False)] + (
        rng.standard_normal((300, 50)) * 0.1 * scale).astype(np.float32)
    e = engine(pkg, 300, 50, kernel)
    e.set_codebook(w)
    b, d = e.bmu(x)
    bo, do = oracle_port.find_bmus(x, w)
    assert (b == bo).all()
    np.testing.assert_allclose(d, do, rtol=1e-12, atol=0)


@pytest.mark.parametrize("kernel", KERNELS)
def test_bmu_exact_mixed_feature_scales(pkg, oracle_port, kernel):
    # features spanning 10 decades (the FP16 subnormal floor enters the window)
    rng = np.random.default_rng(5)
    col = np.logspace(-5, 5, 50).astype(np.float32)
    x = (rng.standard_normal((4000, 50)) * col).astype(np.float32)
    w = x[rng.choice(4000, 256, replace=False)].copy()
    e = engine(pkg, 256, 50, kernel)
    e.set_codebook(w)
    b, _ = e.bmu(x)
    bo, _ = oracle_port.find_bmus(x, w)
    assert (b == bo).all()


# --- tuning: run_study with GPU trials (tune.hpp:125-159) ---------------------

def test_run_study_cuda_matches_reference(pkg, oracle_port, oracle_ref):
    import oracle
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("drop-in library not built")
    x = oracle_port.synth_gmm(3000, 8, 41)
    train, holdout = x[:2400], x[2400:]
    base = oracle.SomConfig(topology="hex", grid_w=5, grid_h=4, n_iters=10, seed=0)
    seeds = [1, 2]
    rt, rh, rf = oracle_ref.run_study(base, 4, seeds, train, holdout)
    gt, gh, gf, _ = dropin.run_study_cuda(base, 4, seeds, train, holdout, concurrency=4)
    assert (gf == rf).all()
    ok = ~rf
    np.testing.assert_allclose(gt[ok], rt[ok], rtol=1e-5)
    np.testing.assert_allclose(gh[ok], rh[ok], rtol=1e-5)


@pytest.mark.parametrize("d", [1, 2, 17, 50, 62])
def test_split_row_image_equals_elementwise_split(pkg, oracle_port, d):
    # the row-image 3xFP16 split (k_split_rows_f16) against the element-wise
    # one (option 98): identical BMUs/distances, and both exact vs the oracle,
    # on resident (tiles split once) and gathered (sampled selection) rows
    from paper_2604_26555_b200 import _lib
    rng = np.random.default_rng(40 + d)
    n, p = 5000 + 37, 300
    x = (rng.normal(size=(n, d)) * rng.uniform(0.1, 10.0, size=d)).astype(np.float32)
    w = x[rng.choice(n, p, replace=False)].copy()
    sel = np.sort(rng.choice(n, n // 3, replace=False)).astype(np.uint32)
    out = {}
    for v1 in (0, 1):
        e = engine(pkg, p, d, 3)
        try:
            e.set_option(98, v1)
            e.set_codebook(w)
            b, dist = e.bmu(x)
            e.bind(x)
            e.set_influence(np.eye(p))
            u, h, _ = e.epoch(0.5, selected=sel)
            ua, ha, _ = e.epoch(0.5)
            out[v1] = (b, dist, u, h, ua, ha)
        finally:
            e.set_option(98, 0)
            e.close()
    ob, od = oracle_port.find_bmus(x, w)
    for v1 in (0, 1):
        assert np.array_equal(out[v1][0], ob)
        np.testing.assert_allclose(out[v1][1], od, rtol=1e-12)
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


def test_bind_reuses_pool_blocks_exactly(pkg, oracle_port):
    # engines reuse the device pool's blocks; a bind from pageable rows must be
    # complete before the engine's own stream reads them (regression: the
    # row-norm max once raced a plain cudaMemcpy and saw the previous engine's
    # data, shrinking the FP16 scale below the error model)
    def data(d, seed):
        rng = np.random.default_rng(seed)
        x = (rng.normal(size=(5037, d)) * rng.uniform(0.1, 10.0, size=d)).astype(np.float32)
        return x, x[rng.choice(5037, 300, replace=False)].copy()
    x0, w0 = data(60, 150)
    e = engine(pkg, 300, 60, 3)
    e.set_codebook(w0)
    e.bmu(x0)
    e.bind(x0)
    e.bmu_bound()
    e.close()
    x, w = data(62, 102)
    e = engine(pkg, 300, 62, 3)
    e.set_codebook(w)
    e.bmu(x)
    e.bind(x)
    b, _ = e.bmu_bound()
    e.close()
    ob, _ = oracle_port.find_bmus(x, w)
    assert np.array_equal(b, ob)


@pytest.mark.parametrize("owner", ["cudaMalloc", "torch"])
def test_bind_device_rows_exact(pkg, oracle_port, owner):
    # caller-owned device rows (tsom_bind_device_data): the K2 row windows may
    # read past the last row only when the allocation has room for it
    # (cuMemGetAddressRange); an exact-size cudaMalloc block and a torch
    # tensor, both against the oracle
    import torch
    n, p, d = 70_001, 256, 50
    x = oracle_port.synth_gmm(n, d, 2613)
    w = x[np.linspace(0, n - 1, p).astype(int)].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("hex", 16, 16), 4.0)
    torch.cuda.init()
    free = None
    if owner == "torch":
        keep = torch.from_numpy(x).cuda()
        ptr = keep.data_ptr()
    else:
        from cuda.bindings import runtime as rt
        err, ptr = rt.cudaMalloc(x.nbytes)
        assert err == rt.cudaError_t.cudaSuccess
        (err,) = rt.cudaMemcpy(ptr, x.ctypes.data, x.nbytes, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
        assert err == rt.cudaError_t.cudaSuccess
        free = (rt, ptr)
    try:
        e = engine(pkg, p, d, 0)
        e.bind_device(ptr, n)
        e.set_codebook(w)
        e.set_influence(infl)
        u, h, dist = e.epoch(0.45, None, want_dist=True)
        e.close()
    finally:
        if free:
            free[0].cudaFree(free[1])
    sel = np.arange(n, dtype=np.uint32)
    uo, ho, _, _, do = oracle_port.run_iteration(x, sel, w, infl, 0.45, 1, 8)
    assert np.max(np.abs(u - uo)) <= 1e-9 * np.max(np.abs(uo))
    np.testing.assert_allclose(h, ho, rtol=1e-9)
    np.testing.assert_allclose(dist, do, rtol=1e-12)


def test_pageable_bind_staging_and_gather_variants(pkg, oracle_port):
    # an 80 MB pageable bind goes through the multi-threaded pinned staging
    # (>= 64 MB); the epoch then runs with the TMA gather and with the cp.async
    # gather (option 97), both against the oracle
    from paper_2604_26555_b200 import _lib
    n, p, d = 400_000, 256, 50
    x = oracle_port.synth_gmm(n, d, 2614)
    assert x.nbytes >= 64 << 20
    w = x[np.linspace(0, n - 1, p).astype(int)].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("hex", 16, 16), 4.0)
    sel = np.sort(np.random.default_rng(3).choice(n, 150_001, replace=False)).astype(np.uint32)
    uo, ho, _, _, do = oracle_port.run_iteration(x, sel, w, infl, 0.45, 1, 8)
    e = engine(pkg, p, d, 0)
    try:
        e.bind(x)
        e.set_codebook(w)
        e.set_influence(infl)
        for kind in (0, 1):
            e.set_option(97, kind)
            u, h, dist = e.epoch(0.45, sel, want_dist=True)
            assert np.max(np.abs(u - uo)) <= 1e-9 * np.max(np.abs(uo))
            np.testing.assert_allclose(h, ho, rtol=1e-9)
            np.testing.assert_allclose(dist, do, rtol=1e-12)
    finally:
        e.set_option(97, 0)
        e.close()
    _lib.release_cached_memory(0)


@pytest.mark.parametrize("sampled", [False, True])
def test_train_epochs_equals_epoch_loop(pkg, oracle_port, sampled):
    # tsom_train_epochs (no host round trip between epochs) against the same
    # schedule through tsom_train_epoch one call at a time: identical codebooks
    n, p, d = 60_000, 64, 20
    x = oracle_port.synth_gmm(n, d, 2615)
    w0 = x[np.linspace(0, n - 1, p).astype(int)].copy()
    dist = oracle_port.lattice_dist("hex", 8, 8)
    etas = [0.5 - 0.04 * t for t in range(8)]
    sigmas = [3.0 - 0.3 * t for t in range(8)]
    out = []
    for multi in (False, True):
        e = pkg.Engine(p, d)
        e.bind(x)
        e.set_codebook(w0)
        e.set_topology_distance(dist)
        if sampled:
            e.sampler_init("adaptive", n // 10, 77)
        if multi:
            e.train_epochs(etas, sigmas, sampled=sampled)
        else:
            for eta, sig in zip(etas, sigmas):
                e.train_epoch(eta, sig, sampled=sampled)
        out.append(e.get_codebook())
        e.close()
    assert np.array_equal(out[0], out[1])


def test_train_epochs_reports_the_failing_epoch(pkg, oracle_port):
    # a schedule whose third epoch violates the accumulation-term guard: the
    # multi-epoch call names epoch 2, and the codebook is the one the
    # per-epoch loop leaves when it raises at the same epoch
    n, p, d = 20_000, 16, 8
    x = oracle_port.synth_gmm(n, d, 2616)
    w0 = x[np.linspace(0, n - 1, p).astype(int)].copy()
    dist = oracle_port.lattice_dist("rect", 4, 4)
    etas, sigmas = [0.5, 0.4, 1e7, 0.3], [2.0, 1.8, 1.6, 1.4]
    books = []
    for multi in (False, True):
        e = pkg.Engine(p, d)
        e.bind(x)
        e.set_codebook(w0)
        e.set_topology_distance(dist)
        if multi:
            with pytest.raises(pkg.NumericalFault, match=r"term out of range.*\(epoch 2\)"):
                e.train_epochs(etas, sigmas)
        else:
            e.train_epoch(etas[0], sigmas[0])
            e.train_epoch(etas[1], sigmas[1])
            with pytest.raises(pkg.NumericalFault, match="term out of range"):
                e.train_epoch(etas[2], sigmas[2])
        books.append(e.get_codebook())
        e.close()
    assert np.array_equal(books[0], books[1])


@pytest.mark.parametrize("kw", DROPIN_CONFIGS, ids=lambda k: f"{k['topology']}")
def test_train_device_vs_golden(pkg, kw):
    """toposom_b200::train_device (every step on the device) vs the reference loop +
    SerialExecutor: same bars as the drop-in loop."""
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "train_runs.npz"))
    i = DROPIN_CONFIGS.index(kw)
    cfg = dropin.TrainConfig(**kw)
    w, qe, ref, _ = dropin.train_device(cfg, g["x"], log_qe=True)
    assert rel_maxnorm(w, g[f"w{i}"]) <= 1e-4
    np.testing.assert_allclose(qe, g[f"qe{i}"], rtol=1e-5)
    # the refresh schedule is the reference's
    w2, _, ref2, _ = dropin.train_cuda(cfg, g["x"])
    assert np.array_equal(ref, ref2)


def test_train_device_config1(pkg, oracle_port):
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "config1_20k.npz"))
    x = oracle_port.synth_gmm(int(g["n"]), 50, int(g["seed"]))
    cfg = dropin.TrainConfig(topology="rect", grid_w=10, grid_h=10, n_iters=10,
                             seed=int(g["seed"]))
    w, _, _, _ = dropin.train_device(cfg, x)
    assert rel_maxnorm(w, g["w"]) <= 1e-4


def test_train_device_streamed_equals_resident(pkg):
    # the device loop over rows streamed from host memory every epoch gives the
    # codebook of the resident run
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    g = np.load(os.path.join(GOLDEN, "train_runs.npz"))
    cfg = dropin.TrainConfig(**DROPIN_CONFIGS[1])  # MST: refreshes on the device
    w_res, _, ref_res, _ = dropin.train_device(cfg, g["x"])
    w_str, _, ref_str, _ = dropin.train_device(cfg, g["x"], streamed=True)
    assert np.array_equal(ref_res, ref_str)
    assert rel_maxnorm(w_str, w_res.astype(np.float64)) <= 1e-6


@pytest.mark.parametrize("sampling", ["full", "random"])
def test_h_bit_identical_to_reference(pkg, oracle_port, sampling):
    """H is the reference's exactly: each term h[b][j] quantised to the 2^-40
    grid (quantize_term, accum.hpp:34-38), c_b copies summed in integers,
    dequantised once (accum.hpp:40-42) — so the H < 1e-12 freeze rule of
    apply_update (trainer.hpp:350) fires on the same nodes, including nodes
    whose every influence term is below 2^-41 (sigma at its 0.3 floor)."""
    n, p = 30000, 256
    x = oracle_port.synth_gmm(n, 50, 2740)
    w = x[np.linspace(0, n - 1, p).astype(int)].copy()
    dist = oracle_port.lattice_dist("hex", 16, 16)
    sel = None if sampling == "full" else np.sort(
        np.random.default_rng(1).choice(n, 7000, replace=False)).astype(np.uint32)
    ids = np.arange(n, dtype=np.uint32) if sel is None else sel
    for sigma in (4.0, 0.3):
        infl = oracle_port.influence_from_dist(dist, sigma)
        e = pkg.Engine(p, 50)
        e.bind(x)
        e.set_codebook(w)
        e.set_influence(infl)
        u, h, _ = e.epoch(0.4, sel)
        uo, ho, _, _, _ = oracle_port.run_iteration(x, ids, w, infl, 0.4, 1, 4)
        assert np.array_equal(h, ho), f"sigma {sigma}: {np.sum(h != ho)} H values differ"
        assert np.array_equal(h < 1e-12, ho < 1e-12)
        assert np.max(np.abs(u - uo)) <= 1e-9 * np.max(np.abs(uo))


@pytest.mark.parametrize("big,fails", [(2.0**23, True), (2.0**23 - 1.0, False)])
def test_term_guard_is_exact_at_the_boundary(pkg, oracle_port, big, fails):
    """quantize_term (accum.hpp:34-38) rejects |eta h (x - w)| >= 2^22.  Rows at
    0 with BMU node 0 and full influence on node 1 at `big` give the term
    -0.5 * big: exactly 2^22 (the reference throws) or 2^22 - 0.5 (it does
    not).  The engine's cheap norm bound (8.4e6) fails for both, so the exact
    per-node extremes test decides — the same way as the reference, for the
    accumulation pass (tsom_epoch) and for the device epoch, whose update a
    failure skips (the reference throws before apply_update)."""
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((64, 4)) * 1e-3).astype(np.float32)
    w = np.array([[0.0] * 4, [big] * 4], np.float32)
    infl = np.ones((2, 2))
    ref_fails = False
    try:
        oracle_port.run_iteration(x, np.arange(64, dtype=np.uint32), w, infl, 0.5, 1, 1)
    except oracle.OracleError as ex:
        ref_fails = ex.status == 2
    assert ref_fails == fails
    e = pkg.Engine(2, 4)
    e.bind(x)
    e.set_codebook(w)
    e.set_influence(infl)
    if fails:
        with pytest.raises(pkg.NumericalFault, match=r"accumulation term out of range"):
            e.epoch(0.5)
    else:
        e.epoch(0.5)
    e.set_topology_distance(np.zeros((2, 2)))  # influence exp(0) = 1 everywhere
    if fails:
        with pytest.raises(pkg.NumericalFault, match=r"accumulation term out of range"):
            e.train_epoch(0.5, 1.0)
        assert np.array_equal(e.get_codebook(), w)  # no update
        # a legal first epoch (node 1 at 2^21 moves to ~2^20), then eta = 8
        # makes the second epoch's terms ~2^23: the failure names epoch 1 and
        # leaves the weights after epoch 0
        e.set_codebook(w * 0.25)
        e.train_epoch(0.5, 1.0)
        w1 = e.get_codebook()
        e.set_codebook(w * 0.25)
        with pytest.raises(pkg.NumericalFault, match=r"\(epoch 1\)"):
            e.train_epochs([0.5, 8.0], [1.0, 1.0])
        assert np.array_equal(e.get_codebook(), w1)
    else:
        e.train_epoch(0.5, 1.0)
        assert not np.array_equal(e.get_codebook(), w)


def test_term_guard_cheap_bound_over_but_terms_small(pkg, oracle_port):
    """Large values close to each other: the norm bound (|eta| (||x|| + ||w||)
    = 7e6) exceeds 2^22 but every term is tiny — the reference accepts, and so
    must the engine (it used to raise here)."""
    rng = np.random.default_rng(1)
    x = (1e6 + rng.standard_normal((200, 50))).astype(np.float32)
    w = (1e6 + rng.standard_normal((16, 50))).astype(np.float32)
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 4, 4), 2.0)
    uo, ho, _, _, _ = oracle_port.run_iteration(x, np.arange(200, dtype=np.uint32), w, infl,
                                                0.5, 1, 1)
    e = pkg.Engine(16, 50)
    e.bind(x)
    e.set_codebook(w)
    e.set_influence(infl)
    u, h, _ = e.epoch(0.5)
    assert np.array_equal(h, ho)
