"""GPU topology refresh against the reference, bit for bit.

pairwise_sq_dists (topology.hpp:81-108), build_mst (:192-220), build_rng_graph
(:229-258), hop_distances (:292-325) on the device vs the oracle; then whole
device-resident training runs with MST / RNG topologies vs the reference's own
runs (test_oracle.py CONFIGS, golden train_runs.npz).
"""
import os
import time

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


def codebooks():
    rng = np.random.default_rng(3)
    yield "gmm", oracle.port.synth_gmm(300, 50, 2650)
    # integer lattice points: many exactly equal distances -> (w, i, j) tie-breaks
    g = np.stack(np.meshgrid(np.arange(8), np.arange(8)), -1).reshape(-1, 2).astype(np.float32)
    yield "grid", np.concatenate([g, np.zeros((64, 3), np.float32)], 1)
    yield "dups", np.repeat(rng.standard_normal((20, 6)).astype(np.float32), 3, axis=0)


@pytest.mark.parametrize("name,w", list(codebooks()), ids=lambda v: v if isinstance(v, str) else "")
def test_gram_graphs_hops_bit_exact(pkg, oracle_port, name, w):
    P, D = w.shape
    e = pkg.Engine(P, D)
    e.set_codebook(w)
    sq = e.pairwise_sq_dists()
    sq_ref = oracle_port.pairwise_sq_dists(w)
    assert (sq == sq_ref).all(), "FP64 Gram must match bit for bit"
    for kind in ("mst", "rng"):
        edges, hops = e.refresh_topology(kind, want_hops=True)
        eref = oracle_port.build_graph(kind, sq_ref)
        assert edges.shape == eref.shape and (edges == eref).all(), kind
        assert (hops == oracle_port.hop_distances(eref, P)).all(), kind


def k1024_codebooks():
    yield "gmm", oracle.port.synth_gmm(1024, 50, 2651)
    # a 32 x 32 integer grid in 2 of 50 dims: massive exact distance ties
    g = np.stack(np.meshgrid(np.arange(32), np.arange(32)), -1).reshape(-1, 2).astype(np.float32)
    yield "grid", np.concatenate([g, np.zeros((1024, 48), np.float32)], 1)
    # a trained-looking codebook: GMM rows pulled towards their component centres
    x = oracle.port.synth_gmm(1024, 50, 2652)
    c = oracle.port.synth_gmm(16, 50, 2652)
    yield "clustered", (0.9 * c[np.arange(1024) % 16] + 0.1 * x).astype(np.float32)


@pytest.mark.parametrize("name,w", list(k1024_codebooks()),
                         ids=lambda v: v if isinstance(v, str) else "")
def test_graphs_bit_exact_k1024(pkg, oracle_port, name, w):
    """The BASELINE topology size (1024 nodes): Gram, MST and RNG edge lists and
    hop counts bit-identical to the reference's (topology.hpp:81-325)."""
    import oracle as orc
    chk = orc.ref if orc.ref.available else oracle_port
    e = pkg.Engine(1024, 50)
    e.set_codebook(w)
    sq = e.pairwise_sq_dists()
    sq_ref = chk.pairwise_sq_dists(w)
    assert (sq == sq_ref).all()
    for kind in ("mst", "rng"):
        edges, hops = e.refresh_topology(kind, want_hops=True)
        eref = chk.build_graph(kind, sq_ref)
        assert edges.shape == eref.shape and (edges == eref).all(), kind
        assert (hops == chk.hop_distances(eref, 1024)).all(), kind


def test_refresh_timing_k1024(pkg, oracle_port):
    w = oracle_port.synth_gmm(1024, 50, 2651)
    e = pkg.Engine(1024, 50)
    e.set_codebook(w)
    for kind in ("mst", "rng"):
        e.refresh_topology(kind)  # warm
        t = time.perf_counter()
        edges, _ = e.refresh_topology(kind)
        dt = time.perf_counter() - t
        print(f"\n{kind}: {len(edges)} edges, device refresh {dt * 1e3:.1f} ms")
        assert dt < 2.0


def test_resident_mst_run_vs_reference(pkg):
    """CONFIGS[1] of test_oracle.py (MST, 16 nodes, 8 iterations) trained on the device."""
    g = np.load(os.path.join(GOLDEN, "train_runs.npz"))
    x = g["x"]
    cfg = pkg.ResidentConfig(topology="mst", graph_nodes=16, n_iters=8, seed=17)
    e = pkg.Engine(16, x.shape[1])
    e.bind(x)
    w0 = pkg.api.init_sample_draw(x, 16, 17)
    log = pkg.train_resident(cfg, e, w0, log_qe=True)
    w = e.get_codebook()
    rel = np.max(np.abs(w.astype(np.float64) - g["w1"])) / np.max(np.abs(g["w1"]))
    assert rel <= 1e-4
    np.testing.assert_allclose([r["qe_train"] for r in log], g["qe1"], rtol=1e-5)
    assert [int(r["refreshed"]) for r in log] == g["refresh1"].tolist()


@pytest.mark.parametrize("kind", ["rng", "mst"])
def test_resident_graph_run_vs_oracle(pkg, oracle_port, kind):
    x = oracle_port.synth_gmm(2000, 12, 2652)
    ocfg = oracle.SomConfig(topology=kind, nodes=36, n_iters=10, seed=9)
    wo, qeo, refo = oracle_port.train(ocfg, x, log_qe=True)
    cfg = pkg.ResidentConfig(topology=kind, graph_nodes=36, n_iters=10, seed=9)
    e = pkg.Engine(36, 12)
    e.bind(x)
    log = pkg.train_resident(cfg, e, pkg.api.init_sample_draw(x, 36, 9), log_qe=True)
    w = e.get_codebook()
    assert np.max(np.abs(w.astype(np.float64) - wo)) / np.max(np.abs(wo)) <= 1e-4
    np.testing.assert_allclose([r["qe_train"] for r in log], qeo, rtol=1e-5)
    assert [int(r["refreshed"]) for r in log] == refo.tolist()
