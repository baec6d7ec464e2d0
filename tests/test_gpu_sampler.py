"""Device samplers (sampling.hpp:46-221) against the reference Sampler.

Bars: every selection identical to toposom::Sampler's for the same seed, over
successive epochs with the adaptive feedback; the adaptive state (last_error,
age) identical after the updates; a sampled device-resident run within the
usual whole-run tolerances of the reference run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


def engine_with_rows(pkg, n):
    e = pkg.Engine(4, 2)
    e.bind(np.zeros((n, 2), np.float32))
    return e


RANDOM_CASES = [  # (n, m, seed, iters)
    (1000, 100, 7, 6), (100_000, 10_000, 2604, 4), (5000, 4999, 3, 3), (3000, 3000, 5, 2),
    (1, 1, 11, 2), (200_000, 150_000, 13, 3), (70_001, 1, 17, 5),
]


@pytest.mark.parametrize("n,m,seed,iters", RANDOM_CASES)
def test_random_sampler_matches_reference(pkg, oracle_ref, n, m, seed, iters):
    ref = oracle_ref.sampler_run("random", n, seed, iters, m0=m, budget_fixed=True)
    e = engine_with_rows(pkg, n)
    e.sampler_init("random", m, seed)
    for t in range(iters):
        sel = e.sampler_select()
        assert len(sel) == len(ref[t])
        assert (sel == ref[t]).all(), f"epoch {t}: {np.count_nonzero(sel != ref[t])} ids differ"


ADAPTIVE_CASES = [  # (n, rho, m0, seed, iters, alpha, beta)
    (20_000, 0.1, 0, 11, 6, 1.0, 1.0), (5000, 0.5, 0, 19, 5, 0.5, 2.0),
    (1000, 1.0, 1000, 23, 3, 1.0, 1.0), (300_000, 0.05, 0, 2608, 4, 1.0, 1.0),
]


@pytest.mark.parametrize("n,rho,m0,seed,iters,alpha,beta", ADAPTIVE_CASES)
def test_adaptive_sampler_matches_reference(pkg, oracle_ref, n, rho, m0, seed, iters, alpha,
                                            beta):
    dist = np.random.default_rng(seed).random(n) * 10.0
    fixed = m0 > 0
    ref = oracle_ref.sampler_run("adaptive", n, seed, iters, rho=rho, m0=m0, budget_fixed=fixed,
                                 alpha=alpha, beta=beta, dist_by_row=dist)
    m = m0 if fixed else max(1, int(np.floor(n * rho)))
    e = engine_with_rows(pkg, n)
    e.sampler_init("adaptive", m, seed, alpha, beta)
    err = np.full(n, 1e30)
    age = np.zeros(n, np.uint32)
    for t in range(iters):
        sel = e.sampler_select()
        assert (sel == ref[t]).all(), f"epoch {t}: {np.count_nonzero(sel != ref[t])} ids differ"
        e.sampler_observe(dist[sel])
        age += 1  # update_adaptive (sampling.hpp:143-157)
        err[sel] = dist[sel]
        age[sel] = 0
    ge, ga = e.sampler_state()
    assert (ge == err).all() and (ga == age).all()


def test_sampler_errors(pkg):
    e = engine_with_rows(pkg, 10)
    with pytest.raises(pkg.InvalidArgument, match="m must be >= 1"):
        e.sampler_init("random", 0, 1)
    with pytest.raises(pkg.InvalidArgument, match="unknown sampling kind"):
        e.sampler_init(5, 1, 1)


@pytest.mark.parametrize("sampling,rho", [("adaptive", 0.3), ("random", 0.4)])
def test_sampled_resident_training_vs_reference(pkg, oracle_port, oracle_ref, sampling, rho):
    import oracle
    x = oracle_port.synth_gmm(6000, 8, 31)
    cfg = oracle.SomConfig(topology="hex", grid_w=6, grid_h=5, n_iters=8, seed=31,
                           sampling=sampling, rho=rho)
    w_ref, qe_ref, _ = oracle_ref.train(cfg, x, log_qe=True)
    rc = pkg.ResidentConfig(topology="hex", grid_w=6, grid_h=5, n_iters=8, seed=31,
                            sampling=sampling, rho=rho)
    e = pkg.Engine(30, 8)
    e.bind(x)
    w0 = pkg.api.init_sample_draw(x, 30, cfg.seed)
    log = pkg.train_resident(rc, e, w0, log_qe=True)
    w = e.get_codebook()
    rel = float(np.max(np.abs(w.astype(np.float64) - w_ref)) / np.max(np.abs(w_ref)))
    assert rel <= 1e-4
    qe = np.array([r["qe_train"] for r in log])
    np.testing.assert_allclose(qe, qe_ref, rtol=1e-5)
