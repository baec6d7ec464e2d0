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


# --- sharded sampler: one reference Sampler over the ranks' rows --------------
#
# Ranks are engines on the same GPU driven from separate threads, joined by an
# in-process loopback group standing in for the NCCL communicator (the sampler
# calls the same allreduce hook either way): the concatenation of the ranks'
# selections must be the reference Sampler's selection over all rows.

def _run_sharded(pkg, sizes, kind, m, seed, iters, alpha=1.0, beta=1.0, dist=None):
    import threading

    world = len(sizes)
    g = pkg.RankGroup(world)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    engines = [engine_with_rows(pkg, s) for s in sizes]
    for r, e in enumerate(engines):
        e.join_group(g, r)
    out = [[None] * iters for _ in range(world)]
    errors = []

    def rank_main(r):
        try:
            e = engines[r]
            e.sampler_init(kind, m, seed, alpha, beta)
            for t in range(iters):
                sel = e.sampler_select()
                out[r][t] = sel.astype(np.int64) + offs[r]
                if dist is not None:
                    e.sampler_observe(dist[out[r][t]])
        except Exception as ex:  # pragma: no cover - reported below
            errors.append(ex)

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    g.close()
    assert not errors, errors
    return [np.concatenate([out[r][t] for r in range(world)]) for t in range(iters)], engines


@pytest.mark.parametrize("sizes", [[12000, 9000, 9001], [1, 29999], [15000, 15000, 3]])
def test_sharded_random_sampler_matches_reference(pkg, oracle_ref, sizes):
    n, m, seed = sum(sizes), 3000, 29
    ref = oracle_ref.sampler_run("random", n, seed, 4, m0=m, budget_fixed=True)
    got, _ = _run_sharded(pkg, [s for s in sizes if s > 0], "random", m, seed, 4)
    for t in range(4):
        assert (got[t] == ref[t]).all(), f"epoch {t}"


@pytest.mark.parametrize("sizes,alpha,beta", [([12000, 9000, 9001], 1.0, 1.0),
                                              ([20000, 10000], 0.5, 2.0), ([7, 29993], 1.0, 1.0)])
def test_sharded_adaptive_sampler_matches_reference(pkg, oracle_ref, sizes, alpha, beta):
    n, seed, iters = sum(sizes), 37, 5
    rho = 0.1
    m = max(1, int(np.floor(n * rho)))
    dist = np.random.default_rng(seed).random(n) * 10.0
    ref = oracle_ref.sampler_run("adaptive", n, seed, iters, rho=rho, alpha=alpha, beta=beta,
                                 dist_by_row=dist)
    got, engines = _run_sharded(pkg, sizes, "adaptive", m, seed, iters, alpha, beta, dist)
    for t in range(iters):
        assert (got[t] == ref[t]).all(), f"epoch {t}: {len(got[t])} vs {len(ref[t])}"
    # the per-rank adaptive state is the reference's, sliced
    err = np.full(n, 1e30)
    age = np.zeros(n, np.uint32)
    for t in range(iters):
        age += 1
        err[ref[t]] = dist[ref[t]]
        age[ref[t]] = 0
    off = 0
    for e, s in zip(engines, sizes):
        ge, ga = e.sampler_state()
        assert (ge == err[off:off + s]).all() and (ga == age[off:off + s]).all()
        off += s


def test_sampler_with_nccl_communicator_world1(pkg, oracle_ref):
    # the NCCL allreduce hook of the sharded sampler (one rank)
    n, seed = 20000, 43
    dist = np.random.default_rng(seed).random(n)
    ref = oracle_ref.sampler_run("adaptive", n, seed, 3, rho=0.2, dist_by_row=dist)
    e = engine_with_rows(pkg, n)
    e.comm_init(e.comm_unique_id(), 0, 1)
    e.sampler_init("adaptive", int(n * 0.2), seed)
    for t in range(3):
        sel = e.sampler_select()
        assert (sel == ref[t]).all()
        e.sampler_observe(dist[sel])
