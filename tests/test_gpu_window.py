"""Evidence for the near-tie window that makes K1's BMUs exact.

K1 decides a row alone when its computed best and second-best values differ
by more than thr = tau (||x||^2 + max||w||^2) (+ an FP16-subnormal floor),
tau = 2^-14; closer rows are re-checked in exact FP64.  That is exact only if
|v / S - d2| < thr / 2 for every value K1 produces.  Here:

  * the raw K1 values of a whole main pass (option 99 bit 7 dump) against
    exact FP64 distances: the largest normalised error must stay below tau / 8
    (measured on the c2 workload: profiles/r02_k1_window.json);
  * rows whose exact top-2 gap is constructed at 0.5 ... 2 thr — the band where
    a too-small window would let K1's rounding pick the wrong node — across
    and within codebook groups, with the winner on either index side: every
    BMU must be the reference's (find_bmus, trainer.hpp:282-308).
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TAU = 2.0 ** -14


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


def k1_dump(pkg, e, n, P):
    import torch
    from paper_2604_26555_b200 import _lib
    L = _lib.load()
    L.tsom_debug_k1_dump.argtypes = [C.c_void_p]
    L.tsom_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
    L.tsom_debug_read.restype = C.c_int64
    gn = 256 if P >= 256 else (P + 31) // 32 * 32
    cols = (P + gn - 1) // gn * gn
    dump = torch.full((n, cols), float("nan"), dtype=torch.float32, device="cuda")
    assert L.tsom_debug_k1_dump(dump.data_ptr()) == 0
    e.set_option(99, 128)
    try:
        e.bmu_bound(None, want_dist=False)
    finally:
        e.set_option(99, 0)
        L.tsom_debug_k1_dump(None)
    sc = np.zeros(4, np.float32)
    L.tsom_debug_read(e.h, 3, sc.ctypes.data, 16)
    return dump[:, :P].cpu().numpy(), float(sc[1])


@pytest.mark.parametrize("kernel", [3, 2])
def test_k1_error_is_far_inside_the_window(pkg, oracle_port, kernel):
    from paper_2604_26555_b200 import _lib
    from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist
    n, P, D = 20000, 1024, 50
    x = oracle_port.synth_gmm(n, D, 2606)
    e = pkg.Engine(P, D)
    e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kernel)
    e.set_option(_lib.TSOM_OPT_ROW_ORDER, 0)  # raw dump is in position order
    e.bind(x)
    e.set_codebook(init_sample_draw(x, P, 2606))
    e.set_topology_distance(lattice_dist("hex", 32, 32))
    for t, (eta, sigma) in enumerate([(0.5, 16.0), (0.45, 14.5), (0.4, 13.0)]):
        v, S = k1_dump(pkg, e, n, P)
        w = e.get_codebook().astype(np.float64)
        xd = x.astype(np.float64)
        x2 = (xd * xd).sum(1)
        w2 = (w * w).sum(1)
        d2 = x2[:, None] + w2[None, :] - 2.0 * xd @ w.T
        err = np.abs(v / S - d2) / (x2[:, None] + w2.max())
        assert np.isfinite(v).all()
        assert err.max() < TAU / 8, f"epoch {t}: max error {err.max():.3e} vs tau {TAU:.3e}"
        e.train_epoch(eta, sigma)


def adversarial_case(seed, P=1024, D=50, per_pair=4):
    """Rows whose exact top-2 gap is f * thr, f in [0.5, 2): row x starts near
    node a and slides along the a-b axis, where the gap |x-b|^2 - |x-a|^2 is
    linear, to the wanted gap; every other row is mirrored through the
    midpoint so node b wins instead (the winner on either index side)."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((P, D)) * 3.0
    pairs = [(p, P - 1 - p) for p in range(0, P // 2, 2)]          # across groups
    pairs += [(p, p + 1) for p in range(1, P // 2, 8)]             # inside a group
    w2max = float((w * w).sum(1).max())
    rows = []
    for k, (a, b) in enumerate(pairs):
        ab = w[b] - w[a]
        for r in range(per_pair):
            u = rng.standard_normal(D)
            x = w[a] + u * (0.4 / np.linalg.norm(u))
            gap0 = float(((x - w[b]) ** 2).sum() - ((x - w[a]) ** 2).sum())
            # the window of the row where it will end up (|x|^2 changes little)
            thr = TAU * (float(((w[a] + w[b]) / 2) @ ((w[a] + w[b]) / 2)) + w2max)
            g = thr * 0.5 * 4.0 ** rng.random()  # [0.5, 2) thr
            x = x + (gap0 - g) / (2.0 * float(ab @ ab)) * ab
            if (k + r) % 2:
                x = w[a] + w[b] - x  # mirrored: b wins by the same gap
            rows.append(x)
    return np.asarray(rows, np.float32), w.astype(np.float32)


@pytest.mark.parametrize("kernel", [3, 2])
@pytest.mark.parametrize("seed", [1, 2])
def test_adversarial_top2_gaps_at_the_window(pkg, oracle_port, kernel, seed):
    from paper_2604_26555_b200 import _lib
    x, w = adversarial_case(seed)
    xd, wd = x.astype(np.float64), w.astype(np.float64)
    d2 = ((xd[:, None, :] - wd[None, :, :]) ** 2).sum(-1)
    srt = np.sort(d2, 1)
    gap = srt[:, 1] - srt[:, 0]
    thr = TAU * ((xd * xd).sum(1) + (wd * wd).sum(1).max())
    ratio = gap / thr
    assert ratio.min() < 0.9 and ratio.max() > 1.1  # the band straddles the window
    assert ((ratio > 0.3) & (ratio < 3.0)).mean() > 0.9
    e = pkg.Engine(w.shape[0], w.shape[1])
    e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kernel)
    e.set_codebook(w)
    b, dist = e.bmu(x)
    bo, do = oracle_port.find_bmus(x, w)
    assert (b == bo).all(), f"{(b != bo).sum()} BMUs differ at gap/thr in [{ratio.min():.2f}, {ratio.max():.2f}]"
    np.testing.assert_allclose(dist, do, rtol=1e-12)
    assert 0 < e.last_recheck_count < len(x)  # some rows decided in FP64, some by K1 alone
