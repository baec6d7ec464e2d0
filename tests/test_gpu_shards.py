"""Out-of-core input from FSOMSHRD shard files (dataset.hpp:171-344), §8(f) row 3.

The engine reads the shard files itself (tsom_bind_shards): TSOM_BIND_COPY
loads them once into HBM, TSOM_BIND_STREAMED preads each epoch's chunks into
pinned staging overlapped with the GPU work.  Bars: a shard-bound epoch equals
the in-memory epoch (BMUs/distances exact, U/H within 1e-9 of max|U| for the
streamed grouping); header errors keep the reference's messages.
"""
import os
import struct

import numpy as np
import pytest

from paper_2604_26555_b200 import shards

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2604_26555_b200 as p
    return p


def _epoch(pkg, bind, x_shape, w, infl, sel, chunk=None, register=True):
    from paper_2604_26555_b200 import _lib
    e = pkg.Engine(w.shape[0], w.shape[1])
    e.set_option(_lib.TSOM_OPT_HOST_REGISTER, int(register))
    if chunk:
        e.set_option(_lib.TSOM_OPT_STREAM_CHUNK, chunk)
    bind(e)
    assert e.rows == x_shape[0]
    e.set_codebook(w)
    e.set_influence(infl)
    out = e.epoch(0.3, sel, want_dist=True)
    return out, e.qe()


@pytest.mark.parametrize("streamed", [False, True])
def test_shard_epoch_equals_in_memory(pkg, oracle_port, tmp_path, streamed):
    n, p = 41000, 128
    x = oracle_port.synth_gmm(n, 50, 2613)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 16, 8), 3.0)
    # uneven shards, including an empty one; chunks straddle shard boundaries
    paths = []
    for i, (a, b) in enumerate([(0, 9000), (9000, 9000), (9000, 23011), (23011, n)]):
        pth = str(tmp_path / f"part-{i:05d}.shard")
        shards.write_one_shard(pth, x[a:b])
        paths.append(pth)
    sel = np.arange(2, n, 3, dtype=np.uint32)
    (u0, h0, d0), qe0 = _epoch(pkg, lambda e: e.bind(x), x.shape, w, infl, sel)
    (u1, h1, d1), qe1 = _epoch(pkg, lambda e: e.bind_shards(paths, streamed=streamed), x.shape,
                               w, infl, sel, chunk=7000)
    np.testing.assert_array_equal(d0, d1)
    if streamed:
        assert np.max(np.abs(u0 - u1)) <= 1e-9 * np.max(np.abs(u0))
        np.testing.assert_allclose(h0, h1, rtol=1e-12)
        np.testing.assert_allclose(qe0[0], qe1[0], rtol=1e-12)
    else:  # identical HBM image -> identical results
        np.testing.assert_array_equal(u0, u1)
        np.testing.assert_array_equal(h0, h1)
        assert qe0 == qe1


def test_pageable_streamed_source(pkg, oracle_port):
    """Streamed caller memory that is not page-locked goes through pinned staging."""
    n, p = 30000, 64
    x = oracle_port.synth_gmm(n, 50, 2614)
    w = x[:p].copy()
    infl = oracle_port.influence_from_dist(oracle_port.lattice_dist("rect", 8, 8), 2.0)
    (u0, h0, d0), _ = _epoch(pkg, lambda e: e.bind(x), x.shape, w, infl, None)
    (u1, h1, d1), _ = _epoch(pkg, lambda e: e.bind(x, streamed=True), x.shape, w, infl, None,
                             chunk=4096, register=False)
    np.testing.assert_array_equal(d0, d1)
    assert np.max(np.abs(u0 - u1)) <= 1e-9 * np.max(np.abs(u0))


def test_shard_header_errors(pkg, tmp_path):
    good = np.ones((5, 4), np.float32)
    e = pkg.Engine(4, 4)
    p = str(tmp_path / "bad-magic.shard")
    with open(p, "wb") as f:
        f.write(b"NOTASHRD" + bytes(16))
    with pytest.raises(RuntimeError, match="not a shard file \\(bad magic\\)"):
        e.bind_shards([p])
    p = str(tmp_path / "ver.shard")
    with open(p, "wb") as f:
        f.write(struct.pack("<8sIQI", b"FSOMSHRD", 2, 5, 4) + good.tobytes())
    with pytest.raises(RuntimeError, match="unsupported shard version 2"):
        e.bind_shards([p])
    p = str(tmp_path / "short.shard")
    with open(p, "wb") as f:
        f.write(b"FSOMSHRD" + struct.pack("<I", 1))
    with pytest.raises(RuntimeError, match="truncated shard header"):
        e.bind_shards([p])
    p = str(tmp_path / "trunc.shard")
    with open(p, "wb") as f:
        f.write(struct.pack("<8sIQI", b"FSOMSHRD", 1, 5, 4) + good.tobytes()[:-4])
    with pytest.raises(RuntimeError, match="truncated or corrupt shard"):
        e.bind_shards([p], streamed=False)
    p = str(tmp_path / "cols.shard")
    shards.write_one_shard(p, np.ones((5, 3), np.float32))
    with pytest.raises(RuntimeError, match="shard column count mismatch"):
        e.bind_shards([p])
    with pytest.raises(RuntimeError, match="cannot open shard"):
        e.bind_shards([str(tmp_path / "missing.shard")])
    # the engine stays usable after a failed bind
    p = str(tmp_path / "ok.shard")
    shards.write_one_shard(p, good)
    e.bind_shards([p])
    assert e.rows == 5


@pytest.mark.parametrize("streamed", [False, True])
def test_dropin_train_from_shard_dir(pkg, oracle_port, tmp_path, streamed):
    """train_with_executor over open_shards(dir) + CudaExecutor == over the matrix."""
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    x = oracle_port.synth_gmm(20000, 50, 2615)
    dropin.write_shards(x, str(tmp_path), 3)  # the reference's own writer
    cfg = dropin.TrainConfig(topology="hex", grid_w=8, grid_h=8, n_iters=6, seed=5)
    w0, qe0, _, _ = dropin.train_cuda(cfg, x, log_qe=True)
    w1, qe1, _, _ = dropin.train_cuda_shards(cfg, str(tmp_path), 50, log_qe=True,
                                             streamed=streamed)
    assert np.max(np.abs(w0.astype(np.float64) - w1)) <= 1e-5 * np.max(np.abs(w0))
    np.testing.assert_allclose(qe0, qe1, rtol=1e-6)
