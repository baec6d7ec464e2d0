"""Multi-rank (data-parallel) host logic on CPU (no GPU in this container).

The engine's N>1 path: each rank reduces its own row shard to
the packed sums [S_b | c_b | sum dist | rows], one allreduce(sum) combines
them, and every rank runs the identical FP64 smoothing.  The engine itself
runs that path with 2/3/4 ranks on the GPU (tests/test_gpu_multirank.py).
Here, on CPU: (1) the decomposition with a real gloo allreduce at world size
2 — per-rank K2 sums restated in numpy from the oracle's BMUs, smoothed with
the K3 algebra, against the single-process reference accumulators; (2) the
engine library's in-process rank group (the reduce the multi-rank epoch
calls), driven from threads without an engine: rank-ordered f64 sums and the
barrier deadline.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2604_26555_b200.hostref import assign_shards


def test_assign_shards_matches_reference():
    # test_parallel.cpp:78-85
    assert assign_shards(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert assign_shards(9, 3) == [(0, 3), (3, 6), (6, 9)]
    assert assign_shards(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert assign_shards(0, 2) == [(0, 0), (0, 0)]
    with pytest.raises(ValueError):
        assign_shards(5, 0)


def shard_sums(x, w, bmu):
    """K2 restated: row sums S_b = sum x_i, counts c_b (FP64)."""
    P, D = w.shape
    S = np.zeros((P, D))
    np.add.at(S, bmu, x.astype(np.float64))
    c = np.bincount(bmu, minlength=P).astype(np.float64)
    return np.concatenate([S.ravel(), c, [0.0, float(len(bmu))]])


def smooth(sums, w, infl, eta):
    """K3 restated: U = eta (h^T S - w H); H = h^T c."""
    P, D = w.shape
    S = sums[:P * D].reshape(P, D)
    c = sums[P * D:P * D + P]
    H = infl.T @ c
    U = eta * (infl.T @ S - w.astype(np.float64) * H[:, None])
    return U, H


def _worker(rank, world, port, path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    g = np.load(path)
    x, w, infl, eta = g["x"], g["w"], g["infl"], float(g["eta"])
    lo, hi = assign_shards(x.shape[0], world)[rank]
    bmu, _ = oracle.port.find_bmus(x[lo:hi], w)
    local = torch.from_numpy(shard_sums(x[lo:hi], w, bmu.astype(np.int64)))
    dist.all_reduce(local)  # the engine's single ncclAllReduce(sum, f64)
    U, H = smooth(local.numpy(), w, infl, eta)
    np.savez(path + f".rank{rank}.npz", U=U, H=H, rows=local.numpy()[-1])
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_epoch_equals_single_process(tmp_path, world):
    P = oracle.port
    x = P.synth_gmm(3001, 12, 2633)  # odd size: ragged shards
    w = x[np.linspace(0, 3000, 36).astype(int)] + np.float32(0.1)
    infl = P.influence_from_dist(P.lattice_dist("hex", 6, 6), 2.0)
    eta = 0.35
    path = str(tmp_path / "inp.npz")
    np.savez(path, x=x, w=w, infl=infl, eta=np.float64(eta))
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    uo, ho, _, _, _ = P.run_iteration(x, np.arange(3001, dtype=np.uint32), w, infl, eta, 1, 1)
    outs = [np.load(path + f".rank{r}.npz") for r in range(world)]
    for o in outs:  # every rank holds the identical, globally reduced result
        assert o["rows"] == 3001
        assert np.max(np.abs(o["U"] - uo)) <= 1e-9 * np.max(np.abs(uo))
        np.testing.assert_allclose(o["H"], ho, rtol=1e-9)
    assert (outs[0]["U"] == outs[1]["U"]).all()


# --- the in-process rank group's reduce (host logic, no GPU) ------------------
#
# tsom_group_* is the reduce the engine's multi-rank epoch uses when its ranks
# are threads of one process (tests/test_gpu_multirank.py drives it through
# the engines on a GPU).  Its host side is checked here directly: the reduce
# is evaluated in rank order whatever the arrival order (parallel.hpp:90-95,
# so every rank and every run gets the same f64 sums), and a rank that misses
# the deadline is named (collect_with_barrier, parallel.hpp:67-86).

def _group_lib():
    import ctypes as C

    from paper_2604_26555_b200 import _lib
    L = _lib.load()
    L.tsom_debug_group_reduce.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_int,
                                          C.c_double]
    L.tsom_debug_group_reduce.restype = C.c_int
    return L


def _reduce_on_threads(world, bufs, op, timeout_s=10.0, skip=(), delays=None):
    import threading
    import time

    from paper_2604_26555_b200 import RankGroup
    L = _group_lib()
    g = RankGroup(world)
    rc = [None] * world

    def rank(r):
        if delays:
            time.sleep(delays[r])
        rc[r] = L.tsom_debug_group_reduce(g.h, r, bufs[r].ctypes.data, bufs[r].nbytes, op,
                                          timeout_s)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world) if r not in skip]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    g.close()
    return rc


@pytest.mark.parametrize("world", [2, 3, 4])
def test_group_f64_reduce_is_rank_ordered(world):
    rng = np.random.default_rng(world)
    vals = [rng.standard_normal(4099) * 10.0 ** rng.integers(-8, 8, 4099) for _ in range(world)]
    want = vals[0].copy()
    for r in range(1, world):
        want = want + vals[r]  # left fold in rank order
    for delays in ([0.0] * world, [0.02 * (world - r) for r in range(world)]):
        bufs = [v.copy() for v in vals]
        rc = _reduce_on_threads(world, bufs, 3, delays=delays)
        assert rc == [-1] * world
        for b in bufs:
            assert (b == want).all()  # bit-identical on every rank, any arrival order


def test_group_integer_reduces():
    a = [np.array([1, 2, 3, 2**31], np.uint32), np.array([5, 6, 7, 2**31 - 1], np.uint32)]
    rc = _reduce_on_threads(2, a, 0)
    assert rc == [-1, -1] and a[0].tolist() == [6, 8, 10, 2**32 - 1] and (a[0] == a[1]).all()
    m = [np.array([3, 9, 2**63], np.uint64), np.array([7, 1, 5], np.uint64),
         np.array([0, 4, 6], np.uint64)]
    rc = _reduce_on_threads(3, m, 1)
    assert rc == [-1] * 3 and m[2].tolist() == [7, 9, 2**63]
    s = [np.array([2**40, 1], np.uint64), np.array([2**40, 2], np.uint64)]
    _reduce_on_threads(2, s, 2)
    assert s[1].tolist() == [2**41, 3]


def test_group_deadline_names_the_late_rank():
    import time
    bufs = [np.zeros(8) for _ in range(3)]
    t0 = time.perf_counter()
    rc = _reduce_on_threads(3, bufs, 3, timeout_s=0.2, skip=(1,))
    assert time.perf_counter() - t0 < 5.0
    # one waiting rank names worker 1, the other sees the broken barrier
    assert sorted(rc[r] for r in (0, 2)) == [-2, 1]
