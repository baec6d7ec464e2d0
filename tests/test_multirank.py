"""Multi-rank (data-parallel) host logic on CPU with gloo, world size 2.

The engine's N>1 path: each rank reduces its own row shard to
the packed sums [S_b | c_b | sum dist | rows], one allreduce(sum) combines
them, and every rank runs the identical FP64 smoothing.  Here the per-rank K2
sums are restated in numpy from the oracle's BMUs, combined with a real gloo
allreduce, smoothed with the K3 algebra, and compared with the single-process
reference accumulators.
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
