"""How contiguous K2's row batches are after the BMU-order re-layout: the c2
workload (1e7 x 50, 32x32 hex) trained epoch by epoch for two schedule
cycles with TSOM_OPT_ROW_ORDER 2 (one re-layout, at the second full pass);
after every epoch the per-position BMUs (debug buffer 10) are stable-sorted
as K2's counting sort does and cut into its pieces (<= 256 rows of one node)
and batches (32 rows).  Prints per epoch: the fraction of batches that are
one contiguous run (one bulk copy), the mean number of runs in the others,
and the fraction of rows in runs of >= 4.
Usage: python scripts/gather_runs_probe.py [n_rows]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist,  # noqa: E402
                                           resolved_sigma0, schedule_value)


def batch_stats(bmu, P):
    order = np.argsort(bmu, kind="stable").astype(np.int64)
    counts = np.bincount(bmu, minlength=P)
    starts = np.concatenate([[0], np.cumsum(counts)])
    # batch id of every sorted slot: node-local index // 32, offset by node
    local = np.arange(len(order)) - np.repeat(starts[:-1], counts)
    nb = (counts + 31) // 32
    boff = np.concatenate([[0], np.cumsum(nb)])
    bid = np.repeat(boff[:-1], counts) + local // 32
    brk = np.ones(len(order), bool)  # a run starts here
    brk[1:] = (order[1:] != order[:-1] + 1) | (bid[1:] != bid[:-1])
    runs_per_batch = np.bincount(bid, weights=brk, minlength=boff[-1])
    contig = runs_per_batch == 1
    run_id = np.cumsum(brk) - 1
    run_len = np.bincount(run_id)
    rows_in_long = run_len[run_len >= 4].sum() / len(order)
    return contig.mean(), runs_per_batch[~contig].mean() if (~contig).any() else 0.0, rows_in_long


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    P, D, seed = 1024, 50, 2606
    x = _lib.synth_gmm_host(n, D, seed)
    e = tsom.Engine(P, D)
    e.set_option(_lib.TSOM_OPT_ROW_ORDER, 2)
    e.bind(x)
    e.set_codebook(init_sample_draw(x, P, seed))
    e.set_topology_distance(lattice_dist("hex", 32, 32))
    L = _lib.load()
    L.tsom_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
    L.tsom_debug_read.restype = C.c_int64
    s0 = resolved_sigma0("hex", 32, 32)
    bmu = np.empty(n, np.uint32)
    for t in range(20):
        eta = schedule_value(0.5, "linear", t % 10, 10, 1e-4)
        sig = schedule_value(s0, "linear", t % 10, 10, 0.3)
        e.train_epoch(eta, sig)
        assert L.tsom_debug_read(e.h, 10, bmu.ctypes.data, bmu.nbytes) == bmu.nbytes
        c, r, lng = batch_stats(bmu, P)
        print(f"epoch {t:2d} sigma {sig:5.2f}: contiguous batches {c:.3f}, runs in the others "
              f"{r:5.1f}, rows in runs >= 4 {lng:.3f}", flush=True)


if __name__ == "__main__":
    main()
