"""Where the host-facing paths spend their time (c2 shape, 1e7 x 50 rows).

- C-ABI tsom_bind_host_data(COPY) from pinned vs pageable rows, and the
  first epoch after a bind (one-time split + scratch allocation);
- the reference loop (train_with_executor + CudaExecutor, libtsom_dropin.so)
  split into executor construction (bind), run_iteration and the rest (the
  reference's own host code: sampler, influence, apply_update).
Prints one JSON line.  Usage: python scripts/bind_breakdown.py [n_rows]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import dropin  # noqa: E402
from paper_2604_26555_b200.hostref import lattice_dist  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    P, D = 1024, bench.D
    pinned = bench.host_gmm_rows(n, 7)
    pageable = np.array(pinned, copy=True)
    w0 = pageable[:P].copy()
    out = {"rows": n}
    dist = lattice_dist("hex", 32, 32)

    def cabi(rows, tag):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e = tsom.Engine(P, D)
        t1 = time.perf_counter()
        e.bind(rows)
        t2 = time.perf_counter()
        e.set_codebook(w0)
        e.set_topology_distance(dist)
        e.train_epoch(0.5, 8.0)
        t3 = time.perf_counter()
        e.train_epoch(0.4, 7.0)
        t4 = time.perf_counter()
        e.get_codebook()
        t5 = time.perf_counter()
        e.close()
        t6 = time.perf_counter()
        out[tag] = {"create_s": t1 - t0, "bind_s": t2 - t1, "first_epoch_s": t3 - t2,
                    "epoch_s": t4 - t3, "get_s": t5 - t4, "close_s": t6 - t5}

    cabi(pinned, "warm")
    for rep in range(2):
        cabi(pinned, f"pinned{rep}")
        cabi(pageable, f"pageable{rep}")
    if dropin.available():
        cfg = dropin.TrainConfig(topology="hex", grid_w=32, grid_h=32, n_iters=10, seed=7)
        for tag, rows in (("dropin_pageable", pageable), ("dropin_pinned", pinned)):
            _, _, _, (tot, ctor, it) = dropin.train_cuda(cfg, rows, profile=True)
            out[tag] = {"total_s": tot, "executor_ctor_s": ctor, "run_iteration_s": it,
                        "reference_host_s": tot - ctor - it}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
