"""Diagnostics: BMU runs in storage order on the c2 workload after the
re-layout — runs per 256-row chunk (a run = consecutive rows with one BMU)
through two schedule cycles (the layout is from the warm-up's second epoch)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist  # noqa: E402

n = 10_000_000
host = bench.host_gmm_rows(n, bench.SEEDS["c2"])
e = tsom.Engine(1024, 50)
e.bind(host)
e.set_codebook(init_sample_draw(host, 1024, bench.SEEDS["c2"]))
e.set_topology_distance(lattice_dist("hex", 32, 32))
etas, sigmas = bench.hex_schedule(bench.EPOCHS)
import ctypes as C  # noqa: E402
L = _lib.load()
L.tsom_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
L.tsom_debug_read.restype = C.c_int64
buf = np.empty(n, np.uint32)
for cyc in range(3):
    for t in range(10):
        e.train_epoch(etas[t], sigmas[t])
        if t % 3 == 0 or t == 9:
            # the engine's own per-position BMUs (storage order): diagnostics read
            L.tsom_debug_read(e.h, 10, buf.ctypes.data, n * 4)
            br = np.concatenate([[True], buf[1:] != buf[:-1]])
            runs = br[: n // 256 * 256].reshape(-1, 256).sum(1)
            print(f"cycle {cyc} epoch {t}: runs/chunk mean {runs.mean():.2f} p50 {np.median(runs):.0f} "
                  f"p99 {np.percentile(runs, 99):.0f} max {runs.max()} total {br.sum()}", flush=True)
