"""Diagnostics: time K1 (main pass) with stages disabled (option 99: bit0 = no
epilogue math, bit1 = no MMAs) to see which stage bounds the kernel."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import lattice_dist  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
for kern in (3,):
    e = tsom.Engine(1024, 50)
    e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kern)
    e.bind_synthetic_gmm(N, 2606)
    rng = np.random.default_rng(0)
    e.set_codebook((rng.standard_normal((1024, 50)) * 3).astype(np.float32))
    e.set_topology_distance(lattice_dist("hex", 32, 32))
    for dbg in (0, 64, 1, 65, 4, 5, 6, 7):
        e.set_option(99, dbg)
        ts = []
        for _ in range(6):
            e.train_epoch(0.1, 3.0)
            ts.append(e.timing_detail()["k1_ms"])
        print(f"kernel={kern} dbg={dbg}: k1 {np.median(ts[1:]):.3f} ms", flush=True)
    e.set_option(99, 0)
    e.close()
