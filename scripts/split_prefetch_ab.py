"""Diagnostics: the gathered split of a rho = 0.1 selection of 1e8 resident
rows with (option 92 = 1) and without (0) the L2 prefetch of each warp's next
chunk; bmu phase minus K1 = split + merge + near-tie path."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
rng = np.random.default_rng(0)
sel = np.sort(rng.choice(N, N // 10, replace=False)).astype(np.uint32)
e = tsom.Engine(1024, 50)
e.bind_synthetic_gmm(N, 2608, 16, 0)
e.set_codebook((rng.standard_normal((1024, 50)) * 2).astype(np.float32))
e.set_influence(np.eye(1024))
for rep in range(3):
    for pf in (0, 1, 2, 3):
        e.set_option(92, pf)
        ts = []
        for _ in range(4):
            e.epoch(0.0, sel)
            t = e.timing_detail()
            ts.append(t["bmu_ms"] - t["k1_ms"])
        print(f"prefetch={pf}: bmu - k1 {np.round(ts, 3).tolist()} ms", flush=True)
