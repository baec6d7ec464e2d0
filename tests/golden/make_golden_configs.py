"""Golden runs of the reference at the BASELINE configuration shapes (K = 1024,
D = 50) on a CPU-tractable N = 1e5 (SURVEY.md §8(c) "run parity"):

    c2: 32x32 hex lattice, full sampling          (c5 reuses it, streamed from shards)
    c3: MST graph, 1024 nodes, refreshed on the reference schedule
    c4: RNG graph, 1024 nodes, adaptive sampler rho = 0.1

Run in the build container (needs oracle/_ref):
    make -C oracle && python tests/golden/make_golden_configs.py
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

R = oracle.ref
assert R.available, "oracle/_ref/libtoposom_ref.so not built"
N, D = 100_000, 50
CASES = {
    "c2": (dict(topology="hex", grid_w=32, grid_h=32), 2606),
    "c3": (dict(topology="mst", nodes=1024), 2607),
    "c4": (dict(topology="rng", nodes=1024, sampling="adaptive", rho=0.1), 2608),
}
out = {}
for name, (kw, seed) in CASES.items():
    t = time.time()
    x = R.synth_gmm(N, D, seed)
    cfg = oracle.SomConfig(n_iters=10, seed=seed, n_threads=os.cpu_count() or 1, **kw)
    w, qe, ref = R.train(cfg, x, log_qe=True)
    out[f"{name}_w"], out[f"{name}_qe"], out[f"{name}_refresh"] = w, qe, ref
    out[f"{name}_seed"] = np.uint64(seed)
    print(f"{name}: {time.time() - t:.1f} s", flush=True)
out["n"] = np.uint64(N)
np.savez_compressed(os.path.join(HERE, "config_shapes_1e5.npz"), **out)
print("written", flush=True)
