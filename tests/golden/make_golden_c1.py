"""Golden run of BASELINE config c1 in full, from the reference itself
(oracle/_ref): 10x10 rectangular lattice, 100,000 x 50 Gaussian-mixture rows
(seed 2604 + 1), 10 epochs, eta0 0.5 linear, sigma0 auto,
full sampling, sample_draw init.  Run in the build container:

    make -C oracle && python tests/golden/make_golden_c1.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

R = oracle.ref
assert R.available, "oracle/_ref/libtoposom_ref.so not built"
seed, n = 2605, 100_000
x = R.synth_gmm(n, 50, seed)
cfg = oracle.SomConfig(topology="rect", grid_w=10, grid_h=10, n_iters=10, seed=seed,
                       n_threads=os.cpu_count() or 1)
w, qe, ref = R.train(cfg, x, log_qe=True)
np.savez_compressed(os.path.join(HERE, "config1_1e5.npz"), w=w, qe=qe, refresh=ref,
                    seed=np.uint64(seed), n=np.uint64(n))
print("config1_1e5.npz written", qe)
