"""Generate golden vectors from the reference itself (oracle/_ref, built from
/root/reference/proj/include by oracle/Makefile).  Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

The .npz files are committed so the GPU box (which has no /root/reference)
checks against the reference's own outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from test_oracle import CONFIGS  # noqa: E402

R = oracle.ref
assert R.available, "oracle/_ref/libtoposom_ref.so not built"

# 1. hot path on the SURVEY §8(d) Gaussian mixture, K=100 rect lattice (config 1 shape)
x = R.synth_gmm(4000, 50, 2601)
w = x[[int(i) for i in np.linspace(0, 3999, 100)]] + np.float32(0.125)
infl = R.influence_from_dist(R.lattice_dist("rect", 10, 10), 3.5)
sel = np.arange(0, 4000, 2, dtype=np.uint32)
b, d = R.find_bmus(x, w)
u, h, ur, hr, dist = R.run_iteration(x, sel, w, infl, 0.45, 1, 1)
np.savez_compressed(os.path.join(HERE, "hot_path.npz"), x=x, w=w, infl=infl, sel=sel,
                    eta=np.float64(0.45), bmu=b, dist=d, u=u, h=h, u_raw=ur, h_raw=hr,
                    sel_dist=dist)

# 2. whole training runs (lattice / MST / RNG+adaptive / rect+random+momentum)
xt = R.synth_gmm(300, 8, 2610)
out = {"x": xt}
for i, cfg in enumerate(CONFIGS):
    wt, qe, ref = R.train(cfg, xt, log_qe=True)
    out[f"w{i}"], out[f"qe{i}"], out[f"refresh{i}"] = wt, qe, ref
np.savez_compressed(os.path.join(HERE, "train_runs.npz"), **out)

# 3. config-1 shape training run (10x10 rect, D=50, 10 epochs) on 20k rows
xc = R.synth_gmm(20000, 50, 2601)
cfg = oracle.SomConfig(topology="rect", grid_w=10, grid_h=10, n_iters=10, seed=2601, n_threads=8)
wc, qec, _ = R.train(cfg, xc, log_qe=True)
np.savez_compressed(os.path.join(HERE, "config1_20k.npz"), w=wc, qe=qec, seed=np.uint64(2601),
                    n=np.uint64(20000))
print("golden vectors written")
