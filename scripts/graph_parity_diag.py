"""Diagnostics: how far do graph-topology runs (c3 MST, c4 RNG) drift from the
reference's own runs, for the device-resident loop and for the drop-in loop."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import dropin  # noqa: E402

G = np.load("tests/golden/config_shapes_1e5.npz")
for name, kw, dkw in [("c3", dict(topology="mst", graph_nodes=1024), dict(topology="mst", nodes=1024)),
                      ("c4", dict(topology="rng", graph_nodes=1024, sampling="adaptive", rho=0.1),
                       dict(topology="rng", nodes=1024, sampling="adaptive", rho=0.1))]:
    seed = int(G[f"{name}_seed"])
    x = oracle.port.synth_gmm(int(G["n"]), 50, seed)
    ref_w, ref_qe = G[f"{name}_w"], G[f"{name}_qe"]
    e = tsom.Engine(1024, 50)
    e.bind(x)
    log = tsom.train_resident(tsom.ResidentConfig(n_iters=10, seed=seed, **kw), e,
                              tsom.api.init_sample_draw(x, 1024, seed), log_qe=True)
    w = e.get_codebook()
    qe = np.array([r["qe_train"] for r in log])
    rel = np.max(np.abs(w.astype(np.float64) - ref_w)) / np.max(np.abs(ref_w))
    print(name, "resident: codebook rel", f"{rel:.2e}", "qe rel per epoch",
          np.array2string(np.abs(qe - ref_qe) / ref_qe, precision=2), flush=True)
    cfg = dropin.TrainConfig(n_iters=10, seed=seed, **dkw)
    wd, qd, _, _ = dropin.train_cuda(cfg, x, log_qe=True)
    rel = np.max(np.abs(wd.astype(np.float64) - ref_w)) / np.max(np.abs(ref_w))
    print(name, "drop-in : codebook rel", f"{rel:.2e}", "qe rel per epoch",
          np.array2string(np.abs(qd - ref_qe) / ref_qe, precision=2), flush=True)

# which nodes deviate?  (resident path, c3)
name, kw = "c3", dict(topology="mst", graph_nodes=1024)
seed = int(G[f"{name}_seed"])
x = oracle.port.synth_gmm(int(G["n"]), 50, seed)
ref_w = G[f"{name}_w"]
e = tsom.Engine(1024, 50)
e.bind(x)
tsom.train_resident(tsom.ResidentConfig(n_iters=10, seed=seed, **kw), e,
                    tsom.api.init_sample_draw(x, 1024, seed))
w = e.get_codebook()
dev = np.max(np.abs(w.astype(np.float64) - ref_w), axis=1) / np.max(np.abs(ref_w))
b, _ = oracle.port.find_bmus(x, ref_w)
hits = np.bincount(b, minlength=1024)
order = np.argsort(-dev)
print("top deviating nodes (dev, bmu-hits):",
      [(int(j), f"{dev[j]:.1e}", int(hits[j])) for j in order[:12]])
print("max dev over nodes with >= 1 hit:", f"{dev[hits > 0].max():.2e}",
      " >= 10 hits:", f"{dev[hits >= 10].max():.2e}", " n empty:", int((hits == 0).sum()))
