import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
G = np.load("tests/golden/config_shapes_1e5.npz")
name, kw = "c4", dict(topology="rng", graph_nodes=1024, sampling="adaptive", rho=0.1)
seed = int(G[f"{name}_seed"])
x = oracle.port.synth_gmm(int(G["n"]), 50, seed)
ref_w = G[f"{name}_w"]
e = tsom.Engine(1024, 50)
e.bind(x)
tsom.train_resident(tsom.ResidentConfig(n_iters=10, seed=seed, **kw), e,
                    tsom.api.init_sample_draw(x, 1024, seed))
w = e.get_codebook()
dev = np.max(np.abs(w.astype(np.float64) - ref_w), axis=1) / np.max(np.abs(ref_w))
hits = np.bincount(oracle.port.find_bmus(x, ref_w)[0], minlength=1024)
order = np.argsort(-dev)
print([(int(j), f"{dev[j]:.1e}", int(hits[j])) for j in order[:20]])
for th in (1, 5, 10, 20, 50, 100):
    print(th, f"{dev[hits >= th].max():.2e}", int((hits >= th).sum()))
