"""Diagnostics: how many (128-row tile, 256-node group) pairs of K1 a
triangle-inequality bound could skip on the c2 workload with the rows in BMU
order.  For tile T (centroid c, radius r = max ||x - c||) and group g:
    L = min_{j in g} ||c - w_j|| - r  <=  min_{i in T, j in g} ||x_i - w_j||
and the pair is skippable when L > 0 and L^2 > U^2 (1 + 1e-3), U = max over
the tile of the row's exact best distance (an idealised upper bound: the real
one would come from the previous epoch's distance plus the BMU's move).
Printed per schedule epoch of the second cycle."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
host = bench.host_gmm_rows(n, bench.SEEDS["c2"])
e = tsom.Engine(1024, 50)
e.set_option(9, 0)
e.bind(host)
e.set_codebook(init_sample_draw(host, 1024, bench.SEEDS["c2"]))
e.set_topology_distance(lattice_dist("hex", 32, 32))
etas, sigmas = bench.hex_schedule(bench.EPOCHS)
e.train_epochs(etas, sigmas)
x = torch.from_numpy(np.asarray(host)).cuda().double()
b0, _ = e.bmu_bound(None, want_dist=False)
order = torch.from_numpy(np.argsort(b0, kind="stable").astype(np.int64)).cuda()
xs = x[order]
T = n // 128
xt = xs[: T * 128].view(T, 128, 50)
c = xt.mean(1)
r = (xt - c[:, None, :]).norm(dim=2).max(1).values
for t in range(10):
    e.train_epoch(etas[t], sigmas[t])
    w = torch.from_numpy(e.get_codebook()).cuda().double()
    b, d = e.bmu_bound(None, want_dist=True)
    best = torch.from_numpy(d).cuda()[order][: T * 128].view(T, 128)
    U = best.max(1).values
    dc = torch.cdist(c, w)  # T x 1024
    L = dc.view(T, 4, 256).min(2).values - r[:, None]
    skip = (L > 0) & (L * L > (U * U * (1 + 1e-3))[:, None])
    # the same with the stale order's tile of the previous epoch's BMU moved
    print(f"epoch {t} sigma {sigmas[t]:.1f}: skippable (tile, group) pairs {skip.float().mean().item():.3f}"
          f"  median r {r.median().item():.2f} U {U.median().item():.2f} "
          f"min-group L {L.min(1).values.median().item():.2f}", flush=True)
