"""A small workload that touches every kernel of the engine once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  * K1 tcgen05 main + enumerate passes (3xFP16 and 3xTF32), merges, the exact
    re-scan (duplicate nodes), the SIMT kernel, the split kernels;
  * K2 counting sort + TMA row gather (padded and packed rows), piece reduce;
  * K3 smoothing, apply_update, influence, the term guard (cheap path and the
    exact extremes path), the device sampler (random + adaptive, with
    observe), topology refresh (MST + RNG), a streamed epoch, a 2-rank group
    epoch;
  * the BMU-order re-layout (k_order.cu: permute, inverse, id mapping,
    scatter back), K1's chunk-skipping epilogue, K2's contiguous-batch copies,
    and the split image with K1's gather4 mode (multicast over the cluster).

Usage: compute-sanitizer --tool racecheck python scripts/sanitize_target.py
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import lattice_dist  # noqa: E402

P, D, n = 300, 50, 6000
x = _lib.synth_gmm_host(n, D, 11)
w = x[np.linspace(0, n - 1, P).astype(int)].copy()
w[1] = w[0]  # exact duplicates: near-ties for the rows of node 0
dist = np.abs(np.subtract.outer(np.arange(P), np.arange(P))).astype(np.float64)

for kernel in (3, 2, 1):
    e = tsom.Engine(P, D)
    e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kernel)
    e.bind(x)
    e.set_codebook(w)
    e.set_topology_distance(dist)
    e.train_epoch(0.5, 4.0)
    e.bmu(x[:700])
    sel = np.arange(0, n, 3, dtype=np.uint32)
    e.set_influence(np.exp(-dist ** 2 / 8.0))
    e.epoch(0.3, sel, want_dist=True)
    e.qe()
    e.close()

# BMU-ordered rows (re-layout forced at this size), then selections through
# the mapping; the split image + gather4 K1 for a selection
e = tsom.Engine(P, D)
e.set_option(_lib.TSOM_OPT_ROW_ORDER, 2)
e.set_option(93, 0)
e.bind(x)
e.set_codebook(w)
e.set_topology_distance(dist)
e.train_epochs([0.5, 0.4, 0.3], [4.0, 3.0, 2.0])
e.bmu_bound(None)
e.get_rows(10, 100)
e.set_influence(np.exp(-dist ** 2 / 8.0))
e.epoch(0.3, np.arange(n - 1, 0, -2, dtype=np.uint32), want_dist=True)
e.set_option(95, 1)
e.epoch(0.3, np.arange(0, n, 2, dtype=np.uint32), want_dist=True)
e.close()

# packed rows (no 256-B stride), random + adaptive samplers, refresh, guard paths
e = tsom.Engine(P, D)
e.set_option(_lib.TSOM_OPT_PAD_ROWS, 0)
e.bind(x)
e.set_codebook(w)
for kind in ("mst", "rng"):
    e.refresh_topology(kind)
e.sampler_init("random", 1000, 5)
e.train_epoch(0.5, 3.0, sampled=True)
e.sampler_init("adaptive", 900, 5)
e.train_epochs([0.5, 0.4], [3.0, 2.5], sampled=True)
e.close()

e = tsom.Engine(2, 4)  # the exact term-guard path (cheap bound over)
xb = (np.random.default_rng(0).standard_normal((64, 4)) * 1e-3).astype(np.float32)
e.bind(xb)
e.set_codebook(np.array([[0.0] * 4, [2.0 ** 23] * 4], np.float32))
e.set_influence(np.ones((2, 2)))
try:
    e.epoch(0.5)
except tsom.NumericalFault:
    pass
e.close()

# streamed epoch (chunks through the copy stream)
e = tsom.Engine(P, D)
e.set_option(_lib.TSOM_OPT_STREAM_CHUNK, 1024)
e.bind(x, streamed=True)
e.set_codebook(w)
e.set_influence(np.exp(-dist ** 2 / 8.0))
e.epoch(0.5, want_dist=True)
e.close()

# two ranks of one group
g = tsom.RankGroup(2)
ranks = []
for r, (a, b) in enumerate([(0, 3000), (3000, n)]):
    er = tsom.Engine(P, D)
    er.bind(x[a:b])
    er.join_group(g, r)
    er.set_codebook(w)
    er.set_influence(np.exp(-dist ** 2 / 8.0))
    ranks.append(er)
th = [threading.Thread(target=lambda er=er: er.epoch(0.5)) for er in ranks]
for t in th:
    t.start()
for t in th:
    t.join()
for er in ranks:
    er.close()
g.close()
print("sanitize target done, kernel launches:", _lib.kernel_launches())
