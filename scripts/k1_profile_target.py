"""Profile target: the c2 workload (reference-generator rows, 32x32 hex), a
few warm epochs, then single epochs — run under ncu with a kernel filter, e.g.
  ncu -k regex:"k1_bmu_tc<2, false, false>" --launch-skip 3 --launch-count 1 ...
Usage: python scripts/k1_profile_target.py [n_rows] [epochs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist,  # noqa: E402
                                           resolved_sigma0, schedule_value)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
P, D, seed = 1024, 50, 2606
x = _lib.synth_gmm_host(n, D, seed)
e = tsom.Engine(P, D)
e.bind(x)
e.set_codebook(init_sample_draw(x, P, seed))
e.set_topology_distance(lattice_dist("hex", 32, 32))
s0 = resolved_sigma0("hex", 32, 32)
for t in range(epochs):
    e.train_epoch(schedule_value(0.5, "linear", t, 10, 1e-4), schedule_value(s0, "linear", t, 10, 0.3))
print("done", e.timing_detail())
