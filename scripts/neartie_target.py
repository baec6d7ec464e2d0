"""Profile target for the near-tie path: the c2 workload trained for one
schedule cycle (10 epochs), then schedule epochs 0..E-1 of the next cycle one
by one, with only epoch E-1 inside a cudaProfilerStart/Stop range.  Run under
`ncu --profile-from-start off -k regex:... ` (scripts/ncu_neartie.sh).
Usage: python scripts/neartie_target.py [n_rows] [E]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist,  # noqa: E402
                                           resolved_sigma0, schedule_value)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
E = int(sys.argv[2]) if len(sys.argv) > 2 else 6
P, D, seed = 1024, 50, 2606
x = _lib.synth_gmm_host(n, D, seed)
e = tsom.Engine(P, D)
# the bench's steady state: rows re-laid out in BMU order (its 50-epoch timed
# call does it in auto mode; these per-epoch calls ask for it explicitly)
e.set_option(_lib.TSOM_OPT_ROW_ORDER, 2)
e.bind(x)
e.set_codebook(init_sample_draw(x, P, seed))
e.set_topology_distance(lattice_dist("hex", 32, 32))
s0 = resolved_sigma0("hex", 32, 32)
eta = [schedule_value(0.5, "linear", t, 10, 1e-4) for t in range(10)]
sig = [schedule_value(s0, "linear", t, 10, 0.3) for t in range(10)]
e.train_epochs(eta, sig)
for t in range(E):
    if t == E - 1:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    e.train_epoch(eta[t], sig[t])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", e.timing_detail(), "recheck", e.last_recheck_count)
