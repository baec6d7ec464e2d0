"""Epoch time with and without exact sums (TSOM_OPT_DETERMINISTIC) on the c2
workload: 10 epochs in one tsom_train_epochs call, CUDA events, twice each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist,  # noqa: E402
                                           resolved_sigma0, schedule_value)

n, P, D, seed = 10_000_000, 1024, 50, 2606
x = _lib.synth_gmm_host(n, D, seed)
w0 = init_sample_draw(x, P, seed)
s0 = resolved_sigma0("hex", 32, 32)
etas = [schedule_value(0.5, "linear", t, 10, 1e-4) for t in range(10)]
sig = [schedule_value(s0, "linear", t, 10, 0.3) for t in range(10)]
for rep in range(2):
    for exact in (0, 1):
        e = tsom.Engine(P, D)
        e.set_option(_lib.TSOM_OPT_DETERMINISTIC, exact)
        e.bind(x)
        e.set_codebook(w0)
        e.set_topology_distance(lattice_dist("hex", 32, 32))
        e.train_epochs(etas[:3], sig[:3])
        e.set_codebook(w0)
        st = torch.cuda.ExternalStream(e.stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        e.train_epochs(etas, sig)
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        e.train_epoch(0.2, 4.0)
        print(f"exact={exact} ms/epoch={ms:.3f} accum_ms={e.timing_detail()['accum_ms']:.3f}",
              flush=True)
        e.close()
