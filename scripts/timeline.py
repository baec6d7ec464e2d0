"""Kernel timeline of c2 epochs via torch.profiler (CUPTI activity tracing):
per-kernel device time and the idle gaps between consecutive kernels.  The
bench's workload: reference-generator rows bound from the host, a codebook
trained for `warm` epochs of the c2 schedule, then `epochs` epochs in one
tsom_train_epochs call.

Usage: python scripts/timeline.py [n_rows] [epochs] [topology: hex|mst]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist,  # noqa: E402
                                           resolved_sigma0, schedule_value)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P, D, seed, warm = 1024, 50, 2606, 5
x = _lib.synth_gmm_host(n, D, seed)
e = tsom.Engine(P, D)
e.bind(x)
e.set_codebook(init_sample_draw(x, P, seed))
e.set_topology_distance(lattice_dist("hex", 32, 32))
s0 = resolved_sigma0("hex", 32, 32)
sched = [(schedule_value(0.5, "linear", t % 10, 10, 1e-4), schedule_value(s0, "linear", t % 10, 10, 0.3))
         for t in range(warm + epochs)]
e.train_epochs([s[0] for s in sched[:warm]], [s[1] for s in sched[:warm]])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e.train_epochs([s[0] for s in sched[warm:]], [s[1] for s in sched[warm:]])
    torch.cuda.synchronize()
evs = [ev for ev in prof.events() if ev.device_type.name == "CUDA"]
evs = sorted(evs, key=lambda ev: ev.time_range.start)
rows = []
for a, b in zip(evs, evs[1:] + [None]):
    gap = (b.time_range.start - a.time_range.end) if b else 0
    rows.append((a.name[:48], a.time_range.elapsed_us(), gap))
agg = {}
for name, dur, gap in rows:
    d = agg.setdefault(name, [0, 0.0, 0.0])
    d[0] += 1
    d[1] += dur
    d[2] += max(gap, 0)
span = evs[-1].time_range.end - evs[0].time_range.start
busy = sum(r[1] for r in rows)
print(json.dumps({"rows": n, "epochs": epochs, "span_us": span, "busy_us": busy,
                  "per_epoch_us": span / epochs,
                  "kernels": {k: {"n": v[0], "us_per_epoch": round(v[1] / epochs, 1),
                                  "gap_after_us_per_epoch": round(v[2] / epochs, 1)}
                              for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}, indent=1))
