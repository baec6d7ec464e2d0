"""Kernel timeline of c2 epochs via torch.profiler (CUPTI activity tracing):
per-kernel device time and the idle gaps between consecutive kernels on the
engine stream.  Usage: python scripts/timeline.py [n_rows]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import lattice_dist  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
P, D = 1024, 50
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((n, D), device="cuda", generator=g) + 3.0 * torch.randn((16, D), device="cuda",
                                                                          generator=g)[
    torch.randint(0, 16, (n,), device="cuda", generator=g)]
e = tsom.Engine(P, D)
e.bind_device(x.data_ptr(), n)
e.set_codebook(x[:: n // P][:P].cpu().numpy())
e.set_topology_distance(lattice_dist("hex", 32, 32))
for t in range(3):
    e.train_epoch(0.5, 8.0 - t)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for t in range(3):
        e.train_epoch(0.4, 5.0 - t)
    torch.cuda.synchronize()
evs = [ev for ev in prof.events() if ev.device_type.name == "CUDA"]
evs = sorted(evs, key=lambda ev: ev.time_range.start)
rows = []
for a, b in zip(evs, evs[1:] + [None]):
    gap = (b.time_range.start - a.time_range.end) if b else 0
    rows.append((a.name[:40], a.time_range.elapsed_us(), gap))
agg = {}
for name, dur, gap in rows:
    d = agg.setdefault(name, [0, 0.0, 0.0])
    d[0] += 1
    d[1] += dur
    d[2] += max(gap, 0)
span = evs[-1].time_range.end - evs[0].time_range.start
busy = sum(r[1] for r in rows)
print(json.dumps({"epochs": 3, "span_us": span, "busy_us": busy,
                  "kernels": {k: {"n": v[0], "us": round(v[1], 1), "gap_after_us": round(v[2], 1)}
                              for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}, indent=1))
