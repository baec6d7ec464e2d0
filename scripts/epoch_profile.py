"""Per-epoch phase times across the bench's 10-epoch c2 schedule.

bench.py times 50 epochs that cycle through the schedule t % 10 (η 0.5 → 1e-4,
σ σ0 → 0.3), so the collapsed-map epochs (large σ, many near-ties) weigh in
the headline as much as the late ones.  For each schedule position this runs
one tsom_train_epoch (after `cycles` warm cycles) and prints the phase times
and the near-tie / re-check counts, then times one whole cycle through
tsom_train_epochs with CUDA events, and a CUPTI timeline of that cycle
aggregated per kernel.

Usage: python scripts/epoch_profile.py [n_rows] [cycles]"""
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
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 1
P, D, seed, E = 1024, 50, 2606, 10
x = _lib.synth_gmm_host(n, D, seed)
e = tsom.Engine(P, D)
# the bench's steady state: rows re-laid out in BMU order (its 50-epoch timed
# call does it in auto mode; these per-epoch calls ask for it explicitly)
e.set_option(_lib.TSOM_OPT_ROW_ORDER, 2)
e.bind(x)
e.set_codebook(init_sample_draw(x, P, seed))
e.set_topology_distance(lattice_dist("hex", 32, 32))
s0 = resolved_sigma0("hex", 32, 32)
eta = [schedule_value(0.5, "linear", t, E, 1e-4) for t in range(E)]
sig = [schedule_value(s0, "linear", t, E, 0.3) for t in range(E)]
for _ in range(cycles):
    e.train_epochs(eta, sig)
rows = []
for t in range(E):
    e.train_epoch(eta[t], sig[t])
    d = e.timing_detail()
    d = {k: round(v, 3) for k, v in d.items()}
    d.update(epoch=t, sigma=round(sig[t], 3), recheck=e.last_recheck_count)
    rows.append(d)
stream = torch.cuda.ExternalStream(e.stream)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record(stream)
e.train_epochs(eta, sig)
b.record(stream)
torch.cuda.synchronize()
cycle_ms = a.elapsed_time(b)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e.train_epochs(eta, sig)
    torch.cuda.synchronize()
evs = sorted([ev for ev in prof.events() if ev.device_type.name == "CUDA"],
             key=lambda ev: ev.time_range.start)
agg = {}
for ev in evs:
    k = ev.name[:40]
    v = agg.setdefault(k, [0, 0.0])
    v[0] += 1
    v[1] += ev.time_range.elapsed_us()
span = evs[-1].time_range.end - evs[0].time_range.start
seq = [[ev.name[:40], round(ev.time_range.start - evs[0].time_range.start, 1),
        round(ev.time_range.elapsed_us(), 1)] for ev in evs]
busy = sum(v[1] for v in agg.values())
print(json.dumps({"rows": n, "per_epoch": rows, "cycle_ms_events": cycle_ms,
                  "ms_per_epoch_events": cycle_ms / E,
                  "cupti_span_ms": span / 1e3, "cupti_busy_ms": busy / 1e3,
                  "kernels_us_per_epoch": {k: [v[0] / E, round(v[1] / E, 1)] for k, v in
                                           sorted(agg.items(), key=lambda kv: -kv[1][1])},
                  "launches": seq},
                 indent=1))
