"""Kernel timeline of the c4 workload (bench.leg_c4's epochs): 1e8 x 50 rows
resident, RNG topology refreshed on the reference schedule, adaptive sampler
rho = 0.1 on the device.  Two warm-up epochs, then one 10-epoch schedule under
CUPTI (torch.profiler): per-kernel device time per epoch, the span, and the
launches of one epoch in order.
Usage: python scripts/timeline_c4.py [n_rows]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
seed, P, D, E = bench.SEEDS["c4"], bench.P, bench.D, bench.EPOCHS
e = tsom.Engine(P, D)
e.bind_synthetic_gmm(n, seed, 16, 0)
w0 = init_sample_draw(bench.EngineRows(e), P, seed)
e.set_codebook(w0)
e.sampler_init("adaptive", n // 10, seed)
bench.graph_epochs(e, "rng", 2, sampled=True)
e.set_codebook(w0)
e.sampler_init("adaptive", n // 10, seed)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bench.graph_epochs(e, "rng", E, sampled=True)
    torch.cuda.synchronize()
evs = sorted([ev for ev in prof.events() if ev.device_type.name == "CUDA"],
             key=lambda ev: ev.time_range.start)
agg = {}
for ev in evs:
    d = agg.setdefault(ev.name[:48], [0, 0.0])
    d[0] += 1
    d[1] += ev.time_range.elapsed_us()
span = evs[-1].time_range.end - evs[0].time_range.start
t0 = evs[0].time_range.start
k1 = [i for i, ev in enumerate(evs) if "k1_bmu_tc<2, false" in ev.name]
one = evs[k1[5] - 12:k1[6] - 12] if len(k1) > 6 else []
print(json.dumps({"rows": n, "span_ms": span / 1e3, "ms_per_epoch": span / 1e3 / E,
                  "kernels_us_per_epoch": {k: [v[0] / E, round(v[1] / E, 1)]
                                           for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])},
                  "epoch5_launches": [[ev.name[:44], round(ev.time_range.start - t0, 1),
                                       round(ev.time_range.elapsed_us(), 1)] for ev in one]},
                 indent=1))
