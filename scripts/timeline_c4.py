"""Kernel timeline of the c4 leg (bench.run_c4_leg) via torch.profiler: per
kernel device time summed over the timed epochs, both streams."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    out = bench.run_c4_leg(0, epochs=10, warm=2)
evs = [ev for ev in prof.events() if ev.device_type.name == "CUDA"]
agg = {}
for ev in evs:
    d = agg.setdefault(ev.name[:48], [0, 0.0])
    d[0] += 1
    d[1] += ev.time_range.elapsed_us()
span = max(e.time_range.end for e in evs) - min(e.time_range.start for e in evs)
print(json.dumps({"c4": {k: out[k] for k in ("value", "ms_per_epoch")}, "span_ms": span / 1e3,
                  "kernels_ms": {k: [v[0], round(v[1] / 1e3, 3)]
                                 for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]}},
                 indent=1))
