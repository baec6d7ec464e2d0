"""Per-kernel CUPTI times of the c4 leg's sampled epochs: bench.leg_c4's
workload (1e8 x 50 rows resident, RNG topology, adaptive sampler rho = 0.1 on
the device) after a 10-epoch schedule, then 3 more sampled epochs under
torch.profiler; prints JSON {kernel: [launches per epoch, us per epoch]}.
Usage: python scripts/c4_profile.py [n_rows]"""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw, resolved_sigma0  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
seed = bench.SEEDS["c4"]
e = tsom.Engine(bench.P, bench.D)
e.bind_synthetic_gmm(n, seed, 16, 0)
e.set_codebook(init_sample_draw(bench.EngineRows(e), bench.P, seed))
e.sampler_init("adaptive", n // 10, seed)
bench.graph_epochs(e, "rng", bench.EPOCHS, sampled=True)
torch.cuda.synchronize()
E = 3
sig = resolved_sigma0("rng", 0, 0, 0.0) * 0.3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(E):
        e.train_epoch(0.1, sig, sampled=True)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[ev.name[:60]]
        a[0] += 1
        a[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
out = {k: [round(v[0] / E, 1), round(v[1] / E, 1)] for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
json.dump({"rows": n, "epochs": E, "timing": e.timing_detail(), "kernels_us_per_epoch": out}, sys.stdout, indent=1)
