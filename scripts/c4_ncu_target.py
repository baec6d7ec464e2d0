"""Profile target for c4: bench.leg_c4's workload (1e8 x 50 rows resident,
RNG topology, adaptive sampler rho = 0.1 on the device) for a 10-epoch
schedule, then one more sampled epoch inside a cudaProfilerStart/Stop range,
for `ncu --profile-from-start off` (scripts/ncu_c4.sh).
Usage: python scripts/c4_ncu_target.py [n_rows]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

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
torch.cuda.profiler.start()
e.train_epoch(0.1, resolved_sigma0("rng", 0, 0, 0.0) * 0.3, sampled=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", e.timing_detail(), "recheck", e.last_recheck_count)
