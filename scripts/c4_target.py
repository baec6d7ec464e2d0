"""Profile target for the c4 workload (bench.leg_c4's epochs: 1e8 x 50 rows
resident, RNG topology, adaptive sampler rho = 0.1 on the device), run under
ncu with a kernel filter.  Usage: python scripts/c4_target.py [n_rows] [epochs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
e = tsom.Engine(bench.P, bench.D)
e.bind_synthetic_gmm(n, bench.SEEDS["c4"], 16, 0)
e.set_codebook(init_sample_draw(bench.EngineRows(e), bench.P, bench.SEEDS["c4"]))
e.sampler_init("adaptive", n // 10, bench.SEEDS["c4"])
bench.graph_epochs(e, "rng", epochs, sampled=True)
print("done", e.timing_detail())
