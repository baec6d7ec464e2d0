"""Diagnostics: the K2 row gather on the BMU-ordered packed rows — per-row TMA
bulk copies (default) against the cp.async gather (option 97 = 1) — mean
accumulation phase over 20-epoch calls, alternating."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist  # noqa: E402

host = bench.host_gmm_rows(10_000_000, bench.SEEDS["c2"])
e = tsom.Engine(1024, 50)
e.bind(host)
e.set_codebook(init_sample_draw(host, 1024, bench.SEEDS["c2"]))
e.set_topology_distance(lattice_dist("hex", 32, 32))
etas, sigmas = bench.hex_schedule(bench.EPOCHS, 0, 40)
e.train_epochs(etas[:25], sigmas[:25])  # auto re-layout happens here
for rep in range(3):
    for kind in (0, 1):
        e.set_option(97, kind)
        e.train_epochs(etas[:20], sigmas[:20])
        d = e.timing_detail()
        print(f"gather_kind={kind}: accum mean {d['accum_mean_ms']:.3f} ms, k1 {d['k1_ms']:.3f}",
              flush=True)
