"""Diagnostics: K1 over a rho = 0.1 selection of 1e8 resident rows — rows
gathered from the split image (TMA gather4, multicast over the group
cluster; option 99 bit 10 = one CTA per row fetch) against tiles split per
pass (option 95 = 0)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
rng = np.random.default_rng(0)
sel = np.sort(rng.choice(N, N // 10, replace=False)).astype(np.uint32)
for mode, dbgs in ((0, (0,)), (1, (0, 1024))):
    e = tsom.Engine(1024, 50)
    e.set_option(95, mode)
    e.bind_synthetic_gmm(N, 2608, 16, 0)
    e.set_codebook((rng.standard_normal((1024, 50)) * 2).astype(np.float32))
    e.set_influence(np.eye(1024))
    for dbg in dbgs:
        e.set_option(99, dbg)
        ts = []
        for _ in range(4):
            e.epoch(0.0, sel)
            ts.append(e.timing_detail()["k1_ms"])
        print(f"image={mode} dbg={dbg:#x}: k1 {np.round(ts, 3).tolist()} ms "
              f"bmu phase {e.timing_detail()['bmu_ms']:.3f}", flush=True)
    e.set_option(99, 0)
    e.close()
