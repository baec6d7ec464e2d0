"""K1 main pass with and without the cluster multicast of A tiles (option 99
bit 6) at 1e7 and 1e8 rows: mean K1 event time over 4 single epochs each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist  # noqa: E402

for n in (10_000_000, 100_000_000):
    e = tsom.Engine(1024, 50)
    e.bind_synthetic_gmm(n, 2606)
    w0 = e.get_rows(0, 4096)[::4].copy()
    e.set_codebook(w0)
    e.set_topology_distance(lattice_dist("hex", 32, 32))
    for t in range(3):
        e.train_epoch(0.5 - 0.05 * t, 16.0 - 1.5 * t)
    for rep in range(2):
        for mc in (0, 64):
            e.set_option(99, mc)
            ks = []
            for t in range(4):
                e.train_epoch(0.3, 8.0)
                ks.append(e.timing_detail()["k1_ms"])
            print(f"n={n} multicast={bool(mc)} k1_ms={sum(ks)/len(ks):.3f} per1e7={sum(ks)/len(ks)*1e7/n:.3f}", flush=True)
    e.set_option(99, 0)
    e.close()
    tsom.release_cached_memory = None
