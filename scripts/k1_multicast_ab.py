"""A/B of the K1 multicast mode (option 99 bit 6: the 4 codebook-group CTAs of
a cluster each load a quarter of every A tile and multicast it) against the
default (each CTA loads whole tiles; L2 deduplicates).  Prints K1 ms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200.hostref import lattice_dist  # noqa: E402

n, P, D = 10_000_000, 1024, 50
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((n, D), device="cuda", generator=g)
for mode in (0, 64, 0, 64):
    e = tsom.Engine(P, D)
    e.set_option(99, mode)
    e.bind_device(x.data_ptr(), n)
    e.set_codebook(x[:: n // P][:P].cpu().numpy())
    e.set_topology_distance(lattice_dist("hex", 32, 32))
    ks = []
    for t in range(8):
        e.train_epoch(0.5, 8.0 - 0.5 * t)
        ks.append(e.timing_detail()["k1_ms"])
    e.set_option(99, 0)
    e.close()
    print("mode", mode, "k1 ms", sorted(ks[2:])[len(ks[2:]) // 2], flush=True)
