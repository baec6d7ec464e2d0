"""Profile target for the row split kernels: one gathered split with the
element-wise kernel (option 98 = 1) and one with the warp-synchronous kernel, on the
c2 row shape.  Run under ncu -k regex:k_split_rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402

n, d, p = 4_000_000, 50, 1024
rng = np.random.default_rng(1)
x = rng.normal(size=(n, d)).astype(np.float32)
for v1 in (1, 0):
    e = tsom.Engine(p, d)
    e.set_option(98, v1)
    e.set_codebook(x[:p])
    e.bind(x)
    e.set_influence(np.eye(p))
    e.epoch(0.5)                                       # resident split
    e.epoch(0.5, selected=np.arange(0, n, 3, dtype=np.uint32))  # gathered split
    e.close()
print("ok")
