"""Diagnostics: per-tile timeline of K1 on CTA 0 (option 99 bit 5)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import lattice_dist  # noqa: E402

dbg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
e = tsom.Engine(1024, 50)
e.bind_synthetic_gmm(10_000_000, 2606)
rng = np.random.default_rng(0)
e.set_codebook((rng.standard_normal((1024, 50)) * 3).astype(np.float32))
e.set_topology_distance(lattice_dist("hex", 32, 32))
e.set_option(99, dbg | 32)
for _ in range(3):
    e.train_epoch(0.1, 3.0)
buf = (C.c_ulonglong * 4096)()
_lib.load().tsom_debug_k1_trace(buf, 4096)
tr = np.array(buf, dtype=np.int64).reshape(512, 8)
t0 = tr[0, 0]
print("slots: 0 mma-ready 1 mma-issued | set0: 2 tfull 3 pass1 4 arrive | set1: 5 tfull 6 pass1 7 arrive")
for i in range(20, 40):
    r = tr[i] - t0
    print(i, " ".join(f"{v:9d}" for v in r))
d = np.diff(tr[10:500, 0])
print("mma-ready period median", np.median(d), "issue->ready(next)", np.median(tr[11:500, 0] - tr[10:499, 1]))
ev = tr[10:500:2]; od = tr[11:500:2]
print("set0: tfull->pass1", np.median(ev[:, 3] - ev[:, 2]), "pass1->arrive", np.median(ev[:, 4] - ev[:, 3]))
print("set1: tfull->pass1", np.median(od[:, 6] - od[:, 5]), "pass1->arrive", np.median(od[:, 7] - od[:, 6]))
print("mma issued -> epi tfull (even)", np.median(ev[:, 2] - ev[:, 1]))
print("epi arrive(t) -> mma ready(t+2) (even)", np.median(tr[12:500:2, 0] - tr[10:498:2, 4]))
print("mma ready -> issued", np.median(tr[10:500, 1] - tr[10:500, 0]))
