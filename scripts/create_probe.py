import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2604_26555_b200 as tsom
from paper_2604_26555_b200.hostref import lattice_dist
x = np.zeros((1000, 50), np.float32)
d = lattice_dist("hex", 32, 32)
w = np.zeros((1024, 50), np.float32)
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e = tsom.Engine(1024, 50); t1 = time.perf_counter()
    e.set_codebook(w); e.set_topology_distance(d); t2 = time.perf_counter()
    e.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms config {1e3*(t2-t1):.2f} close {1e3*(t3-t2):.2f}", flush=True)
