"""Diagnostics: device topology refresh times (MST, RNG) at K = 1024, and one of
each inside a cudaProfilerStart/Stop range for ncu --profile-from-start off."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2604_26555_b200 as tsom
rng = np.random.default_rng(0)
x = (rng.standard_normal((200000, 50)) * 2).astype(np.float32)
e = tsom.Engine(1024, 50)
e.bind(x)
e.set_codebook(x[:1024].copy())
for kind in ("mst", "rng"):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e.refresh_topology(kind)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(kind, round((t1 - t0) * 1e3, 3), "ms", flush=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
e.refresh_topology("mst")
e.refresh_topology("rng")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
