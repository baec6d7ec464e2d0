"""Timing of the device samplers at scale (diagnostics): select() + observe()
per epoch for N rows (rows are not read: a 1-column dummy dataset is bound)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
RHO = 0.1
for kind in ("random", "adaptive"):
    e = tsom.Engine(4, 1)
    d = torch.zeros(N, dtype=torch.float32, device="cuda")
    e.bind_device(d.data_ptr(), N) if hasattr(e, "bind_device") else e.bind(np.zeros((N, 1), np.float32))
    m = int(N * RHO)
    t0 = time.time()
    e.sampler_init(kind, m, 2608)
    t_init = time.time() - t0
    dist = np.random.default_rng(0).random(m)
    ts = []
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.time()
        sel = e.sampler_select()
        if kind == "adaptive":
            e.sampler_observe(dist[: len(sel)])
        torch.cuda.synchronize()
        ts.append(time.time() - t0)
    print(f"{kind}: N={N} m={m} init {t_init:.2f}s  select(+observe) incl. D2H of the ids: "
          f"{[round(t * 1e3, 1) for t in ts]} ms", flush=True)
