"""Sustained A/B of K1 variants under the power cap: the bench's workload (c2
rows from the reference generator, 10-epoch hex schedule cycled) trained for
`epochs` epochs per tsom_train_epochs call, alternating option-99 modes on
the same engine (0 = default; 64 = cluster multicast of the A tiles).  Per
call: ms/epoch (CUDA events), mean K1 ms, and the SM clock and board power
sampled by NVML every 10 ms during the call.
Usage: python scripts/k1_power_ab.py [epochs] [modes, comma-separated]"""
import json
import os
import statistics
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist,  # noqa: E402
                                           resolved_sigma0, schedule_value)

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 50
modes = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,64,0,64").split(",")]
n, P, D, seed = 10_000_000, 1024, 50, 2606
x = _lib.synth_gmm_host(n, D, seed)
e = tsom.Engine(P, D)
e.bind(x)
w0 = init_sample_draw(x, P, seed)
e.set_topology_distance(lattice_dist("hex", 32, 32))
s0 = resolved_sigma0("hex", 32, 32)
eta = [schedule_value(0.5, "linear", t % 10, 10, 1e-4) for t in range(epochs)]
sig = [schedule_value(s0, "linear", t % 10, 10, 0.3) for t in range(epochs)]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stream = torch.cuda.ExternalStream(e.stream)
out = []
for mode in modes:
    e.set_option(99, mode)
    e.set_codebook(w0)
    e.train_epochs(eta[:10], sig[:10])  # warm (and the same state for each mode)
    e.set_codebook(w0)
    samples, stop = [], threading.Event()

    def run():
        while not stop.is_set():
            try:
                samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(h) / 1e3))
            except Exception:
                pass
            stop.wait(0.01)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    th = threading.Thread(target=run, daemon=True)
    th.start()
    a.record(stream)
    e.train_epochs(eta, sig)
    b.record(stream)
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = a.elapsed_time(b) / epochs
    out.append({"mode": mode, "ms_per_epoch": round(ms, 4),
                "k1_ms": round(e.timing_detail()["k1_ms"], 4),
                "sm_mhz_median": statistics.median(s[0] for s in samples) if samples else None,
                "power_w_median": statistics.median(s[1] for s in samples) if samples else None,
                "samples": len(samples)})
    print(json.dumps(out[-1]), flush=True)
e.set_option(99, 0)
