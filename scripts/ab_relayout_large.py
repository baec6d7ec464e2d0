"""Diagnostics: 10-epoch runs at 1e8+ rows with (row order 2) and without (0)
the one BMU-order re-layout — the c3 shape (MST refreshed on the reference
schedule, 1e8 device-generated rows) and the c5 resident shape (32x32 hex,
1.25e8 rows) — CUDA events around each whole run, alternating."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist  # noqa: E402


def run(kind, n, ro):
    e = tsom.Engine(bench.P, bench.D)
    e.set_option(_lib.TSOM_OPT_ROW_ORDER, ro)
    e.bind_synthetic_gmm(n, 2607, 16, 0)
    w0 = init_sample_draw(bench.EngineRows(e), bench.P, 2607)
    if kind == "hex":
        e.set_topology_distance(lattice_dist("hex", 32, 32))
    out = []
    for rep in range(2):
        e.set_codebook(w0)
        if ro:  # a fresh bind order for every timed run: re-bind
            e.bind_synthetic_gmm(n, 2607, 16, 0)
        st = torch.cuda.ExternalStream(e.stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        if kind == "hex":
            etas, sigmas = bench.hex_schedule(bench.EPOCHS)
            e.train_epochs(etas, sigmas)
        else:
            bench.graph_epochs(e, "mst", bench.EPOCHS)
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / bench.EPOCHS)
    e.close()
    bench.close_engine(None)
    return out


for kind, n in (("mst", 100_000_000), ("hex", 125_000_000)):
    for ro in (0, 2, 0, 2):
        print(f"{kind} n={n} row_order={ro}: ms/epoch {[round(v, 2) for v in run(kind, n, ro)]}",
              flush=True)
