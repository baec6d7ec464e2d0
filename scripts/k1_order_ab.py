"""Diagnostics: K1 main-pass time on the c2 rows in their stored order against
the same rows re-ordered by their BMU, with the epilogue's chunk skip on (option
99 = 0) and off (option 99 bit 8).  Codebook: the c2 bench's after its schedule
cycle (init_sample_draw + 10 epochs)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402
from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
host = bench.host_gmm_rows(N, bench.SEEDS["c2"])
w0 = init_sample_draw(host, bench.P, bench.SEEDS["c2"])
etas, sigmas = bench.hex_schedule(bench.EPOCHS)


def chunk_stats(e, t=7):
    import ctypes
    from paper_2604_26555_b200 import _lib
    buf = (ctypes.c_ulonglong * 4096)()
    _lib.load().tsom_debug_k1_trace(buf, 4096)
    r0, c0 = buf[4094], buf[4095]
    w = e.get_codebook()
    e.set_option(99, 512)
    e.train_epoch(etas[t], sigmas[t])
    e.set_option(99, 0)
    e.set_codebook(w)
    _lib.load().tsom_debug_k1_trace(buf, 4096)
    return (buf[4094] - r0) / max(1, buf[4095] - c0)


def k1_times(e, label, ep=(5, 9)):
    print(f"{label}: pass-2 chunks run {chunk_stats(e):.3f}", flush=True)
    out = {}
    for dbg in (0, 256):
        e.set_option(99, dbg)
        ts = []
        for t in range(ep[0], ep[1] + 1):
            w = e.get_codebook()
            e.train_epoch(etas[t], sigmas[t])
            td = e.timing_detail()
            ts.append(td["k1_ms"])
            e.set_codebook(w)  # keep the codebook fixed across the A/B
        out[dbg] = ts
        print(f"{label} dbg={dbg}: k1 {np.round(ts, 3).tolist()} ms; last epoch "
              f"{ {k: round(v, 3) for k, v in td.items()} }", flush=True)
    e.set_option(99, 0)
    return out


e = tsom.Engine(bench.P, bench.D)
e.bind(host)
e.set_codebook(w0)
e.set_topology_distance(lattice_dist("hex", *bench.P_GRID))
e.train_epochs(etas[:5], sigmas[:5])
w5 = e.get_codebook()
k1_times(e, "stored order, codebook after 5 epochs")
b, _ = e.bmu_bound(None, want_dist=False)
order = np.argsort(b, kind="stable")
e.close()

hs = np.ascontiguousarray(host[order])
for pad in (1, 0):
    for label, rows in (("BMU order", hs), ("stored order", host)):
        e = tsom.Engine(bench.P, bench.D)
        e.set_option(_lib.TSOM_OPT_PAD_ROWS, pad)
        e.bind(rows)
        e.set_codebook(w5)
        e.set_topology_distance(lattice_dist("hex", *bench.P_GRID))
        k1_times(e, f"{label} pad={pad}, codebook after 5 epochs")
        e.close()
