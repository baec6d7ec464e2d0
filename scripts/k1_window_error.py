#!/usr/bin/env python
"""Measure the split-precision error of K1 against the near-tie window.

K1 (tcgen05, 3xFP16 or 3xTF32 split products, FP32 accumulation in TMEM)
computes v_ij = S (||x_i||^2 + ||w_j||^2 - 2 x_i.w_j) per row and node; a row
is decided by K1 alone only when its best and second-best values differ by
more than the window thr_i = tau S (||x_i||^2 + max_j ||w_j||^2) + abs terms,
tau = 2^-14.  BMU exactness rests on |v_ij / S - d2_ij| staying
below tau (||x_i||^2 + max ||w||^2) / 2 for every (i, j).  This script dumps
every raw K1 value of one main pass (option 99 bit 7) on the c2 workload
(reference-generator rows, a codebook trained for some epochs of the c2
schedule) and reports the largest normalised error against exact FP64
distances:

    e_ij = |v_ij / S - d2_ij| / (||x_i||^2 + max_j ||w_j||^2)

Usage: python scripts/k1_window_error.py [--rows 1000000] [--epochs 5] [--kernel 3]
Writes one JSON line (stdout) for profiles/.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def k1_values(eng, n, P):
    """Raw main-pass K1 values [n, groups*gn] (scaled units) and the scale S."""
    import torch
    from paper_2604_26555_b200 import _lib
    L = _lib.load()
    L.tsom_debug_k1_dump.argtypes = [C.c_void_p]
    L.tsom_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
    L.tsom_debug_read.restype = C.c_int64
    gn = 256 if P >= 256 else (P + 31) // 32 * 32
    cols = (P + gn - 1) // gn * gn
    dump = torch.full((n, cols), float("nan"), dtype=torch.float32, device="cuda")
    assert L.tsom_debug_k1_dump(dump.data_ptr()) == 0
    eng.set_option(99, 128)
    try:
        eng.bmu_bound(None, want_dist=False)
    finally:
        eng.set_option(99, 0)
        L.tsom_debug_k1_dump(None)
    sc = np.zeros(4, np.float32)
    L.tsom_debug_read(eng.h, 3, sc.ctypes.data, 16)
    return dump[:, :P], float(sc[1])


def window_error(x, w, v, S, chunk=65536):
    """max / quantiles of e_ij over all (i, j), plus per-row margins."""
    import torch
    X = torch.from_numpy(np.asarray(x, np.float64)).cuda()
    W = torch.from_numpy(np.asarray(w, np.float64)).cuda()
    w2 = (W * W).sum(1)
    w2max = float(w2.max())
    errs, worst = [], (0.0, -1, -1)
    for a in range(0, X.shape[0], chunk):
        Xc = X[a:a + chunk]
        x2 = (Xc * Xc).sum(1)
        d2 = x2[:, None] + w2[None, :] - 2.0 * (Xc @ W.T)
        vc = v[a:a + chunk].double() / S
        e = (vc - d2).abs() / (x2[:, None] + w2max)
        m = float(e.max())
        if m > worst[0]:
            idx = int(e.argmax())
            worst = (m, a + idx // W.shape[0], idx % W.shape[0])
        errs.append(e.flatten()[torch.randint(0, e.numel(), (200_000,), device="cuda")])
    s = torch.cat(errs)
    q = torch.quantile(s.float(), torch.tensor([0.5, 0.99, 0.9999], device="cuda")).tolist()
    return {"max": worst[0], "argmax_row": worst[1], "argmax_node": worst[2],
            "p50": q[0], "p99": q[1], "p9999": q[2]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--kernel", type=int, default=3)
    args = ap.parse_args()
    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200 import _lib
    from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist, resolved_sigma0,
                                               schedule_value)
    P, D, seed = 1024, 50, 2606
    x = _lib.synth_gmm_host(args.rows, D, seed)
    e = tsom.Engine(P, D)
    e.set_option(_lib.TSOM_OPT_BMU_KERNEL, args.kernel)
    e.set_option(_lib.TSOM_OPT_ROW_ORDER, 0)  # raw dump is in position order
    e.bind(x)
    e.set_codebook(init_sample_draw(x, P, seed))
    e.set_topology_distance(lattice_dist("hex", 32, 32))
    s0 = resolved_sigma0("hex", 32, 32)
    out = {"workload": f"c2 rows [0, {args.rows}) (reference generator, seed {seed}), 32x32 hex",
           "kernel": {3: "tcgen05 3xFP16", 2: "tcgen05 3xTF32"}[args.kernel],
           "tau": 2.0 ** -14, "by_epoch": []}
    for t in range(args.epochs + 1):
        v, S = k1_values(e, args.rows, P)
        r = window_error(x, e.get_codebook(), v, S)
        r["epoch"] = t
        r["max_over_tau"] = r["max"] / out["tau"]
        out["by_epoch"].append(r)
        del v
        if t < args.epochs:
            e.train_epoch(schedule_value(0.5, "linear", t, 10, 1e-4),
                          schedule_value(s0, "linear", t, 10, 0.3))
    out["max"] = max(r["max"] for r in out["by_epoch"])
    out["max_over_tau"] = out["max"] / out["tau"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
