"""Out-of-core epoch throughput (BASELINE configs[4] per-GPU slice, §8(f) row 3).

Times one full-sampling training epoch (tsom_train_epoch) over the same rows
bound four ways: resident in HBM, streamed from page-locked host memory,
streamed from pageable host memory through the pinned staging, and streamed
from FSOMSHRD shard files (page cache warm after the first epoch).  The H2D
roofline for the streamed modes is a plain pinned cudaMemcpy of one chunk.

    python scripts/stream_bench.py --rows 20000000 --epochs 3
"""
import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=20_000_000)
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=1 << 20)
    ap.add_argument("--shard-dir", default="/tmp/tsom_stream_shards")
    ap.add_argument("--modes", default="resident,pinned,pageable,shards")
    ap.add_argument("--staging-threads", type=int, default=0, help="0: engine default")
    args = ap.parse_args()

    import numpy as np
    import torch

    import bench
    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200 import _lib, shards
    from paper_2604_26555_b200.hostref import lattice_dist

    n, D, P = args.rows, bench.D, 1024
    host = bench.host_gmm_rows(n, 2602)               # page-locked (torch pinned)
    w0 = host[np.linspace(0, n - 1, P).astype(np.int64)].copy()
    dist = lattice_dist("hex", 32, 32)

    # H2D roofline: pinned chunk copy
    chunk = torch.from_numpy(host[: args.chunk])
    dev = torch.empty_like(chunk, device="cuda")
    for _ in range(3):
        dev.copy_(chunk, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        dev.copy_(chunk, non_blocking=True)
    torch.cuda.synchronize()
    h2d_gbs = 10 * chunk.numel() * 4 / (time.perf_counter() - t0) / 1e9
    del dev

    out = {"rows": n, "d": D, "nodes": P, "chunk_rows": args.chunk,
           "h2d_pinned_gbs": round(h2d_gbs, 1),
           "h2d_bound_rows_per_s": h2d_gbs * 1e9 / (4 * D)}
    modes = args.modes.split(",")
    pageable = None
    if "pageable" in modes:
        pageable = np.array(host, copy=True)          # ordinary malloc'd memory
    if "shards" in modes:
        shutil.rmtree(args.shard_dir, ignore_errors=True)
        t0 = time.perf_counter()
        paths = shards.write_shards(host, args.shard_dir, 8)
        out["shard_write_s"] = round(time.perf_counter() - t0, 2)
    for mode in modes:
        e = tsom.Engine(P, D)
        e.set_option(_lib.TSOM_OPT_STREAM_CHUNK, args.chunk)
        if args.staging_threads:
            e.set_option(_lib.TSOM_OPT_STAGING_THREADS, args.staging_threads)
        t0 = time.perf_counter()
        if mode == "resident":
            e.bind(host)
        elif mode == "pinned":
            e.bind(host, streamed=True)
        elif mode == "pageable":
            e.set_option(_lib.TSOM_OPT_HOST_REGISTER, 0)
            e.bind(pageable, streamed=True)
        elif mode == "shards":
            e.bind_shards(paths, streamed=True)
        bind_s = time.perf_counter() - t0
        e.set_codebook(w0)
        e.set_topology_distance(dist)
        times = []
        for t in range(args.epochs + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e.train_epoch(0.5 * (1 - t / 10), max(0.3, 16.0 * (1 - t / 10)), 0.0, False)
            times.append(time.perf_counter() - t0)
        s = min(times[1:])
        out[mode] = {"epoch_s": round(s, 4), "rows_per_s": n / s, "bind_s": round(bind_s, 3),
                     "frac_of_h2d": (n / s) / out["h2d_bound_rows_per_s"]}
        e.close()
    if "shards" in modes:
        shutil.rmtree(args.shard_dir, ignore_errors=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
