"""Diagnostics: tsom_bind_host_data from pageable rows (c2 shape) against the
staging chunk size (option 94) and staging threads; best of 3 per setting."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402

n = 10_000_000
rows = np.array(bench.host_gmm_rows(n, 7), copy=True)  # pageable
for chunk_mb in (32, 64, 128, 256):
    for thr in (8, 16):
        ts = []
        for _ in range(3):
            e = tsom.Engine(1024, 50)
            e.set_option(94, chunk_mb << 20)
            e.set_option(_lib.TSOM_OPT_STAGING_THREADS, thr)
            t0 = time.perf_counter()
            e.bind(rows)
            ts.append(time.perf_counter() - t0)
            e.close()
        print(f"chunk {chunk_mb} MB threads {thr}: bind {min(ts) * 1e3:.1f} ms "
              f"({rows.nbytes / min(ts) / 1e9:.1f} GB/s)", flush=True)
