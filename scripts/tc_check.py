"""Quick GPU diagnostics for the BMU kernels: parity vs the oracle + timing."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2604_26555_b200 as tsom  # noqa: E402
from paper_2604_26555_b200 import _lib  # noqa: E402

chk = oracle.port
for p, n in [(16, 300), (100, 5000), (256, 20000), (1024, 20000), (1000, 12345)]:
    x = chk.synth_gmm(n, 50, 2600 + p)
    w = x[np.linspace(0, n - 1, p).astype(int)] * np.float32(0.9) + np.float32(0.05)
    bo, do = chk.find_bmus(x, w)
    for kern in (1, 2):
        e = tsom.Engine(p, 50)
        e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kern)
        e.set_codebook(w)
        t = time.time()
        b, d = e.bmu(x)
        dt = time.time() - t
        print(f"P={p} n={n} kernel={kern}: mismatches={(b != bo).sum()} rechecks={e.last_recheck_count}"
              f" maxreldist={np.max(np.abs(d - do) / do):.2e} t={dt*1e3:.1f}ms", flush=True)
        e.close()
# raw error of the tc kernel without the re-check window
p, n = 1024, 50000
x = chk.synth_gmm(n, 50, 7)
w = x[np.linspace(0, n - 1, p).astype(int)] * np.float32(0.9) + np.float32(0.05)
bo, _ = chk.find_bmus(x, w)
for kern in (1, 2):
    e = tsom.Engine(p, 50)
    e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kern)
    e.set_option(_lib.TSOM_OPT_TIE_TAU, 0)
    e.set_codebook(w)
    b, _ = e.bmu(x)
    print(f"tau=0 kernel={kern}: raw mismatches {(b != bo).sum()} / {n}; rechecks {e.last_recheck_count}")
    for tau_log2 in (-20, -18, -16, -14, -12):
        e.set_option(_lib.TSOM_OPT_TIE_TAU, int(2 ** (30 + tau_log2)))
        b, _ = e.bmu(x)
        print(f"   tau=2^{tau_log2}: mismatches {(b != bo).sum()} rechecks {e.last_recheck_count}")
    e.close()
