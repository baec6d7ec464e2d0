import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2604_26555_b200 as tsom
from paper_2604_26555_b200 import _lib
for d in (50, 54, 55, 60, 63, 64, 65, 80, 100):
    rng = np.random.default_rng(d)
    x = rng.standard_normal((500, d)).astype(np.float32) * 2
    w = rng.standard_normal((64, d)).astype(np.float32) * 2
    bo, do = oracle.port.find_bmus(x, w)
    for kern in (1, 2):
        e = tsom.Engine(64, d)
        try:
            e.set_option(_lib.TSOM_OPT_BMU_KERNEL, kern)
        except Exception as ex:
            continue
        e.set_codebook(w)
        b, dist = e.bmu(x)
        mm = np.flatnonzero(b != bo)
        print(d, kern, "mismatch", len(mm), "rechecks", e.last_recheck_count, "dist err", np.max(np.abs(dist - do) / do), mm[:5], b[mm[:5]], bo[mm[:5]])
