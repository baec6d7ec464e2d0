"""CPU checkers for the B200 batch-SOM engine.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product (``paper_2604_26555_b200``) never imports it and has no
CPU fallback.

Two checkers share one numpy-facing API:

* :data:`port` — ``liboracle.so``, a C restatement of the reference hot path
  (``oracle/tsom_oracle.c``; every function cites the reference file:line).
* :data:`ref`  — ``_ref/libtoposom_ref.so``, the reference headers themselves
  compiled by ``oracle/Makefile`` (present when the reference tree was
  available at build time; the built file travels to the GPU box).

Both are pinned against the reference's own known-answer tests in
``tests/test_oracle.py``, and against each other bit-for-bit.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libtoposom_ref.so")

TOPO = {"rect": 0, "rectangular": 0, "hex": 1, "hexagonal": 1, "mst": 2, "rng": 3}
SAMPLING = {"full": 0, "random": 1, "adaptive": 2}
INIT = {"sample_draw": 0, "uniform_box": 1, "pca_plane": 2}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


@dataclass
class SomConfig:
    """Mirror of ``SomConfig`` (trainer.hpp:58-99) + sampler settings."""

    topology: str = "hex"
    grid_w: int = 0
    grid_h: int = 0
    nodes: int = 0
    n_iters: int = 10
    eta0: float = 0.5
    lr_decay: str = "linear"
    sigma0: float = 0.0
    radius_decay: str = "linear"
    sigma_min: float = 0.3
    init_method: str = "sample_draw"
    use_momentum: bool = False
    momentum: float = 0.5
    refresh_warmup: int = 0
    refresh_growth: float = 1.5
    refresh_max_interval: int = 25
    n_chunks: int = 1
    seed: int = 0
    sampling: str = "full"
    budget_fixed: bool = False
    m0: int = 0
    rho: float = 1.0
    alpha: float = 1.0
    beta: float = 1.0
    n_threads: int = 1

    def __post_init__(self):
        if self.topology in ("rect", "rectangular", "hex", "hexagonal") and not self.nodes:
            self.nodes = self.grid_w * self.grid_h

    @property
    def is_lattice(self) -> bool:
        return TOPO[self.topology] in (0, 1)


class _Cfg(C.Structure):
    _fields_ = [
        ("topology", C.c_int),
        ("grid_w", C.c_uint64),
        ("grid_h", C.c_uint64),
        ("nodes", C.c_uint64),
        ("n_iters", C.c_uint64),
        ("eta0", C.c_double),
        ("lr_exponential", C.c_int),
        ("sigma0", C.c_double),
        ("radius_exponential", C.c_int),
        ("sigma_min", C.c_double),
        ("init_method", C.c_int),
        ("use_momentum", C.c_int),
        ("momentum", C.c_double),
        ("refresh_warmup", C.c_uint64),
        ("refresh_growth", C.c_double),
        ("refresh_max_interval", C.c_uint64),
        ("n_chunks", C.c_uint64),
        ("seed", C.c_uint64),
        ("sampling", C.c_int),
        ("budget_fixed", C.c_int),
        ("m0", C.c_uint64),
        ("rho", C.c_double),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("n_threads", C.c_int),
    ]


def _to_cfg(c: SomConfig) -> _Cfg:
    return _Cfg(
        TOPO[c.topology], c.grid_w, c.grid_h, c.nodes, c.n_iters, c.eta0,
        int(c.lr_decay.startswith("exp")), c.sigma0, int(c.radius_decay.startswith("exp")),
        c.sigma_min, INIT[c.init_method], int(c.use_momentum), c.momentum, c.refresh_warmup,
        c.refresh_growth, c.refresh_max_interval, c.n_chunks, c.seed, SAMPLING[c.sampling],
        int(c.budget_fixed), c.m0, c.rho, c.alpha, c.beta, c.n_threads)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def int128_from_pairs(raw: np.ndarray) -> list[int]:
    """(hi, lo) int64 pairs → Python ints (exact int128 values)."""
    raw = raw.reshape(-1, 2)
    return [(int(h) << 64) | (int(l) & 0xFFFFFFFFFFFFFFFF) for h, l in raw]


class _Checker:
    """Common numpy API over either library; ``kind`` is "port" or "reference"."""

    kind = "port"

    def __init__(self, path: str):
        self.path = path
        self._lib = None

    @property
    def available(self) -> bool:
        return os.path.exists(self.path)

    @property
    def lib(self):
        if self._lib is None:
            if not self.available:
                raise OracleError(-1, f"{self.path} not built (run `make -C oracle`)")
            self._lib = C.CDLL(self.path)
            self._bind(self._lib)
        return self._lib


class PortChecker(_Checker):
    kind = "port"

    def _bind(self, L):
        sz = C.c_size_t
        L.orc_config_sizeof.restype = sz
        assert L.orc_config_sizeof() == C.sizeof(_Cfg), "orc_config layout mismatch"
        L.orc_synth_gmm.argtypes = [_f32p, sz, sz, C.c_uint64, sz, C.c_void_p]
        L.orc_synth_uniform.argtypes = [_f32p, sz, sz, C.c_uint64]
        L.orc_synth_rings.argtypes = [_f32p, sz, C.c_double, C.c_uint64]
        L.orc_find_bmus.argtypes = [_f32p, sz, _f32p, sz, sz, _u32p, _f64p]
        L.orc_mean_bmu_distance.argtypes = [_f32p, sz, _f32p, sz, sz]
        L.orc_mean_bmu_distance.restype = C.c_double
        L.orc_accumulate_selection.argtypes = [_f32p, sz, _u32p, sz, _f32p, sz, sz, _f64p,
                                               C.c_double, sz, C.c_int, _f64p, _f64p, _i64p,
                                               _i64p, C.c_void_p]
        L.orc_apply_update.argtypes = [_f32p, _f32p, sz, sz, _f64p, _f64p, C.c_int, C.c_double,
                                       C.POINTER(C.c_int64)]
        L.orc_schedule_value.argtypes = [C.c_double, C.c_int, sz, sz, C.c_double]
        L.orc_schedule_value.restype = C.c_double
        L.orc_lattice_dist.argtypes = [C.c_int, sz, sz, _f64p]
        L.orc_influence_from_dist.argtypes = [_f64p, sz, C.c_double, _f64p]
        L.orc_influence_from_hops.argtypes = [_u16p, sz, C.c_double, _f64p]
        L.orc_pairwise_sq_dists.argtypes = [_f32p, sz, sz, _f64p]
        L.orc_build_mst.argtypes = [_f64p, sz, _u32p]
        L.orc_build_mst.restype = sz
        L.orc_build_rng_graph.argtypes = [_f64p, sz, _u32p]
        L.orc_build_rng_graph.restype = sz
        L.orc_hop_distances.argtypes = [_u32p, sz, sz, _u16p]
        L.orc_quantize_term.argtypes = [C.c_double, C.POINTER(C.c_int)]
        L.orc_quantize_term.restype = C.c_int64
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_rng_sizeof.restype = sz
        L.orc_rng_init_stream.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.orc_rng_init.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_gaussian.argtypes = [C.c_void_p]
        L.orc_rng_gaussian.restype = C.c_double
        L.orc_select_random.argtypes = [sz, sz, C.c_void_p, _u32p]
        L.orc_select_adaptive.argtypes = [_f64p, _u32p, sz, C.c_double, C.c_double, sz,
                                          C.c_void_p, _u32p]
        L.orc_update_adaptive.argtypes = [_f64p, _u32p, sz, _u32p, sz, _f64p]
        L.orc_init_sample_draw.argtypes = [_f32p, sz, sz, sz, C.c_uint64, _f32p]
        L.orc_train.argtypes = [C.POINTER(_Cfg), _f32p, sz, sz, _f32p, C.c_void_p, C.c_void_p]

    # --- data -------------------------------------------------------------
    def synth_gmm(self, n, d=50, seed=2604, n_comp=16):
        out = np.empty((n, d), np.float32)
        self.lib.orc_synth_gmm(out, n, d, seed, n_comp, None)
        return out

    def synth_uniform(self, n, d, seed):
        out = np.empty((n, d), np.float32)
        self.lib.orc_synth_uniform(out, n, d, seed)
        return out

    def synth_rings(self, n, noise, seed):
        out = np.empty((n, 2), np.float32)
        self.lib.orc_synth_rings(out, n, noise, seed)
        return out

    def rng_draws(self, seed, stream, n):
        L = self.lib
        buf = C.create_string_buffer(L.orc_rng_sizeof())
        L.orc_rng_init_stream(buf, seed, stream)
        nxt = np.array([L.orc_rng_next(buf) for _ in range(n)], np.uint64)
        L.orc_rng_init_stream(buf, seed, stream)
        gs = np.array([L.orc_rng_gaussian(buf) for _ in range(n)], np.float64)
        return nxt, gs

    def mt19937_64_default(self, k):
        """k-th output of a default-seeded (5489) mt19937_64."""
        L = self.lib
        buf = C.create_string_buffer(L.orc_rng_sizeof())
        L.orc_rng_init(buf, 5489)
        x = 0
        for _ in range(k):
            x = L.orc_rng_next(buf)
        return x

    # --- hot path ---------------------------------------------------------
    def find_bmus(self, x, w):
        x, w = _f32(x), _f32(w)
        n, d = x.shape
        bm = np.empty(n, np.uint32)
        dist = np.empty(n, np.float64)
        self.lib.orc_find_bmus(x, n, w, w.shape[0], d, bm, dist)
        return bm, dist

    def mean_bmu_distance(self, x, w):
        x, w = _f32(x), _f32(w)
        return self.lib.orc_mean_bmu_distance(x, x.shape[0], w, w.shape[0], x.shape[1])

    def run_iteration(self, data, selected, w, influence, eta, n_chunks=1, workers=1):
        """Returns (U[P,d] f64, H[P] f64, U_raw int128 pairs, H_raw, distances)."""
        data, w, infl, sel = _f32(data), _f32(w), _f64(influence), _u32(selected)
        p, d = w.shape
        u = np.zeros((p, d)); h = np.zeros(p)
        ur = np.zeros(2 * p * d, np.int64); hr = np.zeros(2 * p, np.int64)
        dist = np.zeros(max(len(sel), 1))
        st = self.lib.orc_accumulate_selection(data, data.shape[0], sel, len(sel), w, p, d, infl,
                                               float(eta), n_chunks, workers, u, h, ur, hr,
                                               dist.ctypes.data)
        if st:
            raise OracleError(st, "numerical fault" if st == 2 else "out of range")
        return u, h, ur, hr, dist[:len(sel)]

    def apply_update(self, w, prev, u, h, use_momentum=False, momentum=0.5):
        w, prev = _f32(w).copy(), _f32(prev).copy()
        bad = C.c_int64(-1)
        st = self.lib.orc_apply_update(w, prev, w.shape[0], w.shape[1], _f64(u), _f64(h),
                                       int(use_momentum), momentum, C.byref(bad))
        if st:
            raise OracleError(st, f"numerical fault: non-finite weight update at node {bad.value}")
        return w, prev

    def schedule_value(self, v0, kind, t, total, floor_v):
        return self.lib.orc_schedule_value(v0, int(kind.startswith("exp")), t, total, floor_v)

    def lattice_dist(self, kind, w, h):
        out = np.empty((w * h, w * h))
        self.lib.orc_lattice_dist(TOPO[kind], w, h, out)
        return out

    def influence_from_dist(self, dist, sigma):
        dist = _f64(dist)
        out = np.empty_like(dist)
        self.lib.orc_influence_from_dist(dist, dist.size, sigma, out)
        return out

    def influence_from_hops(self, hops, sigma):
        hops = np.ascontiguousarray(hops, np.uint16)
        out = np.empty(hops.shape)
        self.lib.orc_influence_from_hops(hops, hops.size, sigma, out)
        return out

    def pairwise_sq_dists(self, w):
        w = _f32(w)
        out = np.empty((w.shape[0], w.shape[0]))
        self.lib.orc_pairwise_sq_dists(w, w.shape[0], w.shape[1], out)
        return out

    def build_graph(self, kind, sq):
        sq = _f64(sq)
        p = sq.shape[0]
        edges = np.zeros(max(2, p * (p - 1)), np.uint32)
        if kind == "mst":
            ne = self.lib.orc_build_mst(sq, p, edges)
        else:
            ne = self.lib.orc_build_rng_graph(sq, p, edges)
        return edges[: 2 * ne].reshape(-1, 2)

    def hop_distances(self, edges, p):
        edges = _u32(edges)
        out = np.empty((p, p), np.uint16)
        st = self.lib.orc_hop_distances(edges, edges.size // 2, p, out)
        if st:
            raise OracleError(st, "hop_distances: graph is disconnected")
        return out

    def quantize_term(self, term):
        st = C.c_int(0)
        q = self.lib.orc_quantize_term(term, C.byref(st))
        if st.value:
            raise OracleError(st.value, "numerical fault: accumulation term out of range (|term| >= 2^22)")
        return q

    def train(self, cfg: SomConfig, data, log_qe=False):
        data = _f32(data)
        n, d = data.shape
        w = np.empty((cfg.nodes, d), np.float32)
        qe = np.zeros(cfg.n_iters) if log_qe else None
        ref = np.zeros(cfg.n_iters, np.uint8)
        st = self.lib.orc_train(C.byref(_to_cfg(cfg)), data, n, d, w,
                                qe.ctypes.data if log_qe else None, ref.ctypes.data)
        if st:
            raise OracleError(st, "train failed")
        return w, qe, ref


class RefChecker(PortChecker):
    """The reference itself (oracle/_ref).  Same Python API as the port."""

    kind = "reference"

    def _bind(self, L):
        sz = C.c_size_t
        L.ref_last_error.restype = C.c_char_p
        L.ref_config_sizeof.restype = sz
        assert L.ref_config_sizeof() == C.sizeof(_Cfg), "ref_config layout mismatch"
        L.ref_find_bmus.argtypes = [_f32p, sz, _f32p, sz, sz, _u32p, _f64p]
        L.ref_mean_bmu_distance.argtypes = [_f32p, sz, _f32p, sz, sz, C.POINTER(C.c_double)]
        L.ref_run_iteration.argtypes = [_f32p, sz, sz, _u32p, sz, _f32p, sz, _f64p, C.c_double,
                                        sz, sz, _f64p, _f64p, _i64p, _i64p, C.c_void_p]
        L.ref_apply_update.argtypes = [_f32p, _f32p, sz, sz, _i64p, _i64p, C.c_int, C.c_double]
        L.ref_lattice_dist.argtypes = [C.c_int, sz, sz, _f64p]
        L.ref_influence_from_dist.argtypes = [_f64p, sz, C.c_double, _f64p]
        L.ref_influence_from_hops.argtypes = [_u16p, sz, C.c_double, _f64p]
        L.ref_pairwise_sq_dists.argtypes = [_f32p, sz, sz, _f64p]
        L.ref_build_graph.argtypes = [C.c_int, _f64p, sz, _u32p, C.POINTER(C.c_size_t)]
        L.ref_hop_distances.argtypes = [_u32p, sz, sz, _u16p]
        L.ref_synth_gmm.argtypes = [_f32p, sz, sz, C.c_uint64, sz]
        L.ref_synth_uniform.argtypes = [_f32p, sz, sz, C.c_uint64]
        L.ref_synth_rings.argtypes = [_f32p, sz, C.c_double, C.c_uint64]
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_uint64, sz, np.ctypeslib.ndpointer(np.uint64), _f64p]
        L.ref_sampler_run.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, sz, C.c_uint64,
                                      C.c_double, C.c_double, sz, C.c_void_p, _u32p,
                                      np.ctypeslib.ndpointer(np.uintp)]
        L.ref_train.argtypes = [C.POINTER(_Cfg), _f32p, sz, sz, _f32p, C.c_void_p, C.c_void_p]
        L.ref_run_study.argtypes = [C.POINTER(_Cfg), sz, np.ctypeslib.ndpointer(np.uint64), sz,
                                    _f32p, sz, _f32p, sz, sz, _f64p, _f64p,
                                    np.ctypeslib.ndpointer(np.uint8)]

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def synth_gmm(self, n, d=50, seed=2604, n_comp=16):
        out = np.empty((n, d), np.float32)
        self._check(self.lib.ref_synth_gmm(out, n, d, seed, n_comp))
        return out

    def synth_uniform(self, n, d, seed):
        out = np.empty((n, d), np.float32)
        self._check(self.lib.ref_synth_uniform(out, n, d, seed))
        return out

    def synth_rings(self, n, noise, seed):
        out = np.empty((n, 2), np.float32)
        self._check(self.lib.ref_synth_rings(out, n, noise, seed))
        return out

    def rng_draws(self, seed, stream, n):
        nxt = np.empty(n, np.uint64)
        gs = np.empty(n)
        self._check(self.lib.ref_rng_draws(seed, stream, n, nxt, gs))
        return nxt, gs

    def find_bmus(self, x, w):
        x, w = _f32(x), _f32(w)
        n, d = x.shape
        bm = np.empty(n, np.uint32)
        dist = np.empty(n, np.float64)
        self._check(self.lib.ref_find_bmus(x, n, w, w.shape[0], d, bm, dist))
        return bm, dist

    def mean_bmu_distance(self, x, w):
        x, w = _f32(x), _f32(w)
        out = C.c_double()
        self._check(self.lib.ref_mean_bmu_distance(x, x.shape[0], w, w.shape[0], x.shape[1],
                                                   C.byref(out)))
        return out.value

    def run_iteration(self, data, selected, w, influence, eta, n_chunks=1, workers=1):
        data, w, infl, sel = _f32(data), _f32(w), _f64(influence), _u32(selected)
        p, d = w.shape
        u = np.zeros((p, d)); h = np.zeros(p)
        ur = np.zeros(2 * p * d, np.int64); hr = np.zeros(2 * p, np.int64)
        dist = np.zeros(max(len(sel), 1))
        self._check(self.lib.ref_run_iteration(data, data.shape[0], d, sel, len(sel), w, p, infl,
                                               float(eta), n_chunks, workers, u, h, ur, hr,
                                               dist.ctypes.data))
        return u, h, ur, hr, dist[:len(sel)]

    def apply_update_raw(self, w, prev, u_raw, h_raw, use_momentum=False, momentum=0.5):
        w, prev = _f32(w).copy(), _f32(prev).copy()
        self._check(self.lib.ref_apply_update(w, prev, w.shape[0], w.shape[1],
                                              np.ascontiguousarray(u_raw, np.int64),
                                              np.ascontiguousarray(h_raw, np.int64),
                                              int(use_momentum), momentum))
        return w, prev

    def lattice_dist(self, kind, w, h):
        out = np.empty((w * h, w * h))
        self._check(self.lib.ref_lattice_dist(TOPO[kind], w, h, out))
        return out

    def influence_from_dist(self, dist, sigma):
        dist = _f64(dist)
        out = np.empty_like(dist)
        self._check(self.lib.ref_influence_from_dist(dist, dist.size, sigma, out))
        return out

    def influence_from_hops(self, hops, sigma):
        hops = np.ascontiguousarray(hops, np.uint16)
        out = np.empty(hops.shape)
        self._check(self.lib.ref_influence_from_hops(hops, hops.size, sigma, out))
        return out

    def pairwise_sq_dists(self, w):
        w = _f32(w)
        out = np.empty((w.shape[0], w.shape[0]))
        self._check(self.lib.ref_pairwise_sq_dists(w, w.shape[0], w.shape[1], out))
        return out

    def build_graph(self, kind, sq):
        sq = _f64(sq)
        p = sq.shape[0]
        cap = max(1, p * (p - 1) // 2)
        edges = np.zeros(2 * cap, np.uint32)
        ne = C.c_size_t(cap)
        self._check(self.lib.ref_build_graph(TOPO[kind], sq, p, edges, C.byref(ne)))
        return edges[: 2 * ne.value].reshape(-1, 2)

    def hop_distances(self, edges, p):
        edges = _u32(edges)
        out = np.empty((p, p), np.uint16)
        self._check(self.lib.ref_hop_distances(edges, edges.size // 2, p, out))
        return out

    def sampler_run(self, kind, n, seed, iters, rho=1.0, m0=0, budget_fixed=False, alpha=1.0,
                    beta=1.0, dist_by_row=None):
        m = m0 if budget_fixed else max(1, int(np.floor(n * rho)))
        out = np.zeros(iters * max(m, n if kind == "full" else m), np.uint32)
        ms = np.zeros(iters, np.uintp)
        db = None if dist_by_row is None else _f64(dist_by_row)
        self._check(self.lib.ref_sampler_run(SAMPLING[kind], int(budget_fixed), m0, rho, n, seed,
                                             alpha, beta, iters,
                                             None if db is None else db.ctypes.data, out, ms))
        res, off = [], 0
        for t in range(iters):
            res.append(out[off: off + int(ms[t])].copy())
            off += int(ms[t])
        return res

    def run_study(self, base: SomConfig, n_trials, seeds, train, holdout):
        """run_study (tune.hpp:125-159) with the default SearchSpace: per trial
        (seed-major) qe_train, qe_holdout, failed."""
        train, holdout = _f32(train), _f32(holdout)
        seeds = np.ascontiguousarray(seeds, np.uint64)
        k = n_trials * len(seeds)
        qt, qh, fl = np.empty(k), np.empty(k), np.zeros(k, np.uint8)
        self._check(self.lib.ref_run_study(C.byref(_to_cfg(base)), n_trials, seeds, len(seeds),
                                           train, train.shape[0], holdout, holdout.shape[0],
                                           train.shape[1], qt, qh, fl))
        return qt, qh, fl.astype(bool)

    def train(self, cfg: SomConfig, data, log_qe=False):
        data = _f32(data)
        n, d = data.shape
        w = np.empty((cfg.nodes, d), np.float32)
        qe = np.zeros(cfg.n_iters) if log_qe else None
        ref = np.zeros(cfg.n_iters, np.uint8)
        self._check(self.lib.ref_train(C.byref(_to_cfg(cfg)), data, n, d, w,
                                       qe.ctypes.data if log_qe else None, ref.ctypes.data))
        return w, qe, ref


port = PortChecker(PORT_PATH)
ref = RefChecker(REF_PATH)


def best():
    """The reference itself when built, else the C restatement."""
    return ref if ref.available else port
