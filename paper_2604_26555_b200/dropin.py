"""ctypes binding of libtsom_dropin.so: the reference's own training loop
(toposom::train_with_executor, trainer.hpp:466-523) with the B200
CudaExecutor swapped in (include/toposom_b200/cuda_executor.hpp).

This is the end-to-end public path a reference user takes (``train_cuda``):
host DataMatrix in, trained codebook out, every epoch's data pass on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib

_HERE = os.path.dirname(os.path.abspath(__file__))
DROPIN_PATH = os.path.join(_HERE, "libtsom_dropin.so")

TOPO = {"rect": 0, "rectangular": 0, "hex": 1, "hexagonal": 1, "mst": 2, "rng": 3}
SAMPLING = {"full": 0, "random": 1, "adaptive": 2}
INIT = {"sample_draw": 0, "uniform_box": 1, "pca_plane": 2}


@dataclass
class TrainConfig:
    """SomConfig (trainer.hpp:58-99) + Sampler settings (sampling.hpp:183-221)."""

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
        if TOPO[self.topology] in (0, 1) and not self.nodes:
            self.nodes = self.grid_w * self.grid_h


class _Cfg(C.Structure):
    _fields_ = [("topology", C.c_int), ("grid_w", C.c_uint64), ("grid_h", C.c_uint64),
                ("nodes", C.c_uint64), ("n_iters", C.c_uint64), ("eta0", C.c_double),
                ("lr_exponential", C.c_int), ("sigma0", C.c_double),
                ("radius_exponential", C.c_int), ("sigma_min", C.c_double),
                ("init_method", C.c_int), ("use_momentum", C.c_int), ("momentum", C.c_double),
                ("refresh_warmup", C.c_uint64), ("refresh_growth", C.c_double),
                ("refresh_max_interval", C.c_uint64), ("n_chunks", C.c_uint64),
                ("seed", C.c_uint64), ("sampling", C.c_int), ("budget_fixed", C.c_int),
                ("m0", C.c_uint64), ("rho", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double), ("n_threads", C.c_int)]


def _cfg(c) -> _Cfg:
    return _Cfg(TOPO[c.topology], c.grid_w, c.grid_h, c.nodes, c.n_iters, c.eta0,
                int(c.lr_decay.startswith("exp")), c.sigma0, int(c.radius_decay.startswith("exp")),
                c.sigma_min, INIT[c.init_method], int(c.use_momentum), c.momentum,
                c.refresh_warmup, c.refresh_growth, c.refresh_max_interval, c.n_chunks, c.seed,
                SAMPLING[c.sampling], int(c.budget_fixed), c.m0, c.rho, c.alpha, c.beta,
                c.n_threads)


_dl = None


def load():
    global _dl
    if _dl is None:
        _lib.load()
        if not os.path.exists(DROPIN_PATH):
            raise ImportError(f"{DROPIN_PATH} missing (built where the reference headers exist)")
        L = C.CDLL(DROPIN_PATH)
        L.tsom_dropin_last_error.restype = C.c_char_p
        L.tsom_dropin_config_sizeof.restype = C.c_size_t
        assert L.tsom_dropin_config_sizeof() == C.sizeof(_Cfg), "config layout mismatch"
        L.tsom_dropin_train.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.c_size_t, C.c_size_t,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_uint,
                                        C.POINTER(C.c_double)]
        L.tsom_dropin_run_study.argtypes = [C.POINTER(_Cfg), C.c_size_t, C.c_void_p, C.c_size_t,
                                            C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                            C.c_size_t, C.c_int, C.c_uint, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.POINTER(C.c_double)]
        L.tsom_dropin_find_bmus.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                            C.c_size_t, C.c_void_p, C.c_void_p, C.c_int]
        L.tsom_dropin_train_shards.argtypes = [C.POINTER(_Cfg), C.c_char_p, C.c_size_t,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                               C.c_uint, C.POINTER(C.c_double)]
        L.tsom_dropin_write_shards.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_char_p,
                                               C.c_size_t]
        _dl = L
    return _dl


def available() -> bool:
    return os.path.exists(DROPIN_PATH)


def run_study_cuda(base, n_trials: int, seeds, train: np.ndarray, holdout: np.ndarray,
                   device: int = 0, concurrency: int = 4):
    """run_study (tune.hpp:125-159, default SearchSpace) with every trial trained
    and scored on the GPU (toposom_b200::run_study_cuda), up to `concurrency`
    trials at once.  Returns (qe_train, qe_holdout, failed, seconds), seed-major."""
    L = load()
    train = np.ascontiguousarray(train, np.float32)
    holdout = np.ascontiguousarray(holdout, np.float32)
    seeds = np.ascontiguousarray(seeds, np.uint64)
    k = n_trials * len(seeds)
    qt, qh, fl = np.empty(k), np.empty(k), np.zeros(k, np.uint8)
    secs = C.c_double()
    st = L.tsom_dropin_run_study(C.byref(_cfg(base)), n_trials, seeds.ctypes.data, len(seeds),
                                 train.ctypes.data, train.shape[0], holdout.ctypes.data,
                                 holdout.shape[0], train.shape[1], device, concurrency,
                                 qt.ctypes.data, qh.ctypes.data, fl.ctypes.data, C.byref(secs))
    if st:
        _lib._raise(st, L.tsom_dropin_last_error().decode())
    return qt, qh, fl.astype(bool), secs.value


def _engine_flags(engines: int, exact: bool = False) -> int:
    assert 1 <= engines <= 15
    return ((engines if engines > 1 else 0) << 8) | ((1 if exact else 0) << 28)


def train_device(cfg, data: np.ndarray, device: int = 0, log_qe: bool = False,
                 streamed: bool = False, engines: int = 1, exact: bool = False):
    """toposom_b200::train_device: the reference's epoch loop with every step on
    the device (sampler, refresh, influence, BMU, accumulate, update).  engines
    > 1 splits the rows over that many engines on `device` joined by an
    in-process rank group (the multi-GPU epoch on one GPU).
    Returns (weights, qe_log, refresh_log, seconds)."""
    L = load()
    data = np.ascontiguousarray(data, np.float32)
    n, d = data.shape
    w = np.empty((cfg.nodes, d), np.float32)
    qe = np.zeros(cfg.n_iters) if log_qe else None
    ref = np.zeros(cfg.n_iters, np.uint8)
    secs = (C.c_double * 3)()
    flags = (1 if streamed else 0) | 32 | _engine_flags(engines, exact)
    st = L.tsom_dropin_train(C.byref(_cfg(cfg)), data.ctypes.data, n, d, w.ctypes.data,
                             qe.ctypes.data if log_qe else None, ref.ctypes.data, device, flags,
                             secs)
    if st:
        _lib._raise(st, L.tsom_dropin_last_error().decode())
    return w, qe, ref, secs[0]


def train_cuda(cfg, data: np.ndarray, device: int = 0, log_qe: bool = False,
               streamed: bool = False, bmu_kernel: int = 0, force_distances: bool = False,
               profile: bool = False, engines: int = 1, exact: bool = False):
    """Reference train_with_executor + CudaExecutor.  Returns (weights, qe_log, refresh_log, s);
    with profile=True, s = (total, executor construction incl. bind, sum of run_iteration).
    engines > 1: the executor splits the rows over that many engines (the
    ThreadedExecutor shape, parallel.hpp:99-140, with engines as workers)."""
    L = load()
    data = np.ascontiguousarray(data, np.float32)
    n, d = data.shape
    w = np.empty((cfg.nodes, d), np.float32)
    qe = np.zeros(cfg.n_iters) if log_qe else None
    ref = np.zeros(cfg.n_iters, np.uint8)
    secs = (C.c_double * 3)()
    flags = ((1 if streamed else 0) | ((bmu_kernel & 3) << 1) | (8 if force_distances else 0)
             | (16 if profile else 0) | _engine_flags(engines, exact))
    st = L.tsom_dropin_train(C.byref(_cfg(cfg)), data.ctypes.data, n, d, w.ctypes.data,
                             qe.ctypes.data if log_qe else None, ref.ctypes.data, device, flags,
                             secs)
    if st:
        _lib._raise(st, L.tsom_dropin_last_error().decode())
    return w, qe, ref, (tuple(secs) if profile else secs[0])


def train_cuda_shards(cfg, shard_dir: str, d: int, device: int = 0, log_qe: bool = False,
                      streamed: bool = True, bmu_kernel: int = 0, chunk_rows: int = 65536):
    """Reference train_with_executor over open_shards(shard_dir) (dataset.hpp:277-302)
    with the CudaExecutor reading the shard files itself."""
    L = load()
    w = np.empty((cfg.nodes, d), np.float32)
    qe = np.zeros(cfg.n_iters) if log_qe else None
    ref = np.zeros(cfg.n_iters, np.uint8)
    secs = C.c_double()
    flags = (1 if streamed else 0) | ((bmu_kernel & 3) << 1)
    st = L.tsom_dropin_train_shards(C.byref(_cfg(cfg)), os.fsencode(shard_dir), chunk_rows,
                                    w.ctypes.data, qe.ctypes.data if log_qe else None,
                                    ref.ctypes.data, device, flags, C.byref(secs))
    if st:
        _lib._raise(st, L.tsom_dropin_last_error().decode())
    return w, qe, ref, secs.value


def write_shards(data: np.ndarray, out_dir: str, n_shards: int):
    """The reference's own write_shards (dataset.hpp:252-275)."""
    L = load()
    data = np.ascontiguousarray(data, np.float32)
    st = L.tsom_dropin_write_shards(data.ctypes.data, data.shape[0], data.shape[1],
                                    os.fsencode(out_dir), n_shards)
    if st:
        _lib._raise(st, L.tsom_dropin_last_error().decode())
