"""Reference-shaped Python API over the B200 engine.

Mirrors the toposom free functions and the Executor seam (paths relative to
/root/reference/proj/include/toposom):

* :func:`find_bmus`            — trainer.hpp:282-308
* :func:`map_samples`          — trainer.hpp:534-541
* :func:`mean_bmu_distance`    — trainer.hpp:377-398 (= quantization_error, metrics.hpp:28-30)
* :class:`CudaExecutor`        — the Executor concept (trainer.hpp:440-460, parallel.hpp:99-140)
* :func:`train_resident`       — train_with_executor (trainer.hpp:466-523) for lattice
                                 topologies with every per-epoch step on the device

Errors follow the reference's exception types: ``ValueError`` for
std::invalid_argument, ``IndexError`` for std::out_of_range and
:class:`NumericalFault` (a RuntimeError) for "numerical fault: ...".
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._lib import Engine, InvalidArgument, NumericalFault, OutOfRange  # noqa: F401
from .hostref import (RefreshState, Rng, init_sample_draw, lattice_dist,  # noqa: F401
                      resolved_sigma0, schedule_value)


def _as_rows(a) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float32)
    if a.ndim != 2:
        raise InvalidArgument(1, "DataMatrix: expected a 2-D rows x cols array")
    return a


def find_bmus(chunk, weights, device: int = 0):
    """BMU index (ties → lowest node) and Euclidean distance per row."""
    chunk, weights = _as_rows(chunk), _as_rows(weights)
    if chunk.shape[1] != weights.shape[1]:
        raise InvalidArgument(1, "find_bmus: dimension mismatch")
    with Engine(weights.shape[0], weights.shape[1], device) as eng:
        eng.set_codebook(weights)
        return eng.bmu(chunk, want_dist=True)


def map_samples(weights, data, device: int = 0):
    data = _as_rows(data)
    if data.shape[0] == 0:
        return np.empty(0, np.uint32), np.empty(0)
    return find_bmus(data, weights, device)


def mean_bmu_distance(data, weights, device: int = 0) -> float:
    data, weights = _as_rows(data), _as_rows(weights)
    if data.shape[1] != weights.shape[1]:
        raise InvalidArgument(1, "mean_bmu_distance: dimension mismatch")
    if data.shape[0] == 0:
        raise InvalidArgument(1, "mean_bmu_distance: empty data")
    with Engine(weights.shape[0], weights.shape[1], device) as eng:
        eng.set_codebook(weights)
        eng.bind(data)
        s, c = eng.qe()
    return s / c


quantization_error = mean_bmu_distance


@dataclass
class Accumulators:
    """Float64 view of ``IterationAccumulators`` (accum.hpp:45-69)."""

    u: np.ndarray  # P x d
    h: np.ndarray  # P

    def u_value(self, node: int, k: int) -> float:
        return float(self.u[node, k])

    def h_value(self, node: int) -> float:
        return float(self.h[node])


class CudaExecutor:
    """Drop-in for SerialExecutor / ThreadedExecutor (trainer.hpp:440-460).

    ``run_iteration`` has the reference call shape; ``n_chunks`` is accepted and
    ignored because the result is chunk-invariant by contract (test_trainer.cpp:315-333).
    """

    def __init__(self, data, nodes: int, device: int = 0, streamed: bool = False):
        data = _as_rows(data)
        self.engine = Engine(nodes, data.shape[1], device)
        self.engine.bind(data, streamed=streamed)
        self._infl = None  # host copy of the influence matrix last uploaded

    def run_iteration(self, selected, weights, influence, eta, n_chunks=1, distances=None):
        eng = self.engine
        eng.set_codebook(weights)
        # upload only when the matrix changed: compared by content (an object
        # identity key would miss a matrix updated in place, or a new temporary
        # that reuses a freed object's address)
        infl = np.ascontiguousarray(influence, np.float64)
        if self._infl is None or not np.array_equal(infl, self._infl):
            eng.set_influence(infl, -1)
            self._infl = infl.copy()
        want = distances is not None
        sel = None if selected is None else np.asarray(selected, np.uint32)
        u, h, d = eng.epoch(eta, sel, want_dist=want)
        if want:
            distances.clear()
            distances.extend(d.tolist())
        return Accumulators(u, h)

    def workers(self) -> int:
        return 1

    def barrier_wait_s(self) -> float:
        return self.engine.barrier_wait_s


@dataclass
class ResidentConfig:
    """Subset of SomConfig (trainer.hpp:58-99) the device-resident loop supports
    (lattices, or MST/RNG graphs refreshed on the device; full, random or
    adaptive sampling by the device sampler, sampling.hpp:183-221)."""

    topology: str = "hex"       # "rect" | "hex" | "mst" | "rng"
    grid_w: int = 32
    grid_h: int = 32
    graph_nodes: int = 0        # graph kinds: node count
    refresh_warmup: int = 0     # 0 = auto: 10% of n_iters (trainer.hpp:81-85)
    refresh_growth: float = 1.5
    refresh_max_interval: int = 25
    n_iters: int = 10
    eta0: float = 0.5
    lr_decay: str = "linear"
    sigma0: float = 0.0
    radius_decay: str = "linear"
    sigma_min: float = 0.3
    use_momentum: bool = False
    momentum: float = 0.5
    seed: int = 0
    sampling: str = "full"      # "full" | "random" | "adaptive"
    rho: float = 1.0            # proportional budget (resolve_budget, sampling.hpp:30-40)
    m0: int = 0                 # fixed budget when budget_fixed
    budget_fixed: bool = False
    alpha: float = 1.0          # adaptive difficulty / staleness exponents
    beta: float = 1.0

    @property
    def lattice(self) -> bool:
        return self.topology in ("rect", "rectangular", "hex", "hexagonal")

    @property
    def nodes(self) -> int:
        return self.grid_w * self.grid_h if self.lattice else self.graph_nodes


def resolve_budget(cfg, n: int) -> int:
    """resolve_budget (sampling.hpp:30-40)."""
    if n < 1:
        raise InvalidArgument(1, "resolve_budget: N must be >= 1")
    if cfg.budget_fixed:
        if cfg.m0 == 0:
            raise InvalidArgument(1, "resolve_budget: fixed budget m0 must be >= 1")
        return int(cfg.m0)
    if not (0.0 < cfg.rho <= 1.0):
        raise InvalidArgument(1, "resolve_budget: rho must be in (0, 1]")
    return max(1, int(math.floor(n * cfg.rho)))


def train_resident(cfg: ResidentConfig, engine: Engine, init_weights=None, log_qe=False):
    """train_with_executor (trainer.hpp:466-523) with full sampling, every epoch on
    the device: topology refresh (graphs, on the schedule of should_refresh),
    influence, BMU, accumulate, allreduce, smoothing, update.  The host only
    evaluates the schedules.  Returns the per-iteration log."""
    if init_weights is None:
        raise InvalidArgument(1, "train_resident: pass init weights (init_sample_draw)")
    engine.set_codebook(init_weights)
    refresh = None
    if cfg.lattice:
        engine.set_topology_distance(lattice_dist(cfg.topology, cfg.grid_w, cfg.grid_h))
    elif cfg.topology in ("mst", "rng"):
        warm = cfg.refresh_warmup if cfg.refresh_warmup else cfg.n_iters // 10
        refresh = RefreshState(warm, cfg.refresh_growth, cfg.refresh_max_interval)
    else:
        raise InvalidArgument(1, f"unknown topology kind: '{cfg.topology}'")
    sigma0 = resolved_sigma0(cfg.topology, cfg.grid_w, cfg.grid_h, cfg.sigma0)
    sampled = cfg.sampling != "full"
    if sampled:
        engine.sampler_init(cfg.sampling, resolve_budget(cfg, engine.rows), cfg.seed, cfg.alpha,
                            cfg.beta)
    # the schedules and the refresh points depend only on t, so the epochs
    # between two refreshes (all of them for lattices) go to the device in one
    # tsom_train_epochs call; with log_qe every epoch is its own call
    log = []
    for t in range(cfg.n_iters):
        refreshed = refresh is not None and refresh.should_refresh(t)
        if refreshed:
            refresh.mark(t)
        log.append({"iter": t, "refreshed": refreshed,
                    "eta": schedule_value(cfg.eta0, cfg.lr_decay, t, cfg.n_iters, 1e-4),
                    "sigma": schedule_value(sigma0, cfg.radius_decay, t, cfg.n_iters,
                                            cfg.sigma_min)})
    t = 0
    while t < cfg.n_iters:
        if log[t]["refreshed"]:
            engine.refresh_topology(cfg.topology)  # from the current device codebook
        t1 = t + 1
        if not log_qe:
            while t1 < cfg.n_iters and not log[t1]["refreshed"]:
                t1 += 1
        seg = log[t:t1]
        engine.train_epochs([e["eta"] for e in seg], [e["sigma"] for e in seg], cfg.momentum,
                            cfg.use_momentum, sampled=sampled)
        if log_qe:
            s, c = engine.qe()
            log[t]["qe_train"] = s / c
        t = t1
    return log


__all__ = ["find_bmus", "map_samples", "mean_bmu_distance", "quantization_error",
           "CudaExecutor", "Accumulators", "ResidentConfig", "train_resident", "Engine",
           "NumericalFault", "InvalidArgument", "OutOfRange", "Rng", "init_sample_draw",
           "schedule_value", "lattice_dist", "resolve_budget", "math"]
