"""Host-side pieces of the training loop that surround the GPU hot path.

These are the cheap, per-run / per-epoch host computations the reference's
``train_with_executor`` performs around ``run_iteration`` (paths relative to
/root/reference/proj/include/toposom).  They are part of the host driver, not a
compute fallback: none of them touches samples.

* :class:`Rng`              — rng.hpp:12-91 (mt19937_64 + splitmix seed streams)
* :func:`init_sample_draw`  — trainer.hpp:192-211 (Floyd pick of P rows)
* :func:`schedule_value`    — trainer.hpp:132-139
* :func:`resolved_sigma0`   — trainer.hpp:75-80
* :func:`lattice_dist`      — topology.hpp:114-149
* :func:`assign_shards`     — parallel.hpp:28-41 (row shards per rank/GPU)
* :class:`RefreshState`     — should_refresh / refresh bookkeeping, topology.hpp:68-72, 423-451
"""
from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1
SEED_STREAM = {"split": 1, "init": 2, "sampler": 3, "synth": 4, "trial": 5}


def mix_seed(seed: int, stream: int) -> int:
    """splitmix64 stream derivation (rng.hpp:12-17)."""
    z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Rng:
    """std::mt19937_64 with the reference's hand-rolled draws (rng.hpp:30-91)."""

    _N, _M = 312, 156

    def __init__(self, seed: int, stream: str | int | None = None):
        if stream is not None:
            s = SEED_STREAM[stream] if isinstance(stream, str) else int(stream)
            seed = mix_seed(seed, s)
        mt = [0] * self._N
        mt[0] = seed & _M64
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt, self.mti = mt, self._N
        self._cached = None

    def _twist(self):
        mt, N, M = self.mt, self._N, self._M
        for i in range(N):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % N] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + M) % N] ^ xa
        self.mti = 0

    def next(self) -> int:
        if self.mti >= self._N:
            self._twist()
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64

    def index(self, n: int) -> int:
        if n < 1:
            raise ValueError("Rng::index: n must be >= 1")
        limit = _M64 - (_M64 % n)
        while True:
            x = self.next()
            if x < limit:
                return x % n

    def real01(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53


def init_sample_draw(data: np.ndarray, nodes: int, seed: int) -> np.ndarray:
    """init_weights(sample_draw) (trainer.hpp:192-211)."""
    n = data.shape[0]
    if n < 1:
        raise ValueError("init_weights: empty training data")
    rng = Rng(seed, "init")
    if nodes <= n:
        chosen: list[int] = []
        seen: set[int] = set()
        for j in range(n - nodes, n):
            t = rng.index(j + 1)
            pick = j if t in seen else t
            chosen.append(pick)
            seen.add(pick)
        picks = chosen
    else:
        picks = [rng.index(n) for _ in range(nodes)]
    return np.ascontiguousarray(data[np.asarray(picks, np.int64)], np.float32)


def schedule_value(v0: float, kind: str, t: int, total: int, floor_v: float) -> float:
    if total < 1:
        raise ValueError("schedule_value: T must be >= 1")
    if t >= total:
        raise ValueError("schedule_value: t must be < T")
    frac = float(t) / float(total)
    v = v0 * (1.0 - frac) if kind == "linear" else v0 * math.exp(-3.0 * frac)
    return max(floor_v, v)


def resolved_sigma0(topology: str, grid_w: int, grid_h: int, sigma0: float = 0.0) -> float:
    if sigma0 > 0.0:
        return sigma0
    if topology in ("rect", "rectangular", "hex", "hexagonal"):
        return max(1.0, float(max(grid_w, grid_h)) / 2.0)
    return 3.0


def lattice_dist(kind: str, width: int, height: int) -> np.ndarray:
    """Euclidean lattice distances (topology.hpp:114-149), float64 P x P."""
    r, c = np.divmod(np.arange(width * height), width)
    if kind in ("rect", "rectangular"):
        xy = np.stack([r.astype(np.float64), c.astype(np.float64)], 1)
    else:
        xy = np.stack([c + np.where(r % 2 == 1, 0.5, 0.0), r * 0.86602540378443864676], 1)
    dx = xy[:, None, 0] - xy[None, :, 0]
    dy = xy[:, None, 1] - xy[None, :, 1]
    out = np.sqrt(dx * dx + dy * dy)
    np.fill_diagonal(out, 0.0)
    return out


def assign_shards(n: int, workers: int) -> list[tuple[int, int]]:
    """Contiguous near-equal partition (parallel.hpp:28-41): the first n % G
    slices get one extra item; a slice may be empty when G > n."""
    if workers < 1:
        raise ValueError("assign_shards: G must be >= 1")
    base, extra = divmod(n, workers)
    out, begin = [], 0
    for g in range(workers):
        cnt = base + (1 if g < extra else 0)
        out.append((begin, begin + cnt))
        begin += cnt
    return out


class RefreshState:
    """Graph refresh schedule (RefreshPolicy topology.hpp:68-72; should_refresh
    :423-435; the counters refresh_topology updates :447-450)."""

    def __init__(self, warmup_iters: int, growth: float = 1.5, max_interval: int = 25):
        if not growth > 1.0:
            raise ValueError("config: refresh growth must be > 1")
        self.warmup, self.growth, self.max_interval = warmup_iters, growth, max_interval
        self.last_refresh_iter = -1
        self.refresh_count = 0
        self.post_warmup_refreshes = 0

    def should_refresh(self, it: int) -> bool:
        if it < self.warmup:
            return True
        raw = math.ceil(math.pow(self.growth, float(self.post_warmup_refreshes)))
        interval = self.max_interval if raw >= float(self.max_interval) else int(raw)
        interval = min(self.max_interval, interval)
        return it - self.last_refresh_iter >= interval

    def mark(self, it: int):
        self.last_refresh_iter = it
        self.refresh_count += 1
        if it >= self.warmup:
            self.post_warmup_refreshes += 1
