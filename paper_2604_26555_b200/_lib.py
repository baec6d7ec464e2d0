"""ctypes binding of the tsom_* C-ABI (include/tsom_b200.h).

This is the binding a Python maintainer of the reference would add; it loads
the in-tree ``libtsom_b200.so`` and raises if it is missing — there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtsom_b200.so")

TSOM_OK = 0
TSOM_ERR_INVALID = 1
TSOM_ERR_NUMERICAL = 2
TSOM_ERR_RANGE = 3
TSOM_ERR_CUDA = 4
TSOM_ERR_NCCL = 5
TSOM_ERR_TIMEOUT = 6

TSOM_BIND_COPY = 0
TSOM_BIND_STREAMED = 1

TSOM_OPT_BMU_KERNEL = 1
TSOM_OPT_TIE_TAU = 2
TSOM_OPT_STREAM_CHUNK = 3
TSOM_OPT_DETERMINISTIC = 4
TSOM_OPT_HOST_REGISTER = 5
TSOM_OPT_STAGING_THREADS = 6
TSOM_OPT_BARRIER_TIMEOUT_MS = 7
TSOM_OPT_PAD_ROWS = 8
TSOM_OPT_ROW_ORDER = 9

# Every symbol include/tsom_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "tsom_create", "tsom_destroy", "tsom_last_error", "tsom_version", "tsom_set_option",
    "tsom_bind_host_data", "tsom_bind_device_data", "tsom_bind_synthetic_gmm", "tsom_rows",
    "tsom_set_codebook", "tsom_get_codebook", "tsom_set_influence", "tsom_epoch", "tsom_bmu",
    "tsom_bmu_bound", "tsom_qe", "tsom_set_topology_distance", "tsom_train_epoch",
    "tsom_last_recheck_count", "tsom_comm_unique_id", "tsom_comm_init", "tsom_last_timing",
    "tsom_stream", "tsom_last_timing_detail", "tsom_kernel_launches", "tsom_refresh_topology",
    "tsom_pairwise_sq_dists", "tsom_bind_shards", "tsom_active_bmu_kernel",
    "tsom_sampler_init", "tsom_sampler_select", "tsom_sampler_observe", "tsom_sampler_state",
    "tsom_mt_selftest", "tsom_release_cached_memory", "tsom_train_epochs",
    "tsom_get_prev_update", "tsom_barrier_wait_s", "tsom_group_create", "tsom_group_join",
    "tsom_group_destroy", "tsom_device_bytes", "tsom_synth_gmm_host", "tsom_get_rows",
]

SAMPLER_KINDS = {"full": 0, "random": 1, "adaptive": 2}  # SamplingKind, sampling.hpp:163


class TsomError(RuntimeError):
    """Error from the engine; ``status`` is the C-ABI code."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class InvalidArgument(TsomError, ValueError):
    pass


class NumericalFault(TsomError):
    pass


class OutOfRange(TsomError, IndexError):
    pass


class BarrierTimeout(TsomError):
    """A rank missed the reduce barrier's deadline (collect_with_barrier,
    parallel.hpp:67-86: std::runtime_error "reduce barrier timed out ...")."""


def _raise(status: int, msg: str):
    cls = {TSOM_ERR_INVALID: InvalidArgument, TSOM_ERR_NUMERICAL: NumericalFault,
           TSOM_ERR_RANGE: OutOfRange, TSOM_ERR_TIMEOUT: BarrierTimeout}.get(status, TsomError)
    raise cls(status, msg)


_lib = None
_vp = C.c_void_p


def _point_at_nccl_wheel():
    """The engine dlopens NCCL lazily; prefer the NCCL wheel torch is linked
    against, so one process never holds two different libnccl.so.2."""
    if os.environ.get("TSOM_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["TSOM_NCCL_LIB"] = cand
            return


def load():
    """Load libtsom_b200.so (built by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (there is no CPU fallback)")
    _point_at_nccl_wheel()
    L = C.CDLL(LIB_PATH)
    u32, u64, i64, i32 = C.c_uint32, C.c_uint64, C.c_int64, C.c_int
    L.tsom_create.argtypes = [i32, u32, u32, C.POINTER(_vp)]
    L.tsom_destroy.argtypes = [_vp]
    L.tsom_last_error.argtypes = [_vp]
    L.tsom_last_error.restype = C.c_char_p
    L.tsom_version.restype = C.c_char_p
    L.tsom_set_option.argtypes = [_vp, i32, i64]
    L.tsom_bind_host_data.argtypes = [_vp, _vp, u64, u32]
    L.tsom_bind_device_data.argtypes = [_vp, _vp, u64]
    L.tsom_bind_synthetic_gmm.argtypes = [_vp, u64, u64, u32, u64]
    L.tsom_rows.argtypes = [_vp]
    L.tsom_rows.restype = u64
    L.tsom_set_codebook.argtypes = [_vp, _vp]
    L.tsom_get_codebook.argtypes = [_vp, _vp]
    L.tsom_get_prev_update.argtypes = [_vp, _vp]
    L.tsom_set_influence.argtypes = [_vp, _vp, i64]
    L.tsom_epoch.argtypes = [_vp, _vp, u64, C.c_double, _vp, _vp, _vp]
    L.tsom_bmu.argtypes = [_vp, _vp, u64, _vp, _vp]
    L.tsom_bmu_bound.argtypes = [_vp, _vp, u64, _vp, _vp]
    L.tsom_qe.argtypes = [_vp, _vp, u64, C.POINTER(C.c_double), C.POINTER(u64)]
    L.tsom_set_topology_distance.argtypes = [_vp, _vp]
    L.tsom_train_epoch.argtypes = [_vp, C.c_double, C.c_double, C.c_double, u32]
    L.tsom_train_epochs.argtypes = [_vp, u32, _vp, _vp, C.c_double, u32, C.POINTER(u32)]
    L.tsom_sampler_init.argtypes = [_vp, i32, u64, u64, C.c_double, C.c_double]
    L.tsom_sampler_select.argtypes = [_vp, _vp, C.POINTER(u64)]
    L.tsom_sampler_observe.argtypes = [_vp, _vp]
    L.tsom_sampler_state.argtypes = [_vp, _vp, _vp]
    L.tsom_mt_selftest.argtypes = [u64, u64]
    L.tsom_mt_selftest.restype = i32
    L.tsom_release_cached_memory.argtypes = [i32]
    L.tsom_last_recheck_count.argtypes = [_vp]
    L.tsom_last_recheck_count.restype = u64
    L.tsom_active_bmu_kernel.argtypes = [_vp]
    L.tsom_active_bmu_kernel.restype = C.c_int
    L.tsom_comm_unique_id.argtypes = [_vp, C.c_char_p]
    L.tsom_comm_init.argtypes = [_vp, C.c_char_p, i32, i32]
    L.tsom_last_timing.argtypes = [_vp] + [C.POINTER(C.c_float)] * 4
    L.tsom_last_timing_detail.argtypes = [_vp, C.POINTER(C.c_float)]
    L.tsom_kernel_launches.restype = u64
    L.tsom_refresh_topology.argtypes = [_vp, i32, _vp, u64, C.POINTER(u64), _vp]
    L.tsom_pairwise_sq_dists.argtypes = [_vp, _vp]
    L.tsom_bind_shards.argtypes = [_vp, C.POINTER(C.c_char_p), u32, u32]
    L.tsom_stream.argtypes = [_vp]
    L.tsom_stream.restype = _vp
    L.tsom_synth_gmm_host.argtypes = [_vp, u64, u64, u32, u64, u32, u32]
    L.tsom_get_rows.argtypes = [_vp, u64, u64, _vp]
    L.tsom_device_bytes.argtypes = [_vp]
    L.tsom_device_bytes.restype = u64
    L.tsom_barrier_wait_s.argtypes = [_vp]
    L.tsom_barrier_wait_s.restype = C.c_double
    L.tsom_group_create.argtypes = [i32, C.POINTER(_vp)]
    L.tsom_group_join.argtypes = [_vp, _vp, i32]
    L.tsom_group_destroy.argtypes = [_vp]
    for name in EXPORTS:
        getattr(L, name)  # every declared entry point must resolve
    _lib = L
    return L


def kernel_launches() -> int:
    return int(load().tsom_kernel_launches())


def release_cached_memory(device: int = 0) -> None:
    """Trim the per-device pool engines allocate from (cf. torch.cuda.empty_cache)."""
    st = load().tsom_release_cached_memory(int(device))
    if st:
        raise RuntimeError(f"tsom_release_cached_memory failed ({st})")


def synth_gmm_host(n: int, d: int = 50, seed: int = 2604, n_comp: int = 16,
                   threads: int = 0, out=None, row0: int = 0) -> np.ndarray:
    """The reference's Gaussian-mixture rows, generated on all
    host cores (no GPU); value-identical to Rng(seed, synth) in sequence.
    row0: first row of the stream (a rank's slice of one dataset)."""
    L = load()
    if out is None:
        out = np.empty((n, d), np.float32)
    assert out.shape == (n, d) and out.dtype == np.float32 and out.flags.c_contiguous
    st = L.tsom_synth_gmm_host(out.ctypes.data if n else None, row0, n, d, seed, n_comp, threads)
    if st:
        _raise(st, "tsom_synth_gmm_host: bad arguments")
    return out


def mt_selftest(seed: int, jump: int) -> int:
    """Host-side check of the MT19937-64 jump-ahead (0 = jumped state and
    outputs equal sequential generation); needs no GPU."""
    return int(load().tsom_mt_selftest(int(seed), int(jump)))


def version() -> str:
    return load().tsom_version().decode()


def _ptr(a):
    return None if a is None else a.ctypes.data


class Engine:
    """One GPU, one P x d codebook: thin RAII wrapper of ``tsom_engine``."""

    def __init__(self, nodes: int, dims: int, device: int = 0):
        self.L = load()
        self.nodes, self.dims, self.device = int(nodes), int(dims), int(device)
        h = _vp()
        st = self.L.tsom_create(self.device, self.nodes, self.dims, C.byref(h))
        if st:
            _raise(st, f"tsom_create failed (status {st}); see stderr")
        self.h = h
        self._keep = None  # host rows kept alive in streamed mode

    def close(self):
        if getattr(self, "h", None):
            self.L.tsom_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, st):
        if st:
            _raise(st, self.L.tsom_last_error(self.h).decode())

    # --- configuration ----------------------------------------------------
    def set_option(self, key: int, value: int):
        self._check(self.L.tsom_set_option(self.h, key, int(value)))

    def bind(self, rows: np.ndarray, streamed: bool = False):
        rows = np.ascontiguousarray(rows, np.float32)
        assert rows.ndim == 2 and rows.shape[1] == self.dims, "bind: rows must be n x d"
        flags = TSOM_BIND_STREAMED if streamed else TSOM_BIND_COPY
        self._keep = rows if streamed else None
        self._check(self.L.tsom_bind_host_data(self.h, _ptr(rows), rows.shape[0], flags))

    def bind_shards(self, paths, streamed: bool = True):
        """FSOMSHRD files (dataset.hpp:171-344), rows in the given order."""
        arr = (C.c_char_p * len(paths))(*[os.fsencode(p) for p in paths])
        flags = TSOM_BIND_STREAMED if streamed else TSOM_BIND_COPY
        self._check(self.L.tsom_bind_shards(self.h, arr, len(paths), flags))

    def bind_device(self, ptr: int, n_rows: int):
        self._check(self.L.tsom_bind_device_data(self.h, ptr, n_rows))

    def bind_synthetic_gmm(self, n_rows: int, seed: int, n_comp: int = 16, row_offset: int = 0):
        self._check(self.L.tsom_bind_synthetic_gmm(self.h, n_rows, seed, n_comp, row_offset))

    @property
    def rows(self) -> int:
        return int(self.L.tsom_rows(self.h))

    def get_rows(self, row0: int = 0, n=None, out=None) -> np.ndarray:
        """Resident rows [row0, row0 + n) back on the host (n x d f32)."""
        n = self.rows - row0 if n is None else int(n)
        if out is None:
            out = np.empty((n, self.dims), np.float32)
        assert out.shape == (n, self.dims) and out.dtype == np.float32 and out.flags.c_contiguous
        self._check(self.L.tsom_get_rows(self.h, int(row0), n, _ptr(out) if n else None))
        return out

    def set_codebook(self, w: np.ndarray):
        w = np.ascontiguousarray(w, np.float32)
        assert w.shape == (self.nodes, self.dims)
        self._check(self.L.tsom_set_codebook(self.h, _ptr(w)))

    def get_codebook(self) -> np.ndarray:
        w = np.empty((self.nodes, self.dims), np.float32)
        self._check(self.L.tsom_get_codebook(self.h, _ptr(w)))
        return w

    def set_influence(self, h: np.ndarray, key: int = -1):
        h = np.ascontiguousarray(h, np.float64)
        assert h.shape == (self.nodes, self.nodes)
        self._check(self.L.tsom_set_influence(self.h, _ptr(h), int(key)))

    def set_topology_distance(self, dist: np.ndarray):
        dist = np.ascontiguousarray(dist, np.float64)
        assert dist.shape == (self.nodes, self.nodes)
        self._check(self.L.tsom_set_topology_distance(self.h, _ptr(dist)))

    # --- hot path ---------------------------------------------------------
    def epoch(self, eta: float, selected=None, want_dist: bool = False):
        """Executor::run_iteration: returns (U [P,d] f64, H [P] f64, distances|None)."""
        sel = None if selected is None else np.ascontiguousarray(selected, np.uint32)
        n = self.rows if sel is None else len(sel)
        u = np.empty((self.nodes, self.dims))
        hh = np.empty(self.nodes)
        dist = np.empty(max(n, 1)) if want_dist else None
        self._check(self.L.tsom_epoch(self.h, _ptr(sel), 0 if sel is None else len(sel),
                                      float(eta), _ptr(u), _ptr(hh), _ptr(dist)))
        return u, hh, (dist[:n] if want_dist else None)

    def bmu(self, rows: np.ndarray, want_dist: bool = True):
        rows = np.ascontiguousarray(rows, np.float32)
        n = rows.shape[0]
        b = np.empty(max(n, 1), np.uint32)
        d = np.empty(max(n, 1)) if want_dist else None
        self._check(self.L.tsom_bmu(self.h, _ptr(rows), n, _ptr(b), _ptr(d)))
        return b[:n], (d[:n] if want_dist else None)

    def bmu_bound(self, selected=None, want_dist: bool = True):
        sel = None if selected is None else np.ascontiguousarray(selected, np.uint32)
        n = self.rows if sel is None else len(sel)
        b = np.empty(max(n, 1), np.uint32)
        d = np.empty(max(n, 1)) if want_dist else None
        self._check(self.L.tsom_bmu_bound(self.h, _ptr(sel), 0 if sel is None else len(sel),
                                          _ptr(b), _ptr(d)))
        return b[:n], (d[:n] if want_dist else None)

    def qe(self, selected=None):
        sel = None if selected is None else np.ascontiguousarray(selected, np.uint32)
        s = C.c_double()
        c = C.c_uint64()
        self._check(self.L.tsom_qe(self.h, _ptr(sel), 0 if sel is None else len(sel),
                                   C.byref(s), C.byref(c)))
        return s.value, c.value

    def train_epoch(self, eta: float, sigma: float, momentum: float = 0.0,
                    use_momentum: bool = False, sampled: bool = False):
        """One device-resident epoch; sampled=True lets the device sampler
        (sampler_init) pick the rows and, if adaptive, observe their distances."""
        self._check(self.L.tsom_train_epoch(self.h, float(eta), float(sigma), float(momentum),
                                            (1 if use_momentum else 0) | (2 if sampled else 0)))

    def train_epochs(self, etas, sigmas, momentum: float = 0.0, use_momentum: bool = False,
                     sampled: bool = False):
        """len(etas) device-resident epochs back to back (no host round trip
        between them); a numerical fault names the failing epoch."""
        eta = np.ascontiguousarray(etas, np.float64)
        sig = np.ascontiguousarray(sigmas, np.float64)
        assert eta.shape == sig.shape and eta.ndim == 1 and len(eta) >= 1
        failed = C.c_uint32()
        self._check(self.L.tsom_train_epochs(self.h, len(eta), _ptr(eta), _ptr(sig),
                                             float(momentum),
                                             (1 if use_momentum else 0) | (2 if sampled else 0),
                                             C.byref(failed)))

    # --- device sampler (sampling.hpp:183-221) -------------------------------
    def sampler_init(self, kind, m: int, seed: int, alpha: float = 1.0, beta: float = 1.0):
        k = SAMPLER_KINDS[kind] if isinstance(kind, str) else int(kind)
        self._check(self.L.tsom_sampler_init(self.h, k, int(m), int(seed) & (2**64 - 1),
                                             float(alpha), float(beta)))

    def sampler_select(self) -> np.ndarray:
        """Sampler::select() on the device: sorted uint32 row ids."""
        out = np.empty(self.rows, np.uint32)
        m = C.c_uint64()
        self._check(self.L.tsom_sampler_select(self.h, _ptr(out), C.byref(m)))
        return out[: m.value].copy()

    def sampler_observe(self, distances=None):
        """Sampler::observe for the last selection (distances in selection order;
        None = those of the last sampled epoch)."""
        d = None if distances is None else np.ascontiguousarray(distances, np.float64)
        self._check(self.L.tsom_sampler_observe(self.h, _ptr(d)))

    def sampler_state(self):
        e = np.empty(self.rows, np.float64)
        a = np.empty(self.rows, np.uint32)
        self._check(self.L.tsom_sampler_state(self.h, _ptr(e), _ptr(a)))
        return e, a

    @property
    def active_bmu_kernel(self) -> int:
        """1 SIMT, 2 tcgen05 3xTF32, 3 tcgen05 3xFP16."""
        return int(self.L.tsom_active_bmu_kernel(self.h))

    @property
    def last_recheck_count(self) -> int:
        return int(self.L.tsom_last_recheck_count(self.h))

    def last_timing(self):
        v = [C.c_float() for _ in range(4)]
        self._check(self.L.tsom_last_timing(self.h, *[C.byref(x) for x in v]))
        return {"bmu_ms": v[0].value, "accum_ms": v[1].value, "smooth_ms": v[2].value,
                "total_ms": v[3].value}

    def refresh_topology(self, kind: str, want_hops: bool = False):
        """Device refresh_topology: returns (edges [m, 2] uint32, hops [P, P] or None)."""
        k = {"mst": 2, "rng": 3}[kind]
        P = self.nodes
        cap = max(1, P * (P - 1) // 2)
        edges = np.empty(2 * cap, np.uint32)
        ne = C.c_uint64()
        hops = np.empty((P, P), np.uint16) if want_hops else None
        self._check(self.L.tsom_refresh_topology(self.h, k, _ptr(edges), cap, C.byref(ne),
                                                 _ptr(hops)))
        return edges[: 2 * ne.value].reshape(-1, 2).copy(), hops

    def pairwise_sq_dists(self) -> np.ndarray:
        out = np.empty((self.nodes, self.nodes))
        self._check(self.L.tsom_pairwise_sq_dists(self.h, _ptr(out)))
        return out

    def timing_detail(self):
        v = (C.c_float * 8)()
        self._check(self.L.tsom_last_timing_detail(self.h, v))
        keys = ["k1_ms", "bmu_ms", "accum_ms", "smooth_ms", "update_ms", "total_ms", "sample_ms",
                "accum_mean_ms"]
        return dict(zip(keys, list(v)))

    @property
    def stream(self) -> int:
        return int(self.L.tsom_stream(self.h) or 0)

    # --- multi-GPU --------------------------------------------------------
    def comm_unique_id(self) -> bytes:
        buf = C.create_string_buffer(128)
        self._check(self.L.tsom_comm_unique_id(self.h, buf))
        return buf.raw

    def comm_init(self, uid: bytes, rank: int, world: int):
        assert len(uid) == 128
        self._check(self.L.tsom_comm_init(self.h, uid, rank, world))

    def join_group(self, group: "RankGroup", rank: int):
        """Make this engine rank `rank` of an in-process rank group (the epoch
        reduce and the sharded sampler then go through it instead of NCCL)."""
        self._check(self.L.tsom_group_join(self.h, group.h, int(rank)))

    @property
    def device_bytes(self) -> int:
        """Device memory held by this engine's buffers."""
        return int(self.L.tsom_device_bytes(self.h))

    @property
    def barrier_wait_s(self) -> float:
        """Seconds spent in reduce barriers (ThreadedExecutor::barrier_wait_s)."""
        return float(self.L.tsom_barrier_wait_s(self.h))


class RankGroup:
    """In-process rank group (tsom_group_*): engines driven from separate
    threads joined by an ordered host-memory reduce with a barrier deadline."""

    def __init__(self, world: int):
        self.L = load()
        self.world = int(world)
        h = _vp()
        st = self.L.tsom_group_create(self.world, C.byref(h))
        if st:
            _raise(st, "tsom_group_create failed")
        self.h = h

    def close(self):
        if self.h:
            self.L.tsom_group_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
