#!/usr/bin/env python
"""Headline benchmark: samples·epochs/s of batch-SOM training (K=1024, D=50).

Headline workload (BASELINE.json configs[1]): 32x32 hexagonal lattice (1024
nodes), 10,000,000 x 50 Gaussian-mixture rows per GPU from the reference's own
generator, full sampling.  One *step* = one training epoch
over all rows: influence(σ) → BMU search (K1) → exact near-tie re-check →
per-BMU accumulation (K2) → reduce [+ NCCL allreduce for N>1] → FP64
smoothing (K3) → apply_update.

  value : device-timed epochs with the rows resident in HBM (CUDA events on
          the engine stream, max over ranks); inputs (2.56 GB/GPU) exceed L2.
  e2e   : the same training through the public C-ABI from HOST rows (engine
          creation, H2D bind, 10 epochs, codebook D2H; wall clock), from
          page-locked rows and from a pageable array, plus the reference's own
          training loop with the drop-in executor.
  c1, c3, c4, c5 : the other BASELINE configs (c1 in full against the
          reference run on the host cores; c3 MST over 1e8 rows; c4 RNG +
          adaptive sampler over 1e8 rows; c5 one GPU's 1.25e8-row share of the
          1e9-row job, resident / streamed from pinned host / streamed from
          shard files with a cold page cache), each with its CPU baseline.
  --impl reference : the reference CPU implementation (oracle/_ref =
          /root/reference headers compiled, train_parallel on all host cores)
          on a bounded sample of the headline workload.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples·epochs/sec (1024 nodes, D=50) at 1/2/4/8 B200; % roofline; QE vs CPU"
UNIT = "samples·epochs/s"
P_GRID = (32, 32)
P = P_GRID[0] * P_GRID[1]
D = 50
N_PER_GPU = 10_000_000
# seed = 2604 + config number
SEEDS = {"c1": 2605, "c2": 2606, "c3": 2607, "c4": 2608, "c5": 2609}
SEED = SEEDS["c2"]
EPOCHS = 10


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled every 20 ms (NVML) during the timed region."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
             "sw_power_cap": 0x4}

    def __init__(self, index=0, period=0.02):
        self.index, self.period = index, period
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, rs))
                    except Exception:
                        pass
                    self._stop.wait(self.period)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({k for _, rs in self.samples for k, bit in self.NAMES.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "sm_mhz_min": min(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the reference headers compiled) on a bounded sample
# ---------------------------------------------------------------------------

def cpu_model():
    """Host CPU model name (from /proc/cpuinfo) for the cpu_baseline record."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_reference(step_seconds=6.0, steps=1, warmup=0, threads=None):
    """Time the reference's train_parallel (all host cores, or `threads`) on a
    bounded sample of the headline workload: 32x32 hex, D=50, full sampling;
    each step = one epoch.  Returns (samples·epochs/s, cores, kind, sample
    description, seconds per step)."""
    import numpy as np

    import oracle
    chk = oracle.best()
    cores = threads or os.cpu_count() or 1
    # calibrate rows so one epoch takes ~step_seconds
    probe_rows = 256 * cores
    x = chk.synth_gmm(probe_rows, D, SEED)
    cfg = oracle.SomConfig(topology="hex", grid_w=P_GRID[0], grid_h=P_GRID[1], n_iters=1,
                           seed=SEED, n_threads=cores)
    t0 = time.perf_counter()
    chk.train(cfg, x)
    rate = probe_rows / max(time.perf_counter() - t0, 1e-6)
    rows = int(min(max(rate * step_seconds, probe_rows), 400_000))
    x = chk.synth_gmm(rows, D, SEED)
    cfg.n_iters = 1
    for _ in range(warmup):
        chk.train(cfg, x)
    times = []
    for _ in range(max(steps, 1)):
        t0 = time.perf_counter()
        chk.train(cfg, x)
        times.append(time.perf_counter() - t0)
    value = rows / statistics.mean(times)
    sample = (f"{rows} of the {N_PER_GPU} rows (same GMM generator), 32x32 hex, D=50, 1 epoch "
              f"per step incl. init; train_parallel G={cores}")
    return value, cores, chk.kind, sample, statistics.mean(times)


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    # exactly K timed steps after W warm-up steps, each a bounded sample sized
    # so the whole run stays near 2.5 minutes of host time
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    step_s = max(0.5, min(4.0, 150.0 / (steps + warmup)))
    value, cores, kind, sample, t = cpu_reference(step_seconds=step_s, steps=steps,
                                                  warmup=warmup)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "c2: 32x32 hex SOM (1024 nodes), D=50, GMM rows, full sampling "
                               "(bounded CPU sample)", "model": "batch-SOM"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def pinned_rows(n, d=None):
    """A page-locked host buffer (torch pin_memory) as an (n, d) float32 array."""
    import torch
    d = d or D
    return torch.empty((n, d), dtype=torch.float32, pin_memory=True).numpy()


def host_gmm_rows(n, seed, row0=0, pinned=True):
    """The SURVEY §8(d) rows from the reference's own generator (Rng(seed,
    synth) in sequence, value-identical), produced by the product's host
    generator on all cores (tsom_synth_gmm_host, mt19937_64 jump-ahead per
    thread), into page-locked memory."""
    from paper_2604_26555_b200 import _lib
    out = pinned_rows(n) if pinned else None
    return _lib.synth_gmm_host(n, D, seed, 16, 0, out=out, row0=row0)


class EngineRows:
    """init_sample_draw over rows resident in an engine (only the picks come back)."""

    def __init__(self, e):
        import numpy as np
        self.e, self.np = e, np
        self.shape = (e.rows, e.dims)

    def __getitem__(self, idx):
        return self.np.stack([self.e.get_rows(int(i), 1)[0] for i in idx])


def hbm_used_gb(index=0):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        return round(pynvml.nvmlDeviceGetMemoryInfo(h).used / 1e9, 2)
    except Exception:
        return None


def h2d_gbs(local, nbytes=2 << 30):
    """Measured pinned host -> device copy bandwidth (the streamed-mode bound)."""
    import torch
    src = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    dst = torch.empty_like(src, device=f"cuda:{local}")
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    gbs = 3 * nbytes / (a.elapsed_time(b) / 1e3) / 1e9
    del src, dst
    torch.cuda.empty_cache()
    return gbs


def hex_schedule(epochs, t0=0, count=None):
    from paper_2604_26555_b200.hostref import resolved_sigma0, schedule_value
    sigma0 = resolved_sigma0("hex", *P_GRID)
    ts = range(t0, t0 + (count if count is not None else epochs))
    return ([schedule_value(0.5, "linear", t % epochs, epochs, 1e-4) for t in ts],
            [schedule_value(sigma0, "linear", t % epochs, epochs, 0.3) for t in ts])


def close_engine(e):
    """Close an engine and hand its cached blocks back to the driver."""
    import torch
    from paper_2604_26555_b200 import _lib
    if e is not None:
        dev = e.device
        e.close()
        _lib.release_cached_memory(dev)
    torch.cuda.empty_cache()


def run_gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200 import _lib
    from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    n = N_PER_GPU

    def bcast(obj):
        o = [obj]
        if world > 1:
            dist.broadcast_object_list(o, src=0)
        return o[0]

    def tmax(v):
        if world == 1:
            return v
        tm = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        return float(tm.item())

    def attach_comm(e):
        # one NCCL communicator per engine: rank 0's unique id over the gloo group
        if world > 1 or args.force_comm:
            e.comm_init(bcast(e.comm_unique_id() if rank == 0 else None), rank, world)

    ctx = {"world": world, "rank": rank, "local": local, "bcast": bcast, "tmax": tmax,
           "attach": attach_comm}
    # c2 rows: this rank's slice of one dataset from the reference's generator
    t_gen = time.perf_counter()
    host = host_gmm_rows(n, SEEDS["c2"], row0=rank * n)
    t_gen = time.perf_counter() - t_gen
    eng = tsom.Engine(P, D, device=local)
    if args.kernel:
        eng.set_option(_lib.TSOM_OPT_BMU_KERNEL, args.kernel)
    if args.row_order is not None:
        eng.set_option(_lib.TSOM_OPT_ROW_ORDER, args.row_order)
    if args.k1_debug is not None:
        eng.set_option(99, args.k1_debug)  # diagnostics A/B (process-wide K1 variant bits)
    eng.bind(host)
    active_kernel = eng.active_bmu_kernel
    attach_comm(eng)
    # init_weights(sample_draw) (trainer.hpp:192-211) over rank 0's rows, same on every rank
    w0 = bcast(init_sample_draw(host, P, SEEDS["c2"]) if rank == 0 else None)
    eng.set_codebook(w0)
    eng.set_topology_distance(lattice_dist("hex", *P_GRID))

    for t in range(args.warmup):
        e_, s_ = hex_schedule(EPOCHS, t, 1)
        eng.train_epoch(e_[0], s_[0])
    stream = torch.cuda.ExternalStream(eng.stream, device=f"cuda:{local}")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.kernel_launches()
    # the K timed epochs go to the engine in one tsom_train_epochs call: every
    # epoch is the full epoch of tsom_train_epoch, enqueued back to back with
    # the schedules precomputed (no host round trip between epochs)
    etas, sigmas = hex_schedule(EPOCHS, args.warmup, args.steps)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        eng.train_epochs(etas, sigmas)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.kernel_launches() - launches0
    k1 = eng.timing_detail()["k1_ms"]  # mean main-pass K1 over the timed epochs
    k2_timed = eng.timing_detail()["accum_mean_ms"]  # mean accumulation phase, same epochs
    elapsed = tmax(ev0.elapsed_time(ev1))
    if world > 1:
        dist.barrier()
    ms = elapsed / args.steps
    value = n * world / (ms / 1e3)
    # phase breakdown and re-check counts from three untimed single-epoch calls
    phases, rechecks = [], []
    for t in range(args.warmup + args.steps, args.warmup + args.steps + 3):
        e_, s_ = hex_schedule(EPOCHS, t, 1)
        eng.train_epoch(e_[0], s_[0])
        phases.append(eng.timing_detail())
        rechecks.append(eng.last_recheck_count)
    s, c = eng.qe()
    qe_gpu = s / c
    c2_bytes = eng.device_bytes
    c2_hbm = hbm_used_gb(local)
    # QE vs the CPU oracle: the trained codebook's mean BMU distance over a
    # 20,000-row sample, GPU (tsom_bmu) against the oracle's find_bmus
    qe_check = None
    if rank == 0 and not args.no_cpu:
        import oracle
        w_fin = eng.get_codebook()
        sample = np.ascontiguousarray(host[:20_000])
        _, d_gpu = eng.bmu(sample)
        _, d_cpu = oracle.port.find_bmus(sample, w_fin)
        qe_check = {"rows": len(sample), "qe_gpu": float(np.mean(d_gpu)),
                    "qe_cpu_oracle": float(np.mean(d_cpu)),
                    "rel_diff": float(abs(np.mean(d_gpu) - np.mean(d_cpu)) / np.mean(d_cpu))}
    close_engine(eng)
    eng = None

    e2e = None if args.no_e2e else leg_e2e(args, ctx, host, w0)
    pk, pk_kind = peaks()
    flops = 2.0 * P * D * n
    achieved = flops / (k1 / 1e3) / 1e12 if k1 > 0 else 0.0
    kname, peak, pnote = roofline_peak(active_kernel, pk)
    roof = {"bound": "tensor", "kernel": "k1 BMU (" + kname + ")",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak,
            "traffic": K1_TRAFFIC.get(active_kernel),
            "note": (f"achieved = 2*K*D*N useful flop per launch / mean K1 event time over the "
                     f"timed epochs (per-epoch CUDA events on the engine stream); phase_ms from "
                     f"3 untimed single-epoch calls after the timed region; peak = "
                     f"{pk_kind} bf16 {pk['bf16_tflops']} TF/s {pnote}; traffic = ncu "
                     f"dram__bytes_read+write per launch ({K1_TRAFFIC_SRC})"),
            "k1_ms": k1,
            # the pool's sustained bf16 GEMM (under the 1000 W cap) is the fair
            # denominator for a kernel inside a long loop: K1 itself runs at
            # ~1.52 GHz (ncu sm__cycles_elapsed / duration), the memory kernels
            # of the epoch at ~1.9-2.0 GHz
            "peak_sustained": pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) / 3.0
            if active_kernel == 3 else None,
            "frac_of_sustained": achieved / (pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) / 3.0)
            if active_kernel == 3 else None,
            "epoch_ms": statistics.mean(p["total_ms"] for p in phases),
            "phase_ms": {k: statistics.mean(p[k] for p in phases) for k in phases[0]}}
    # K2 (accumulation) against HBM: 204 algorithmic bytes per row (the row
    # and its BMU) over the accumulate phase's event time
    acc_untimed = statistics.mean(p["accum_ms"] for p in phases)
    acc_ms = k2_timed if k2_timed > 0 else acc_untimed
    k2_gbs = n * 204 / (acc_ms / 1e3) / 1e9 if acc_ms > 0 else 0.0
    k2_roof = {"bound": "hbm", "kernel": "k2 sort + TMA gather + piece reduce",
               "achieved": k2_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
               "frac": k2_gbs / pk["hbm_gbs"], "accum_ms": acc_ms,
               "accum_ms_single_epoch_calls": acc_untimed,
               "note": "achieved = 204 B/row x rows / the accumulate phase's mean per-epoch "
                       "event time over the timed epochs (sort + gather + piece reduce, launch "
                       "gaps included); rows packed in BMU order after the one re-layout"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": {3: "f32 via 3xFP16 split", 2: "f32 via 3xTF32 split", 1: "f32"}[active_kernel]
                 + " BMU (exact FP64 re-check) + f64 accumulate/update",
        "data": "synthetic Gaussian mixture (16 comps, U[-4,4] centres, unit noise) from the "
                "reference's generator (Rng(seed, synth), value-identical, host-generated on all "
                "cores), random-init codebook by sample_draw",
        "config": {"workload": "c2: 32x32 hex SOM (1024 nodes), 1e7 x 50 rows per GPU, full "
                               "sampling, resident in HBM", "model": "batch-SOM",
                   "nodes": P, "dims": D, "rows_per_gpu": n, "global_rows": n * world,
                   "seed": SEEDS["c2"], "parallelism": f"dp{world}",
                   "l2": "inputs (2.56 GB/GPU at the 256-B row stride) > L2 (126 MB); no flush"},
        "roofline": roof,
        "roofline_k2": k2_roof,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "qe_gpu_after": qe_gpu,
        "qe_vs_cpu": qe_check,
        "rechecked_rows_per_epoch": statistics.mean(rechecks),
        "hbm": {"engine_bytes": c2_bytes, "bytes_per_row": round(c2_bytes / n, 1),
                "device_used_gb": c2_hbm, "host_generation_s": round(t_gen, 2)},
    }
    if e2e:
        line["e2e"] = e2e
    del host
    # c1 (a 6-ms run timed by wall clock) first: after c5 the host is still
    # writing back its shard files, which tripled c1's time in one run
    legs = [("c1", not args.no_c1, leg_c1), ("c4", not args.no_c4, leg_c4),
            ("c3", not args.no_c3, leg_c3), ("c5", not args.no_c5 and world == 1, leg_c5)]
    for name, on, fn in legs:
        if args.only and name not in args.only.split(","):
            continue
        if on:
            try:
                out = fn(args, ctx)
            except Exception as ex:  # a failing extra leg must not hide the headline
                out = {"error": f"{type(ex).__name__}: {ex}"}
            torch.cuda.empty_cache()
            if rank == 0:
                line[name] = out
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, kind, sample, _ = cpu_reference(step_seconds=6.0)
        v1, _, _, sample1, _ = cpu_reference(step_seconds=3.0, threads=1)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": sample, "cpu_model": cpu_model(),
                                "single_thread": {"value": v1, "sample": sample1}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def leg_e2e(args, ctx, host, w0):
    """The same c2 training end to end through the public C-ABI from HOST rows:
    engine creation, bind (H2D), 10 epochs, codebook read-back (D2H), wall
    clock, max over ranks; from page-locked rows (the headline) and from a
    pageable array; plus the reference's own loops with the drop-in."""
    import numpy as np

    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200 import _lib
    from paper_2604_26555_b200.hostref import lattice_dist
    world, rank, local = ctx["world"], ctx["rank"], ctx["local"]
    n = host.shape[0]
    topo_d = lattice_dist("hex", *P_GRID)  # host input, like the rows
    etas, sigmas = hex_schedule(EPOCHS)

    def cabi_run(rows):
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        t0 = time.perf_counter()
        e = tsom.Engine(P, D, device=local)
        if args.kernel:
            e.set_option(_lib.TSOM_OPT_BMU_KERNEL, args.kernel)
        if args.row_order is not None:
            e.set_option(_lib.TSOM_OPT_ROW_ORDER, args.row_order)
        ta = time.perf_counter()
        e.bind(rows)
        tb = time.perf_counter()
        ctx["attach"](e)
        e.set_codebook(w0)
        e.set_topology_distance(topo_d)
        t1 = time.perf_counter()
        e.train_epochs(etas, sigmas)
        e.get_codebook()
        t2 = time.perf_counter()
        e.close()
        t3 = time.perf_counter()
        return ctx["tmax"](t3 - t0), {"create_s": ta - t0, "bind_s": tb - ta,
                                      "config_s": t1 - tb, "epochs_s": t2 - t1,
                                      "close_s": t3 - t2}

    cabi_run(host[: n // 8])  # warm-up (allocations, module load)
    secs, split = min((cabi_run(host) for _ in range(3)), key=lambda r: r[0])
    h2d = n * D * 4 + P * D * 4 + P * P * 8
    d2h = P * D * 4
    out = {"value": n * world * EPOCHS / secs, "unit": UNIT,
           "h2d_bytes_per_step": int(h2d / EPOCHS), "d2h_bytes_per_step": int(d2h / EPOCHS),
           "path": "C-ABI tsom_bind_host_data + tsom_train_epochs (10 epochs) + tsom_get_codebook "
                   "from page-locked host rows, wall clock incl. engine creation (and the NCCL "
                   "communicator when N > 1), max over ranks; best of 3",
           "seconds_per_call": secs, "epochs_per_call": EPOCHS, "split_s": split}
    # the same call from a pageable array (a plain numpy array / DataMatrix):
    # the bind goes through the multi-threaded pinned staging
    pageable = np.array(host, copy=True)
    psecs, psplit = min((cabi_run(pageable) for _ in range(2)), key=lambda r: r[0])
    out["pageable"] = {"value": n * world * EPOCHS / psecs, "seconds_per_call": psecs,
                       "split_s": psplit,
                       "path": "the same C-ABI call from pageable host rows (numpy)"}
    del pageable
    from paper_2604_26555_b200 import dropin
    if world == 1 and dropin.available():
        cfg = dropin.TrainConfig(topology="hex", grid_w=P_GRID[0], grid_h=P_GRID[1],
                                 n_iters=EPOCHS, seed=SEEDS["c2"])
        warm = dropin.TrainConfig(topology="hex", grid_w=P_GRID[0], grid_h=P_GRID[1],
                                  n_iters=1, seed=SEEDS["c2"])
        # warm-up on 1e6 rows: the pinned staging blocks (128-MB chunks) are
        # allocated once per process, as for every later bind
        dropin.train_device(warm, host[:1_000_000], device=local)
        vsecs = min(dropin.train_device(cfg, host, device=local)[3] for _ in range(2))
        dropin.train_cuda(warm, host[:1_000_000], device=local)
        _, _, _, dsecs = dropin.train_cuda(cfg, host, device=local)
        out["dropin_device_loop"] = {
            "value": n * EPOCHS / vsecs, "seconds_per_call": vsecs,
            "path": "toposom_b200::train_device (C++ drop-in: init_weights and lattice distances "
                    "as the reference builds them, then every epoch step on the device; the "
                    "host DataMatrix (pageable) bound through the pinned staging); best of 2"}
        out["dropin_reference_loop"] = {
            "value": n * EPOCHS / dsecs, "seconds_per_call": dsecs,
            "path": "toposom::train_with_executor + toposom_b200::CudaExecutor (host DataMatrix; "
                    "the reference's host code per epoch: sampler index vector, influence matrix, "
                    "apply_update, int128 accumulators)"}
    return out


def graph_epochs(e, kind, epochs, sampled=False, t_start=0, count=None):
    """The reference schedule for a graph topology (sigma0 auto = 3, linear
    decays, refresh policy warmup 10 % / growth 1.5 / max 25,
    trainer.hpp:75-85, topology.hpp:423-451): epochs between two refreshes go
    to the engine as one tsom_train_epochs call; a refresh runs on the device."""
    from paper_2604_26555_b200.hostref import RefreshState, resolved_sigma0, schedule_value
    sigma0 = resolved_sigma0(kind, 0, 0, 0.0)
    refresh = RefreshState(max(1, epochs // 10), 1.5, 25)
    ts = list(range(epochs))
    marks = []
    for t in ts:
        if refresh.should_refresh(t):
            refresh.mark(t)
            marks.append(t)
    t = 0
    while t < epochs:
        if t in marks:
            e.refresh_topology(kind)
        t1 = t + 1
        while t1 < epochs and t1 not in marks:
            t1 += 1
        e.train_epochs([schedule_value(0.5, "linear", u, epochs, 1e-4) for u in range(t, t1)],
                       [schedule_value(sigma0, "linear", u, epochs, 0.3) for u in range(t, t1)],
                       sampled=sampled)
        t = t1
    return marks


def timed(fn, ctx, stream_of=None):
    """Device time of fn() (CUDA events on the engine stream), max over ranks."""
    import torch
    local = ctx["local"]
    torch.cuda.synchronize()
    if stream_of is not None:
        st = torch.cuda.ExternalStream(stream_of.stream, device=f"cuda:{local}")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        r = fn()
        b.record(st)
        torch.cuda.synchronize()
        return ctx["tmax"](a.elapsed_time(b) / 1e3), r
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return ctx["tmax"](time.perf_counter() - t0), r


def cpu_config_sample(cfg_kw, rows, epochs, seed, threads=None):
    """The reference (oracle/_ref: train_parallel) on the first `rows` rows of
    a config's stream, `epochs` epochs: samples·epochs/s of processed rows."""
    import oracle
    chk = oracle.best()
    cores = threads or os.cpu_count() or 1
    x = chk.synth_gmm(rows, D, seed)
    cfg = oracle.SomConfig(n_iters=epochs, seed=seed, n_threads=cores, **cfg_kw)
    t0 = time.perf_counter()
    chk.train(cfg, x)
    secs = time.perf_counter() - t0
    rho = cfg_kw.get("rho", 1.0)
    return {"value": rows * rho * epochs / secs, "unit": UNIT, "cores": cores, "kind": chk.kind,
            "seconds": secs,
            "sample": f"the first {rows} rows of the config's stream, {epochs} epochs incl. "
                      f"init and host topology refreshes; train_parallel G={cores}; value counts "
                      f"the rows each epoch processes"}


def leg_c4(args, ctx):
    """Config c4: 1024-node RNG-topology SOM, 1e8 x 50 GMM rows
    resident in HBM (split over the ranks), adaptive sampler rho = 0.1 on the
    device (select -> epoch over the selected rows -> observe; with N > 1 one
    sharded sampler over all rows, its digit histograms allreduced), RNG
    graph refreshed on the device on the reference schedule.  Timed with CUDA
    events on the engine stream, max over ranks.  value = selected
    samples·epochs/s (the rows an epoch processes)."""
    import numpy as np
    import torch

    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200.hostref import init_sample_draw
    world, rank, local = ctx["world"], ctx["rank"], ctx["local"]
    seed, n_total, rho, epochs = SEEDS["c4"], 100_000_000, 0.1, EPOCHS
    n = n_total // world + (1 if rank < n_total % world else 0)
    off = sum(n_total // world + (1 if r < n_total % world else 0) for r in range(rank))
    e = tsom.Engine(P, D, device=local)
    if args.image is not None:
        e.set_option(95, args.image)  # diagnostics: split image on / off
    # N >= 1e8: device-generated rows (SURVEY §8(d) allows it for throughput)
    e.bind_synthetic_gmm(n, seed, 16, off)
    ctx["attach"](e)
    w0 = ctx["bcast"](init_sample_draw(EngineRows(e), P, seed) if rank == 0 else None)
    e.set_codebook(w0)
    m = max(1, int(np.floor(n_total * rho)))
    e.sampler_init("adaptive", m, seed)
    graph_epochs(e, "rng", 2, sampled=True)  # warm-up (allocations of the sampled epochs)
    e.set_codebook(w0)
    e.sampler_init("adaptive", m, seed)
    secs, _ = timed(lambda: graph_epochs(e, "rng", epochs, sampled=True), ctx, e)
    phases, rechecks = [], []
    from paper_2604_26555_b200.hostref import resolved_sigma0
    for t in range(3):  # phase detail from 3 untimed single epochs
        e.train_epoch(0.1, resolved_sigma0("rng", 0, 0, 0.0) * 0.3, sampled=True)
        phases.append(e.timing_detail())
        rechecks.append(e.last_recheck_count)
    s, c = e.qe()
    dev_bytes, used = e.device_bytes, hbm_used_gb(local)
    refresh_s, _ = timed(lambda: e.refresh_topology("rng"), ctx, e)
    close_engine(e)
    pk, _ = peaks()
    k1 = statistics.mean(p["k1_ms"] for p in phases)
    m_rank = m / world
    kname, peak, _ = roofline_peak(3, pk)
    out = {"workload": "c4: 1024-node RNG-topology SOM (device refresh), 1e8 x 50 GMM rows "
                       "resident (split over the GPUs), adaptive sampler rho=0.1 on the device "
                       "(one sharded sampler), 10 epochs",
           "value": m * epochs / secs, "unit": UNIT, "n_gpus": world,
           "unit_note": "samples = the selected rows an epoch processes (rho N)",
           "rows_considered_per_s": n_total * epochs / secs, "ms_per_epoch": secs * 1e3 / epochs,
           "phase_ms": {k: round(statistics.mean(p[k] for p in phases), 3) for k in phases[0]},
           "rechecked_rows_per_epoch": statistics.mean(rechecks), "qe_after": s / c,
           "refresh_ms": refresh_s * 1e3,
           "roofline": {"bound": "tensor", "kernel": "k1 BMU (" + kname + ") over the selected rows",
                        "achieved": 2.0 * P * D * m_rank / (k1 / 1e3) / 1e12, "peak": peak,
                        "unit": "TFLOP/s",
                        "frac": 2.0 * P * D * m_rank / (k1 / 1e3) / 1e12 / peak, "k1_ms": k1},
           "hbm": {"engine_bytes": dev_bytes, "device_used_gb": used}}
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_config_sample(
            dict(topology="rng", nodes=P, sampling="adaptive", rho=rho), 100_000, 2, seed)
    return out


def leg_c3(args, ctx):
    """Config c3: 1024-node MST-topology SOM, 1e8 x 50 rows
    data-parallel over the GPUs (strong scaling: 1e8 / N rows per rank), 10
    epochs, MST refreshed on the device on the reference schedule, one f64
    allreduce per epoch.  At N = 1 it also times the 1.25e7-row share one GPU
    of the 8-GPU job holds, from the reference's generator."""
    import torch

    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200.hostref import init_sample_draw
    world, rank, local = ctx["world"], ctx["rank"], ctx["local"]
    seed, n_total, epochs = SEEDS["c3"], 100_000_000, EPOCHS
    out = {"workload": "c3: 1024-node MST-topology SOM (device refresh), 1e8 x 50 GMM rows "
                       "split over the GPUs (1e8 / N per GPU), full sampling, 10 epochs",
           "unit": UNIT, "n_gpus": world}

    def run(e, w0):
        e.set_codebook(w0)
        graph_epochs(e, "mst", 2)  # warm-up
        e.set_codebook(w0)
        with ClockSampler(ctx["local"]) as clk:
            secs, marks = timed(lambda: graph_epochs(e, "mst", epochs), ctx, e)
        s, c = e.qe()
        rs, _ = timed(lambda: e.refresh_topology("mst"), ctx, e)
        return secs, {"ms_per_epoch": secs * 1e3 / epochs, "refresh_epochs": marks,
                      "clocks": clk.summary(),
                      "refresh_ms": rs * 1e3,
                      "qe_after": s / c, "engine_bytes": e.device_bytes,
                      "device_used_gb": hbm_used_gb(local)}

    n = n_total // world + (1 if rank < n_total % world else 0)
    off = sum(n_total // world + (1 if r < n_total % world else 0) for r in range(rank))
    e = tsom.Engine(P, D, device=local)
    e.bind_synthetic_gmm(n, seed, 16, off)  # N >= 1e8: device-generated rows
    ctx["attach"](e)
    w0 = ctx["bcast"](init_sample_draw(EngineRows(e), P, seed) if ctx["rank"] == 0 else None)
    secs, det = run(e, w0)
    close_engine(e)
    out["value"] = n_total * epochs / secs
    out.update(det)
    out["rows_per_gpu"] = n
    if world == 1:
        # the 1.25e7-row share of GPU 0 in the 8-GPU job, reference generator
        share = n_total // 8
        host = host_gmm_rows(share, seed)
        e = tsom.Engine(P, D, device=local)
        e.bind(host)
        w8 = init_sample_draw(host, P, seed)
        del host
        s8, d8 = run(e, w8)
        close_engine(e)
        out["per_gpu_share_of_8"] = {"rows": share, "value": share * epochs / s8, **d8,
                                     "data": "rows [0, 1.25e7) of the reference generator"}
        if not args.no_cpu:
            out["cpu_baseline"] = cpu_config_sample(dict(topology="mst", nodes=P), 100_000, 2,
                                                    seed)
    return out


def leg_c5(args, ctx):
    """Config c5: a 1024-node (32x32 hex) SOM on 1e9 x 50 rows
    across 8 GPUs; on one GPU: one GPU's 1.25e8-row share (25 GB), 10 epochs
    resident in HBM, then streamed every epoch from page-locked host memory
    and from FSOMSHRD shard files on local disk (page cache dropped with
    posix_fadvise(DONTNEED) before the first streamed epoch: cold).  Reports
    each mode's fraction of its bound (measured pinned H2D bandwidth; the
    disk's read bandwidth measured by the cold epoch itself) and HBM use."""
    import shutil
    import tempfile

    import numpy as np
    import torch

    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200.hostref import init_sample_draw, lattice_dist
    from paper_2604_26555_b200.shards import write_shards
    local = ctx["local"]
    seed, n, epochs = SEEDS["c5"], 125_000_000, EPOCHS
    topo = lattice_dist("hex", *P_GRID)
    etas, sigmas = hex_schedule(epochs)
    out = {"workload": "c5: 32x32 hex SOM (1024 nodes), one GPU's 1.25e8 x 50-row share of the "
                       "1e9-row, 8-GPU job; resident, streamed from pinned host, streamed from "
                       "FSOMSHRD shards (cold page cache)", "unit": UNIT, "rows": n}
    # resident: the rows generated on the device
    e = tsom.Engine(P, D, device=local)
    e.bind_synthetic_gmm(n, seed, 16, 0)
    w0 = init_sample_draw(EngineRows(e), P, seed)
    e.set_codebook(w0)
    e.set_topology_distance(topo)
    e.train_epochs(etas[:2], sigmas[:2])
    e.set_codebook(w0)
    with ClockSampler(local) as clk:
        secs, _ = timed(lambda: e.train_epochs(etas, sigmas), ctx, e)
    out["resident"] = {"value": n * epochs / secs, "ms_per_epoch": secs * 1e3 / epochs,
                       "clocks": clk.summary(),
                       "engine_bytes": e.device_bytes,
                       "bytes_per_row": round(e.device_bytes / n, 1),
                       "device_used_gb": hbm_used_gb(local)}
    # the same rows to page-locked host memory (25 GB), then streamed every epoch
    host = pinned_rows(n)
    e.get_rows(0, n, host)
    close_engine(e)
    h2d = h2d_gbs(local)
    e = tsom.Engine(P, D, device=local)
    e.bind(host, streamed=True)
    e.set_codebook(w0)
    e.set_topology_distance(topo)
    e.train_epochs(etas[:1], sigmas[:1])
    e.set_codebook(w0)
    k = 3
    secs, _ = timed(lambda: e.train_epochs(etas[:k], sigmas[:k]), ctx)
    bw = n * D * 4 * k / secs / 1e9
    out["streamed_pinned_host"] = {
        "value": n * k / secs, "ms_per_epoch": secs * 1e3 / k, "epochs": k,
        "h2d_gbs_achieved": bw, "h2d_gbs_measured_peak": h2d, "frac_of_h2d": bw / h2d,
        "engine_bytes": e.device_bytes, "timing": "wall clock (host staging in the loop)"}
    close_engine(e)
    # FSOMSHRD shards on local disk, page cache dropped (cold), streamed
    sdir = tempfile.mkdtemp(prefix="tsom_c5_", dir=args.shard_dir)
    try:
        t0 = time.perf_counter()
        paths = write_shards(host, sdir, 16)
        for pth in paths:
            fd = os.open(pth, os.O_RDONLY)
            os.fsync(fd)
            os.close(fd)
        t_write = time.perf_counter() - t0
        del host
        for pth in paths:  # cold: evict the files from the page cache
            fd = os.open(pth, os.O_RDONLY)
            os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
            os.close(fd)
        e = tsom.Engine(P, D, device=local)
        e.bind_shards(paths, streamed=True)
        e.set_codebook(w0)
        e.set_topology_distance(topo)
        cold, _ = timed(lambda: e.train_epochs(etas[:1], sigmas[:1]), ctx)
        warm, _ = timed(lambda: e.train_epochs(etas[1:2], sigmas[1:2]), ctx)
        nbytes = n * D * 4
        out["streamed_shards"] = {
            "value_cold": n / cold, "value_warm": n / warm,
            "ms_per_epoch_cold": cold * 1e3, "ms_per_epoch_warm": warm * 1e3,
            "disk_read_gbs_cold": nbytes / cold / 1e9, "read_gbs_warm": nbytes / warm / 1e9,
            "frac_of_h2d_warm": nbytes / warm / 1e9 / h2d,
            "shards": len(paths), "write_s": t_write,
            "note": "cold = first epoch after posix_fadvise(DONTNEED) on every file (bound by "
                    "the disk); warm = the next epoch, the files then in the page cache "
                    "(bound by the pread staging + H2D)"}
        close_engine(e)
    finally:
        shutil.rmtree(sdir, ignore_errors=True)
    out["value"] = out["resident"]["value"]
    return out


def leg_c1(args, ctx):
    """Config c1 in full: 10x10 rectangular lattice, 1e5 x 50
    rows from the reference's generator, 10 epochs: the device loop
    (toposom_b200::train_device) against the reference's own run on the host
    cores (oracle/_ref train_parallel, G = nproc, and G = 1 on 2 epochs) on
    identical inputs, with the QE of both trained codebooks."""
    import numpy as np

    import oracle
    from paper_2604_26555_b200 import dropin
    if not dropin.available() or ctx["rank"] != 0:
        return {"skipped": "needs libtsom_dropin.so (rank 0)"}
    seed, n = SEEDS["c1"], 100_000
    x = host_gmm_rows(n, seed, pinned=False)
    cfg = dropin.TrainConfig(topology="rect", grid_w=10, grid_h=10, n_iters=EPOCHS, seed=seed)
    dropin.train_device(dropin.TrainConfig(topology="rect", grid_w=10, grid_h=10, n_iters=1,
                                           seed=seed), x, device=ctx["local"])
    # best of 3 whole runs (a 10-ms run: host-side jitter dominates one sample)
    runs = [dropin.train_device(cfg, x, device=ctx["local"], log_qe=True) for _ in range(3)]
    w_gpu, qe_gpu, _, secs = min(runs, key=lambda r: r[3])
    out = {"workload": "c1: 10x10 rect SOM, 1e5 x 50 GMM rows (reference generator), 10 epochs "
                       "(in full)", "unit": UNIT, "value": n * EPOCHS / secs,
           "seconds": secs,
           "path": "toposom_b200::train_device, wall clock (host data), best of 3 runs"}
    if args.no_cpu:
        return out
    chk = oracle.best()
    cores = os.cpu_count() or 1
    ocfg = oracle.SomConfig(topology="rect", grid_w=10, grid_h=10, n_iters=EPOCHS, seed=seed,
                            n_threads=cores)
    t0 = time.perf_counter()
    w_cpu, qe_cpu, _ = chk.train(ocfg, x, log_qe=True)
    t_cpu = time.perf_counter() - t0
    ocfg1 = oracle.SomConfig(topology="rect", grid_w=10, grid_h=10, n_iters=2, seed=seed,
                             n_threads=1)
    t0 = time.perf_counter()
    chk.train(ocfg1, x)
    t1 = time.perf_counter() - t0
    out["cpu_baseline"] = {"value": n * EPOCHS / t_cpu, "unit": UNIT, "cores": cores,
                           "kind": chk.kind, "seconds": t_cpu,
                           "sample": "c1 in full (1e5 rows, 10 epochs, log_qe), train_parallel "
                                     f"G={cores}",
                           "single_thread": {"value": n * 2 / t1, "seconds": t1,
                                             "sample": "c1 rows, 2 epochs, G=1"}}
    out["qe_vs_cpu"] = {"qe_gpu": float(qe_gpu[-1]), "qe_cpu_reference": float(qe_cpu[-1]),
                        "rel_diff": float(abs(qe_gpu[-1] - qe_cpu[-1]) / qe_cpu[-1]),
                        "qe_rel_diff_max_over_epochs": float(np.max(np.abs(qe_gpu - qe_cpu)
                                                                    / qe_cpu)),
                        "codebook_rel_maxnorm": float(np.max(np.abs(w_gpu.astype(np.float64)
                                                                    - w_cpu))
                                                      / np.max(np.abs(w_cpu)))}
    return out


def roofline_peak(kernel, pk):
    """Dense tensor peak the K1 kernel is bounded by, in useful-flop terms."""
    if kernel == 3:  # kind::f16 runs at the bf16 rate; 3 split products per useful MAC
        return "tcgen05 3xFP16", pk["bf16_tflops"] / 3.0, "/ 3 (3xFP16 split)"
    if kernel == 2:  # kind::tf32 runs at half the bf16 rate
        return "tcgen05 3xTF32", pk["bf16_tflops"] / 2.0 / 3.0, "/ 2 (TF32) / 3 (3xTF32 split)"
    return "SIMT FP32", pk.get("fp32_tflops", 75.0), "(FP32 SIMT, nominal)"


# ncu --set full, one launch of K1 at the bench shape (1e7 x 50, K=1024, rows in
# BMU order, A tiles multicast over clusters of 2 group CTAs):
# dram__bytes_read.sum + dram__bytes_write.sum, bytes per launch
# (profiles/r02c_ncu_full_summary.json, scripts/round2d_profiles.sh).  The split A
# tiles are 3.2 GB: each leaves DRAM 1.0-1.16 times over the captures (6.1 GB
# without the multicast, the 4 group CTAs streaming every tile and L2 catching part).
K1_TRAFFIC = {3: 3.721560e9 + 0.320970e9}
K1_TRAFFIC_SRC = "profiles/r02c_ncu_full_summary.json, k1_bmu_tc<2, 0, 0, 1> (clusters of 2): " \
                 "3.72 GB read (the 3.2 GB of split A tiles 1.16 times; each cluster loads a " \
                 "tile once and multicasts it) + 0.32 GB per-group partial-result writes"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 SIMT, 2 tcgen05 3xTF32, 3 tcgen05 3xFP16")
    ap.add_argument("--row-order", type=int, default=None,
                    help="TSOM_OPT_ROW_ORDER for the c2 engines (default: the engine's, 1)")
    ap.add_argument("--image", type=int, default=None, help=argparse.SUPPRESS)  # c4: split image A/B
    ap.add_argument("--k1-debug", type=int, default=None, help=argparse.SUPPRESS)  # option 99 A/B
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the c4 (1e8 rows, adaptive) leg")
    ap.add_argument("--no-c3", action="store_true", help="skip the c3 (MST, 1e8 rows) leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the c5 (1.25e8 rows, streamed) leg")
    ap.add_argument("--no-c1", action="store_true", help="skip the c1 (in full vs the CPU) leg")
    ap.add_argument("--only", default="", help="comma list of extra legs to run (c1,c3,c4,c5)")
    ap.add_argument("--shard-dir", default=None, help="where the c5 leg writes its shard files")
    ap.add_argument("--force-comm", action="store_true", help=argparse.SUPPRESS)  # NCCL at N=1
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
