#!/usr/bin/env python
"""Headline benchmark: samples·epochs/s of batch-SOM training (K=1024, D=50).

Workload (BASELINE.json configs[1]): 32x32 hexagonal lattice (1024 nodes),
10,000,000 x 50 synthetic Gaussian-mixture rows per GPU,
full sampling.  One *step* = one training epoch over all rows: influence(σ)
→ BMU search (K1) → exact near-tie re-check → per-BMU accumulation (K2) →
reduce [+ NCCL allreduce for N>1] → FP64 smoothing (K3) → apply_update.

  value : device-timed epochs with the rows resident in HBM (CUDA events on
          the engine stream, max over ranks); inputs (2 GB/GPU) exceed L2.
  e2e   : the reference's own training loop (train_with_executor) with the
          B200 CudaExecutor, from a host DataMatrix: the timed region includes
          the host→device upload of the rows, every epoch's codebook/influence
          upload and accumulator download (wall clock).
  --impl reference : the reference CPU implementation (oracle/_ref =
          /root/reference headers compiled, train_parallel on all host cores)
          on a bounded sample of the same workload.

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
SEED = 2602  # seed = 2604 + config number - 2 ... config c2
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
    steps = max(1, min(args.steps, 5))
    value, cores, kind, sample, t = cpu_reference(step_seconds=4.0, steps=steps,
                                                  warmup=min(args.warmup, 1))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": min(args.warmup, 1), "ms_per_step": t * 1e3, "higher_is_better": True,
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

def host_gmm_rows(n, seed):
    """Host (pinned) GMM rows of the SURVEY §8(d) shape: centres from the
    reference Rng(seed, synth), component + unit noise drawn on the GPU with
    torch (values do not change dense-loop cost; parity runs use the
    reference generator)."""
    import numpy as np
    import torch

    from paper_2604_26555_b200.hostref import Rng
    r = Rng(seed, "synth")
    centres = np.array([[-4.0 + 8.0 * r.real01() for _ in range(D)] for _ in range(16)],
                       np.float32)
    g = torch.Generator(device="cuda").manual_seed(seed)
    comp = torch.randint(0, 16, (n,), device="cuda", generator=g)
    x = torch.randn((n, D), device="cuda", generator=g, dtype=torch.float32)
    x += torch.from_numpy(centres).cuda()[comp]
    host = torch.empty((n, D), dtype=torch.float32, pin_memory=True)
    host.copy_(x)
    del x, comp
    torch.cuda.empty_cache()
    return host.numpy()


def run_gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200 import _lib
    from paper_2604_26555_b200.hostref import (init_sample_draw, lattice_dist,
                                               resolved_sigma0, schedule_value)

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    n = N_PER_GPU

    # this rank's shard of the workload (weak scaling: n rows per GPU)
    host = host_gmm_rows(n, SEED + rank)
    eng = tsom.Engine(P, D, device=local)
    if args.kernel:
        eng.set_option(_lib.TSOM_OPT_BMU_KERNEL, args.kernel)
    eng.bind(host)
    active_kernel = eng.active_bmu_kernel

    def attach_comm(e):
        # one NCCL communicator per engine: rank 0's unique id over the gloo group
        if world > 1 or args.force_comm:
            uid = [e.comm_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(uid, src=0)
            e.comm_init(uid[0], rank, world)

    attach_comm(eng)
    # init_weights(sample_draw) (trainer.hpp:192-211) over rank 0's rows, same on every rank
    w0 = [init_sample_draw(host, P, SEED) if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(w0, src=0)
    w0 = w0[0]
    eng.set_codebook(w0)
    eng.set_topology_distance(lattice_dist("hex", *P_GRID))
    sigma0 = resolved_sigma0("hex", *P_GRID)

    def epoch(t):
        tt = t % EPOCHS
        eta = schedule_value(0.5, "linear", tt, EPOCHS, 1e-4)
        sigma = schedule_value(sigma0, "linear", tt, EPOCHS, 0.3)
        eng.train_epoch(eta, sigma)

    for t in range(args.warmup):
        epoch(t)
    stream = torch.cuda.ExternalStream(eng.stream, device=f"cuda:{local}")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.kernel_launches()
    k1_ms, total_ms, rechecks, phases = [], [], [], []
    # the K timed epochs go to the engine in one tsom_train_epochs call: every
    # epoch is the full epoch of tsom_train_epoch, enqueued back to back with
    # the schedules precomputed (no host round trip between epochs)
    steps_t = range(args.warmup, args.warmup + args.steps)
    etas = [schedule_value(0.5, "linear", t % EPOCHS, EPOCHS, 1e-4) for t in steps_t]
    sigmas = [schedule_value(sigma0, "linear", t % EPOCHS, EPOCHS, 0.3) for t in steps_t]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        eng.train_epochs(etas, sigmas)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.kernel_launches() - launches0
    k1_ms.append(eng.timing_detail()["k1_ms"])  # mean main-pass K1 over the timed epochs
    elapsed = ev0.elapsed_time(ev1)
    if world > 1:
        tmax = torch.tensor([elapsed], dtype=torch.float64)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        elapsed = float(tmax.item())
        dist.barrier()
    ms = elapsed / args.steps
    value = n * world / (ms / 1e3)
    # phase breakdown and re-check counts from three untimed single-epoch calls
    for t in range(args.warmup + args.steps, args.warmup + args.steps + 3):
        epoch(t)
        det = eng.timing_detail()
        phases.append(det)
        total_ms.append(det["total_ms"])
        rechecks.append(eng.last_recheck_count)
    s, c = eng.qe()
    qe_gpu = s / c
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

    eng.close()
    eng = None
    # e2e through the public C-ABI with HOST buffers (rank 0, N=1): bind the host
    # rows (H2D), run the epochs, read the codebook back (D2H) — all inside the
    # wall-clock region; then the same workload through the reference's own
    # training loop with the CudaExecutor plugin (libtsom_dropin.so).
    e2e = None
    if not args.no_e2e:
        topo_d = lattice_dist("hex", *P_GRID)  # host input, like the rows

        def cabi_run(epochs):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e = tsom.Engine(P, D, device=local)
            if args.kernel:
                e.set_option(_lib.TSOM_OPT_BMU_KERNEL, args.kernel)
            ta = time.perf_counter()
            e.bind(host)
            tb = time.perf_counter()
            attach_comm(e)
            e.set_codebook(w0)
            e.set_topology_distance(topo_d)
            t1 = time.perf_counter()
            e.train_epochs([schedule_value(0.5, "linear", t, epochs, 1e-4) for t in range(epochs)],
                           [schedule_value(sigma0, "linear", t, epochs, 0.3)
                            for t in range(epochs)])
            wf = e.get_codebook()
            t2 = time.perf_counter()
            e.close()
            t3 = time.perf_counter()
            return t3 - t0, {"setup_s": t1 - t0, "epochs_s": t2 - t1, "close_s": t3 - t2,
                             "create_s": ta - t0, "bind_s": tb - ta, "config_s": t1 - tb}
        cabi_run(1)  # warm-up (allocations, module load)
        runs = []
        for _ in range(3):
            secs_r, split_r = cabi_run(EPOCHS)
            if world > 1:  # the job ends when the slowest rank ends
                tm = torch.tensor([secs_r], dtype=torch.float64)
                dist.all_reduce(tm, op=dist.ReduceOp.MAX)
                secs_r = float(tm.item())
            runs.append((secs_r, split_r))
        secs, split = min(runs, key=lambda r: r[0])
        h2d = n * D * 4 + P * D * 4 + P * P * 8
        d2h = P * D * 4
        e2e = {"value": n * world * EPOCHS / secs, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d / EPOCHS), "d2h_bytes_per_step": int(d2h / EPOCHS),
               "path": "C-ABI tsom_bind_host_data + tsom_train_epochs (10 epochs) + tsom_get_codebook "
                       "from pinned host rows, wall clock incl. engine creation (and the "
                       "NCCL communicator when N > 1), max over ranks; device buffers come "
                       "from the engines' per-device caching pool, warm after the warm-up call",
               "seconds_per_call": secs, "epochs_per_call": EPOCHS, "best_of": 3,
               "split_s": split}
        from paper_2604_26555_b200 import dropin
        if world == 1 and dropin.available():
            cfg = dropin.TrainConfig(topology="hex", grid_w=P_GRID[0], grid_h=P_GRID[1],
                                     n_iters=EPOCHS, seed=SEED)
            warm = dropin.TrainConfig(topology="hex", grid_w=P_GRID[0], grid_h=P_GRID[1],
                                      n_iters=1, seed=SEED)
            dropin.train_cuda(warm, host[:200_000], device=local)
            _, _, _, dsecs = dropin.train_cuda(cfg, host, device=local)
            dropin.train_device(warm, host[:200_000], device=local)
            _, _, _, vsecs = dropin.train_device(cfg, host, device=local)
            e2e["dropin_device_loop"] = {
                "value": n * EPOCHS / vsecs, "seconds_per_call": vsecs,
                "path": "toposom_b200::train_device (C++ drop-in: init_weights and lattice "
                        "distances as the reference builds them, then every epoch step on the "
                        "device; host DataMatrix bound through the pinned staging)"}
            e2e["dropin_reference_loop"] = {
                "value": n * EPOCHS / dsecs, "seconds_per_call": dsecs,
                "path": "toposom::train_with_executor + toposom_b200::CudaExecutor "
                        "(host DataMatrix; reference host code per epoch: sampler, influence, "
                        "apply_update, int128 accumulators)"}
    pk, pk_kind = peaks()
    k1 = statistics.mean(k1_ms) if k1_ms else float("nan")
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
            "k1_ms": k1, "epoch_ms": statistics.mean(total_ms) if total_ms else None,
            "phase_ms": {k: statistics.mean(p[k] for p in phases) for k in phases[0]} if phases else None}
    # K2 (accumulation) against HBM: 204 algorithmic bytes per row (the row
    # and its BMU) over the accumulate phase's event time
    acc_ms = statistics.mean(p["accum_ms"] for p in phases) if phases else float("nan")
    k2_gbs = n * 204 / (acc_ms / 1e3) / 1e9 if acc_ms > 0 else 0.0
    k2_roof = {"bound": "hbm", "kernel": "k2 sort + TMA gather + piece reduce",
               "achieved": k2_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
               "frac": k2_gbs / pk["hbm_gbs"], "accum_ms": acc_ms,
               "note": "achieved = 204 B/row x rows / accumulate-phase event time (3 untimed "
                       "epochs); the gather reads ~1.6x that from DRAM (200-B rows at random "
                       "positions touch 2-3 128-B lines)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": {3: "f32 via 3xFP16 split", 2: "f32 via 3xTF32 split", 1: "f32"}[active_kernel]
                 + " BMU (exact FP64 re-check) + f64 accumulate/update",
        "data": "synthetic Gaussian mixture (16 comps, U[-4,4] centres, unit noise), random-init "
                "codebook by sample_draw",
        "config": {"workload": "c2: 32x32 hex SOM (1024 nodes), 1e7 x 50 rows per GPU, full "
                               "sampling, resident in HBM", "model": "batch-SOM",
                   "nodes": P, "dims": D, "rows_per_gpu": n, "global_rows": n * world,
                   "parallelism": f"dp{world}", "l2": "inputs (2 GB/GPU) > L2 (126 MB); no flush"},
        "roofline": roof,
        "roofline_k2": k2_roof,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "qe_gpu_after": qe_gpu,
        "qe_vs_cpu": qe_check,
        "rechecked_rows_per_epoch": statistics.mean(rechecks) if rechecks else None,
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_c4:
        if eng is not None:
            eng.close()
        torch.cuda.empty_cache()
        c4 = run_c4_leg(local, world=world, rank=rank, attach=attach_comm,
                        bcast=(lambda o: (dist.broadcast_object_list(o, src=0), o)[1])
                        if world > 1 else None,
                        tmax=(lambda v: (lambda tm: (dist.all_reduce(tm, op=dist.ReduceOp.MAX),
                                                     float(tm.item()))[1])(
                            torch.tensor([v], dtype=torch.float64))) if world > 1 else None)
        if rank == 0:
            line["c4"] = c4
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


def run_c4_leg(local, n=100_000_000, rho=0.1, epochs=EPOCHS, warm=2, world=1, rank=0,
               attach=None, bcast=None, tmax=None):
    """Config c4: 1024-node RNG-topology SOM, 1e8 x 50 GMM rows
    resident in HBM (split over the ranks: n / world rows each), adaptive
    sampler with rho = 0.1 on the device (select -> epoch over the selected rows
    -> observe; with N > 1 one sharded sampler over all rows, its digit
    histograms allreduced over NCCL), RNG graph refreshed on the device on the
    reference schedule.  Every per-epoch step is on the GPU; timed with CUDA
    events on the engine stream, max over ranks."""
    import numpy as np
    import torch

    import paper_2604_26555_b200 as tsom
    from paper_2604_26555_b200.hostref import (RefreshState, Rng, init_sample_draw,
                                               resolved_sigma0, schedule_value)
    seed = 2608
    n_total = n
    n = n_total // world + (1 if rank < n_total % world else 0)
    r = Rng(seed, "synth")
    centres = np.array([[-4.0 + 8.0 * r.real01() for _ in range(D)] for _ in range(16)],
                       np.float32)
    g = torch.Generator(device=f"cuda:{local}").manual_seed(seed + rank)
    x = torch.randn((n, D), device=f"cuda:{local}", generator=g, dtype=torch.float32)
    comp = torch.randint(0, 16, (n,), device=f"cuda:{local}", generator=g)
    x += torch.from_numpy(centres).to(x.device)[comp]
    del comp

    class _Rows:  # init_sample_draw over device rows: only the picked rows come back
        shape = (n, D)

        def __getitem__(self, idx):
            return x[torch.from_numpy(np.asarray(idx)).to(x.device)].cpu().numpy()

    e = tsom.Engine(P, D, device=local)
    e.bind_device(x.data_ptr(), n)
    if attach is not None:
        attach(e)
    w0 = [init_sample_draw(_Rows(), P, seed) if rank == 0 else None]
    if bcast is not None:
        w0 = bcast(w0)
    e.set_codebook(w0[0])
    m = max(1, int(np.floor(n_total * rho)))
    e.sampler_init("adaptive", m, seed)
    sigma0 = resolved_sigma0("rng", 0, 0, 0.0)
    refresh = RefreshState(max(1, epochs // 10), 1.5, 25)
    stream = torch.cuda.ExternalStream(e.stream, device=f"cuda:{local}")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def epoch(t):
        tt = t % epochs
        if refresh.should_refresh(tt):
            e.refresh_topology("rng")
            refresh.mark(tt)
        eta = schedule_value(0.5, "linear", tt, epochs, 1e-4)
        sigma = schedule_value(sigma0, "linear", tt, epochs, 0.3)
        e.train_epoch(eta, sigma, sampled=True)

    for t in range(warm):
        epoch(t)
    refresh = RefreshState(max(1, epochs // 10), 1.5, 25)
    torch.cuda.synchronize()
    phases, rechecks = [], []
    ev0.record(stream)
    for t in range(epochs):
        epoch(t)
        phases.append(e.timing_detail())
        rechecks.append(e.last_recheck_count)
    ev1.record(stream)
    torch.cuda.synchronize()
    secs = ev0.elapsed_time(ev1) / 1e3
    if tmax is not None:
        secs = tmax(secs)
    s, c = e.qe()
    e.close()
    del x
    torch.cuda.empty_cache()
    return {"workload": "c4: 1024-node RNG-topology SOM (device refresh), 1e8 x 50 GMM rows "
                        "resident (split over the GPUs), adaptive sampler rho=0.1 on the device "
                        "(one sharded sampler), 10 epochs",
            "value": m * epochs / secs, "unit": "selected samples*epochs/s", "n_gpus": world,
            "rows_considered_per_s": n_total * epochs / secs, "ms_per_epoch": secs * 1e3 / epochs,
            "phase_ms": {k: round(statistics.mean(p[k] for p in phases), 3) for k in phases[0]},
            "rechecked_rows_per_epoch": statistics.mean(rechecks),
            "qe_after": s / c}


def roofline_peak(kernel, pk):
    """Dense tensor peak the K1 kernel is bounded by, in useful-flop terms."""
    if kernel == 3:  # kind::f16 runs at the bf16 rate; 3 split products per useful MAC
        return "tcgen05 3xFP16", pk["bf16_tflops"] / 3.0, "/ 3 (3xFP16 split)"
    if kernel == 2:  # kind::tf32 runs at half the bf16 rate
        return "tcgen05 3xTF32", pk["bf16_tflops"] / 2.0 / 3.0, "/ 2 (TF32) / 3 (3xTF32 split)"
    return "SIMT FP32", pk.get("fp32_tflops", 75.0), "(FP32 SIMT, nominal)"


# ncu --set full, one launch of K1 at the bench shape (1e7 x 50, K=1024):
# dram__bytes_read.sum + dram__bytes_write.sum, bytes per launch.  Captures
# (profiles/r01_ncu_full_summary*.json) saw 3.74, 6.61, 5.82 and 5.17 GB read:
# the A tiles (3.2 GB) are read by the 4 codebook-group CTAs and L2 catches a
# run-dependent part of the repeats; the latest capture is reported.
K1_TRAFFIC = {3: 5.170710e9 + 0.319864e9}
K1_TRAFFIC_SRC = "profiles/r01_ncu_full_summary_d.json, k1_bmu_tc<2, 0>: 5.17 GB read (split A " \
                 "tiles 3.2 GB, each read by the 4 node-group CTAs, partly from L2; earlier " \
                 "captures 3.74-6.61 GB) + 0.32 GB per-group partial-result writes"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 SIMT, 2 tcgen05 3xTF32, 3 tcgen05 3xFP16")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the c4 (1e8 rows, adaptive) leg")
    ap.add_argument("--only-c4", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--force-comm", action="store_true", help=argparse.SUPPRESS)  # NCCL at N=1
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.only_c4:  # diagnostics: the c4 leg alone
        import torch
        torch.cuda.set_device(0)
        print(json.dumps(run_c4_leg(0, epochs=args.steps if args.steps < 50 else EPOCHS)),
              flush=True)
        return 0
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
