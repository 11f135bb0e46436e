#!/usr/bin/env python
"""bench.py — B200 Lindblad propagation engine benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C] [--scaling strong|weak]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

Headline workload (BASELINE.json configs[1], "c1"): d = 3 transmon with
leakage, ONE shared P = exp(L dt) (9x9 complex128), 2^20 independent
trajectories, 1,000 propagation steps per pass. One bench "step" = one pass of
the hot path (vec(rho_b) <- P vec(rho_b), 1,000 times, for every trajectory).
metric = trajectory-steps/s (whole job), FP64 GFLOP/s counted as 8 d^4 = 648
flops per trajectory-step.

Multi-GPU: the configs fix the GLOBAL batch. With
--scaling strong (default) rank r of W owns the global trajectory ids
[floor(r B / W), floor((r + 1) B / W)); inputs are keyed on the global id, so
results are independent of W; stepping has no inter-GPU traffic, and config
4's ensemble mean is the engine's one collective (lbg_ensemble_mean_dev over
the engine's own NCCL communicator, lbg_nccl_*). --scaling weak gives every
rank the full per-GPU batch instead. Time = max over ranks of the CUDA-event
time, value = global trajectory-steps / that time.

value: inputs resident in HBM (151 MB state > 126 MB L2, so no L2 flush is
needed), CUDA events on the launching stream, barrier + synchronize around
exactly K passes. e2e: the same metric through the host-buffer C-ABI call
lbg_evolve_shared_p (H2D of rho0, rho0 validation, the steps, D2H of the
final states) timed per call, from pinned buffers and — as lb::MatrixAoS
holds them — from pageable ones; each checked against the device result.
roofline: FP64 pipe bound; peak = the FP64 DMMA throughput measured live by
lbg_fp64_peak() (MEASURED_PEAKS.json has no FP64 figure). cpu_baseline: the
reference (oracle/_ref/libref.so, compiled from /root/reference sources with
its native-fast flags) on the box's host threads.
Extra keys at N = 1: "configs" (c0, c2, c3, c4 and the side tables) and
"strong_scaling_projection" (each batched config timed at B, B/2, B/4, B/8 on
this GPU: T(B) / T(B/W) is the projected W-GPU speed-up, since the shards never
talk while stepping). A one-line text summary precedes the JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # cfg: (d, global batch, steps)
    0: (3, 1, 10000),
    1: (3, 1 << 20, 1000),
    2: (9, 4096, 1000),
    3: (27, 1024, 200),
    4: (9, 65536, 500),
}
WORKLOAD = {
    0: "c0: d=3 single transmon, 1 trajectory x 10,000 steps, complex128 (latency)",
    1: "c1: d=3 shared P (9x9), 2^20 Ginibre trajectories x 1,000 steps, complex128",
    2: "c2: d=9 two transmons, shared P (81x81), 4,096 Ginibre trajectories x 1,000 steps",
    3: "c3: d=27 three transmons, shared P (729x729, 8.5 MB), 1,024 trajectories x 200 steps",
    4: "c4: d=9 sweep, per-trajectory L/P built on GPU, 65,536 trajectories x 500 steps",
}
KERNEL = {0: "chain_kernel", 1: "dfma9_kernel", 2: "smem_cluster_kernel", 3: "tiled_evolve_kernel",
          4: "ptm_expm_kernel+ptm_step_kernel"}


def flops_per_traj_step(d: int) -> int:
    return 8 * d ** 4


def share(rank: int, world: int, batch: int) -> tuple[int, int]:
    """Global trajectory ids [lo, hi) of rank `rank`."""
    return rank * batch // world, (rank + 1) * batch // world


def config_dict(cfg: int, world: int, scaling: str) -> dict:
    """The `config` key, identical in both arms."""
    d, B, S = CONFIGS[cfg]
    strong = scaling == "strong" and cfg != 0
    gb = B if strong else B * world
    return {"workload": WORKLOAD[cfg], "d": d, "global_batch": gb, "steps_per_pass": S, "n_ranks": world,
            "partition": ("rank r owns global ids [floor(rB/W), floor((r+1)B/W))" if strong
                          else "replicas: every rank runs the one trajectory" if cfg == 0
                          else "every rank owns its own batch of B (weak)"),
            "l2": "state larger than L2; no flush needed" if cfg == 1 else "working set L2/SMEM resident"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# ---------------------------------------------------- GPU roofline placement ---
# B200 re-targeting of the reference's CPU model (proj/src/roofline.cpp:62-99:
# characterize -> place -> classify). Levels are where P lives while stepping.
B200_PROFILE = {
    "levels": ["regs/const", "smem", "l2", "hbm"],
    "capacity_bytes": [None, 227 * 1024, 126 * 2 ** 20, 180 * 10 ** 9],
    "bw_gbs": [None, 36895.5, 15363.8, 6465.2],
}


def roofline_place(d: int, batch: int, shared_p: bool, peak_tflops: float, tile: int = 32) -> dict:
    """characterize (8 d^4 flops per trajectory-step; roofline.cpp:62-74), place P
    on the B200 ladder (roofline.cpp:76-87) and classify (roofline.cpp:93-99)."""
    n = d * d
    p_bytes = 16 * n * n
    flops = 8 * d ** 4 * batch
    prof = B200_PROFILE
    if shared_p:
        if d == 3:
            level, bytes_ = 0, 0
        elif p_bytes <= prof["capacity_bytes"][1]:
            sms = min(148, -(-batch // tile))
            level, bytes_ = 1, p_bytes * sms
        elif p_bytes <= prof["capacity_bytes"][2]:
            level, bytes_ = 2, flops / (8 * tile * tile / (16 * 2 * tile))
        else:
            level, bytes_ = 3, p_bytes + 32 * n * batch
    else:
        level, bytes_ = (0, 0) if n <= 81 else (3, (n * n * 16 + 32 * n) * batch)
    ai = flops / bytes_ if bytes_ else float("inf")
    bw = prof["bw_gbs"][level]
    attainable = peak_tflops if bw is None else min(peak_tflops, ai * bw / 1e3)
    return {"level": prof["levels"][level], "ai_flop_per_byte": ai if bytes_ else None,
            "attainable_tflops": attainable}


class Clocks:
    """nvidia-smi samples during the timed region (the recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler must be live before the timed region starts (nvidia-smi
            # takes ~1 s to initialise NVML, longer than a short timed region)
            t0 = time.perf_counter()
            while not self.rows and self.proc.poll() is None and time.perf_counter() - t0 < 10:
                time.sleep(0.01)
            self.rows.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


# --------------------------------------------------------------- reference ---
def cpu_reference_rate(cfg: int, sample: int, threads: int, reps: int = 1, warmup: int = 0):
    """traj-steps/s of the unmodified reference (lb::evolve, native-fast SoA)."""
    from oracle.bindings import Oracle, Reference
    o, r = Oracle(), Reference()
    d, _, S = CONFIGS[cfg]
    if cfg == 4:
        dl = np.array([o.sweep_params(42, b)[0] for b in range(sample)])
        sc = np.array([o.sweep_params(42, b)[1] for b in range(sample)])
        times = []
        for i in range(warmup + reps):
            _, _, secs = r.sweep_batch(dl, sc, steps=S, threads=threads)
            if i >= warmup:
                times.append(secs)
        return sample * S / float(np.mean(times)), times
    P = r.config_propagator(cfg)
    if cfg == 0:
        rho0 = np.zeros((1, 3, 3), complex)
        rho0[0, 0, 0] = 1.0
    else:
        rho0 = o.ginibre_batch(42, cfg, 0, sample, d)
    times = []
    for i in range(warmup + reps):
        _, secs = r.evolve_batch(P, rho0, S, threads=threads)
        if i >= warmup:
            times.append(secs)
    return rho0.shape[0] * S / float(np.mean(times)), times


# trajectories per reference bench step: the full workload for c0-c3 (4.8 / 0.7 /
# 8 s per pass on the GPU box's 16 host threads), 1/16 of it for c4 (the CPU
# builds 65,536 propagators at 8.85 ms each; step cost is data-independent)
REF_SAMPLE = {0: 1, 1: 1 << 20, 2: 4096, 3: 1024, 4: 4096}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = args.config
    d, B, S = CONFIGS[cfg]
    threads = os.cpu_count() or 1
    sample = REF_SAMPLE[cfg]
    value, times = cpu_reference_rate(cfg, sample, threads, reps=args.steps, warmup=args.warmup)
    ms = float(np.mean(times)) * 1e3
    line = {
        "impl": "reference", "metric": "trajectory-steps/s", "value": value, "unit": "traj-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded Ginibre rho0 (counter-based RNG, seed 42), BASELINE config models",
        "gflops": value * flops_per_traj_step(d) / 1e9,
        "config": config_dict(cfg, args.gpus, args.scaling),
        "cpu_baseline": {"value": value, "unit": "traj-steps/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} trajectories x {S} steps per bench step through lb::evolve "
                                   f"(native-fast SoA, -march pinned to x86-64-v4), {threads} std::threads"},
        "e2e": {"value": value, "unit": "traj-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- ours ---
class Runner:
    def __init__(self, torch, lbg, dev, rank):
        self.torch, self.lbg, self.dev, self.rank = torch, lbg, dev, rank
        self.stream = torch.cuda.current_stream(dev)

    def propagator(self, cfg):
        h, ops = self.lbg.config_model(cfg)
        return self.lbg.expm(self.lbg.build_lindbladian(h, ops), 0.1)

    def shared_p_setup(self, cfg, lo, b):
        """P (built on the GPU) and global trajectories [lo, lo + b) on the device."""
        d, _, S = CONFIGS[cfg]
        T = self.torch
        P = self.propagator(cfg)
        if cfg == 0:
            rho0 = np.zeros((1, 3, 3), complex)
            rho0[0, 0, 0] = 1.0
        else:
            rho0 = self.lbg.ginibre_batch(cfg, lo, b, d)
        pt = T.from_numpy(P).to(self.dev)
        xt = T.from_numpy(rho0.reshape(b, d * d)).to(self.dev)
        ws = self.lbg.evolve_workspace(d * d, b)
        work = T.empty(max(ws, 1), dtype=T.uint8, device=self.dev)
        return P, rho0, pt, xt, work

    def time_passes(self, fn, K, W):
        T = self.torch
        for _ in range(W):
            fn()
        T.cuda.synchronize(self.dev)
        if T.distributed.is_initialized():
            T.distributed.barrier()
        evs = [T.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        self.lbg.reset_launch_count()
        evs[0].record(self.stream)
        for k in range(K):
            fn()
            evs[k + 1].record(self.stream)
        T.cuda.synchronize(self.dev)
        launches = self.lbg.launch_count()
        if T.distributed.is_initialized():
            T.distributed.barrier()
        per = [evs[k].elapsed_time(evs[k + 1]) for k in range(K)]
        total = evs[0].elapsed_time(evs[K])
        return total, per, launches


def max_over_ranks(torch, x: float) -> float:
    if torch.distributed.is_initialized():
        on_gpu = torch.distributed.get_backend() == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    return x


class SweepCase:
    """Config 4 through lbg_evolve_sweep_dev on global ids [lo, lo + b), then the
    ensemble mean over ranks (lbg_ensemble_mean_dev on the engine's NCCL comm)."""

    def __init__(self, torch, lbg, dev, lo, b, global_batch, comm=None, mode="auto"):
        self.torch, self.lbg, self.dev, self.B, self.mode = torch, lbg, dev, b, mode
        self.global_batch, self.comm = global_batch, comm
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        h0, hd, hs = lbg.config_sweep_terms()
        _, ops = lbg.config_model(4)
        delta, scale = lbg.sweep_params(lo, b)
        rho0 = np.zeros((9, 9), complex)
        rho0[0, 0] = 1.0
        self.host = (h0, hd, hs, ops, delta, scale, rho0)
        self.args = [T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(rho0), CONFIGS[4][2]]
        self.pops = torch.zeros(b, 9, dtype=torch.float64, device=dev)
        self.ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
        self.work = torch.empty(lbg.sweep_workspace(9, b), dtype=torch.uint8, device=dev)
        self.shared_gpu_group = (torch.distributed.is_initialized() and comm is None
                                 and torch.distributed.get_world_size() > 1)

    def run(self):
        self.lbg.evolve_sweep_dev(*self.args, self.pops, self.ens, self.work, mode=self.mode)
        if self.shared_gpu_group:  # tests only: ranks sharing one GPU cannot form an NCCL comm
            host = self.ens.cpu()
            self.torch.distributed.all_reduce(host)
            self.ens.copy_(host)
            self.lbg.ensemble_mean_dev(self.ens, self.global_batch, None)
        else:
            self.lbg.ensemble_mean_dev(self.ens, self.global_batch, self.comm)

    def e2e(self, reps=2):
        T, dev = self.torch, self.dev
        t0 = time.perf_counter()
        for _ in range(reps):
            args = [T.from_numpy(np.ascontiguousarray(a)).to(dev) for a in self.host]
            self.lbg.evolve_sweep_dev(*args[:6], 0.1, args[6], CONFIGS[4][2], self.pops, self.ens, self.work,
                                      mode=self.mode)
            pops = self.pops.cpu()
            ens = self.ens.cpu()
        s = (time.perf_counter() - t0) / reps
        h2d = sum(a.nbytes for a in self.host)
        return {"value": self.B * CONFIGS[4][2] / s, "unit": "traj-steps/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(pops.numel() * 8 + ens.numel() * 16), "ms_per_call": s * 1e3,
                "call": "lbg_evolve_sweep_dev (host inputs copied in, populations + ensemble copied out)"}


def host_call_e2e(torch, lbg, P, rho0, S, want, pinned, reps):
    """lbg_evolve_shared_p with pinned or pageable caller buffers: median call
    time, and the result against the device path's (`want`)."""
    import ctypes as C
    B, d = rho0.shape[0], rho0.shape[1]
    if pinned:
        pin = torch.empty(B * d * d * 2, dtype=torch.float64).pin_memory()
        pin_out = torch.empty_like(pin).pin_memory()
        host_in = pin.numpy().view(np.complex128).reshape(B, d, d)
        host_out = pin_out.numpy().view(np.complex128).reshape(B, d, d)
        host_in[...] = rho0
    else:
        host_in = np.array(rho0, copy=True)
        host_out = np.empty_like(host_in)
    L = lbg.lib()
    dp = C.POINTER(C.c_double)
    Pc = np.ascontiguousarray(P)

    def call():
        rc = L.lbg_evolve_shared_p(Pc.ctypes.data_as(dp), d, host_in.ctypes.data_as(dp), B, S,
                                   host_out.ctypes.data_as(dp), 0)
        assert rc == 0, L.lbg_last_error()
    call()
    diff = float(np.abs(host_out - want).max())
    call()  # a second untimed call: the first timed one otherwise absorbs one-off host costs
    assert diff <= 1e-12, f"host-buffer result differs from the device path by {diff}"
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
    calls = []
    for _ in range(reps):
        t0 = time.perf_counter()
        call()
        calls.append(time.perf_counter() - t0)
    return float(np.median(calls)), calls, int(host_in.nbytes + Pc.nbytes), int(host_out.nbytes), diff


def run_ours(args):
    import torch

    import paper_2603_18052_b200 as lbg

    rank, world, local = dist_env()
    # LBG_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0 with a gloo
    # process group, to exercise the multi-rank path on a single GPU. No kernel
    # waits on another rank, so sharing a GPU cannot deadlock.
    shared = os.environ.get("LBG_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not torch.distributed.is_initialized():
        if shared:
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=dev)
    lbg.lib()
    R = Runner(torch, lbg, dev, rank)
    cfg = args.config
    d, Bcfg, S = CONFIGS[cfg]
    K, W = args.steps, args.warmup
    strong = args.scaling == "strong" and cfg != 0  # c0 (one trajectory): replicas only
    gb = Bcfg if strong else Bcfg * world
    lo, hi = share(rank, world, gb) if strong else ((0, 1) if cfg == 0 else (rank * Bcfg, (rank + 1) * Bcfg))
    b = hi - lo
    dmma_peak, dfma_peak = lbg.fp64_peak()
    peak = dmma_peak
    traffic = load_traffic()

    comm = None  # the engine's own NCCL communicator (config 4's ensemble mean)
    if cfg == 4 and world > 1 and not shared:
        def bcast(raw):
            obj = [raw]
            torch.distributed.broadcast_object_list(obj, src=0)
            return obj[0]
        comm = lbg.NcclComm(rank, world, bcast)

    # ---- device-resident timed region -----------------------------------
    if cfg == 4:
        sweep = SweepCase(torch, lbg, dev, lo, b, gb, comm)
        fn = sweep.run
    else:
        P, rho0, pt, xt, work = R.shared_p_setup(cfg, lo, b)
        fn = lambda: lbg.evolve_batch_dev(pt, xt, S, work=work, stream=R.stream)  # noqa: E731
    with Clocks(local) as clk:
        total_ms, per_ms, launches = R.time_passes(fn, K, W)
    total_ms = max_over_ranks(torch, total_ms)
    units = gb * S * K
    value = units / (total_ms * 1e-3)
    ms_step = total_ms / K
    kernel_ms = float(np.mean(per_ms))
    achieved = flops_per_traj_step(d) * b * S / (kernel_ms * 1e-3) / 1e12

    # ---- end to end through the host-buffer C-ABI call ---------------------
    if cfg != 4:
        # the device result for the same inputs (one pass from rho0), for the e2e check
        xr = torch.from_numpy(rho0.reshape(b, d * d).copy()).to(dev)
        lbg.evolve_batch_dev(pt, xr, S, work=work, stream=R.stream)
        torch.cuda.synchronize(dev)
        want = xr.cpu().numpy().reshape(b, d, d)
        with Clocks(local) as eclk:  # clocks during the host-buffer calls too
            med, calls, h2d, d2h, diff = host_call_e2e(torch, lbg, P, rho0, S, want, True, 41)
        med_pg, calls_pg, _, _, diff_pg = host_call_e2e(torch, lbg, P, rho0, S, want, False, 11)
        e2e_s = max_over_ranks(torch, med)
        e2e_pg = max_over_ranks(torch, med_pg)
        e2e = {"value": gb * S / e2e_s, "unit": "traj-steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_call": e2e_s * 1e3, "ms_per_call_all": [round(c * 1e3, 3) for c in calls],
               "call": "lbg_evolve_shared_p (pinned host buffers, synchronous); median of 41 (the 35-125 ms call bursts seen before came from the runtime's blocking stream sync; the engine now spin-waits its host round trips: tools/e2e_bursts.py)",
               "max_abs_diff_vs_device": diff, "clocks": eclk.summary(),
               "pageable": {"value": gb * S / e2e_pg, "ms_per_call": e2e_pg * 1e3,
                            "ms_per_call_all": [round(c * 1e3, 3) for c in calls_pg],
                            "max_abs_diff_vs_device": diff_pg,
                            "call": "lbg_evolve_shared_p from pageable buffers (lb::MatrixAoS storage): "
                                    "staged through the pool's pinned buffers; median of 11"}}
    else:
        e2e = sweep.e2e(reps=2)
        e2e["value"] = gb * S / max_over_ranks(torch, e2e["ms_per_call"] * 1e-3)

    line = {
        "metric": "trajectory-steps/s", "value": value, "unit": "traj-steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded Ginibre rho0 (counter-based RNG, seed 42), BASELINE config models",
        "gflops": value * flops_per_traj_step(d) / 1e9,
        "config": config_dict(cfg, world, args.scaling),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic.get(KERNEL[cfg]),
                     "kernel": KERNEL[cfg] if b > 8192 or cfg in (0, 1, 4) else "auto (small-batch share)",
                     "peak_source": f"FP64 DMMA throughput measured live by lbg_fp64_peak() ({dmma_peak:.2f} TF/s; "
                                    f"DFMA loop {dfma_peak:.2f}); MEASURED_PEAKS.json has no FP64 entry",
                     "flops_per_launch": flops_per_traj_step(d) * b * S, "launch_ms": kernel_ms,
                     "trajectories_this_rank": b},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if cfg == 4:
        line["config"]["collective"] = ("lbg_ensemble_mean_dev over the engine's NCCL comm (lbg_nccl_*)"
                                        if comm is not None else
                                        "one rank: lbg_ensemble_mean_dev without a collective"
                                        if world == 1 else "gloo all-reduce stand-in, then lbg_ensemble_mean_dev (ranks share one GPU: tests only)")

    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        try:
            sample = REF_SAMPLE[cfg]
            cv, times = cpu_reference_rate(cfg, sample, threads, reps=1, warmup=0)
            line["cpu_baseline"] = {"value": cv, "unit": "traj-steps/s", "cores": threads, "kind": "reference",
                                    "cpu_model": cpu_model(),
                                    "sample": f"{sample} trajectories x {S} steps through lb::evolve "
                                              f"(native-fast SoA, -march pinned to x86-64-v4), {threads} "
                                              f"std::threads, {times[0]:.2f} s"}
            s1 = max(1, sample // 16)  # the reference's own methodology is single-core
            c1, t1 = cpu_reference_rate(cfg, s1, 1, reps=1, warmup=0)
            line["cpu_baseline"]["value_1core"] = c1
            line["cpu_baseline"]["sample_1core"] = f"{s1} trajectories x {S} steps, 1 thread, {t1[0]:.2f} s"
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "traj-steps/s", "cores": threads, "kind": "reference",
                                    "sample": f"unavailable: {e}"}

    if rank == 0 and world == 1 and not args.no_extra and args.config == 1:
        line["strong_scaling_projection"] = projection(torch, lbg, R)
        line["configs"] = extra_configs(torch, lbg, R, peak)
    if rank == 0:
        print(summary_text(line), flush=True)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    return 0


def projection(torch, lbg, R):
    """Each batched config at its global batch B and at the per-rank shares
    B/2, B/4, B/8 on this GPU; T(B) / T(B/W) is the projected W-GPU speed-up
    (the shards never communicate while stepping; config 4's ensemble mean is
    one 1.3 KB allreduce per pass)."""
    out = {}
    for cfg in (1, 2, 3, 4):
        d, B, S = CONFIGS[cfg]
        row = {}
        for W in (1, 2, 4, 8):
            b = B // W
            if cfg == 4:
                case = SweepCase(torch, lbg, R.dev, 0, b, b)
                tot, per, _ = R.time_passes(case.run, 5, 2)
            else:
                _, _, pt, xt, work = R.shared_p_setup(cfg, 0, b)
                tot, per, _ = R.time_passes(
                    lambda: lbg.evolve_batch_dev(pt, xt, S, work=work, stream=R.stream), 5, 2)
            row[W] = float(np.median(per))  # robust to a pass disturbed by the shared box
        out[f"c{cfg}"] = {"ms_per_pass": {str(W): round(row[W], 4) for W in row},
                          "speedup": {str(W): round(row[1] / row[W], 3) for W in (2, 4, 8)}}
    out["method"] = ("T(B) / T(B/W) on one B200, CUDA events, median of 5 passes after 2 warm-ups; the W-GPU "
                     "run executes exactly the B/W share per GPU")
    return out


def extra_configs(torch, lbg, R, peak):
    out = {}
    for cfg in (0, 2, 3, 4):
        d, B, S = CONFIGS[cfg]
        try:
            # median of 5 passes: the shared box throws occasional 2-3x passes
            if cfg == 4:
                case = SweepCase(torch, lbg, R.dev, 0, B, B)
                total, per, launches = R.time_passes(case.run, 5, 1)
            else:
                _, _, pt, xt, work = R.shared_p_setup(cfg, 0, B)
                total, per, launches = R.time_passes(
                    lambda: lbg.evolve_batch_dev(pt, xt, S, work=work, stream=R.stream), 5, 1)
            ms = float(np.median(per))
            rate = B * S / (ms * 1e-3)
            tf = rate * flops_per_traj_step(d) / 1e12
            entry = {"value": rate, "unit": "traj-steps/s", "ms_per_pass": ms, "gflops": tf * 1e3,
                     "kernel": KERNEL[cfg], "gpu_launches_per_pass": launches // len(per)}
            if cfg == 0:
                entry["ns_per_step"] = ms * 1e6 / S
                entry["bound"] = ("latency: one dependent chain; per step >= 6 dependent FP64 ops x 23 cycles "
                                  "+ a shared-memory round trip (profiles/r01_latency_probe.json)")
            else:
                entry["roofline"] = {"bound": "fp64", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                                     "frac": tf / peak}
            if cfg == 4:
                # the real form executes 2 d^4 flops per traj-step (+ the build), so
                # the reference-form 8 d^4 count would put frac above 1: the
                # roofline is the EXECUTED rate over the whole pass
                # K4-S issues 5,960 DMMA.8x8x4 per trajectory (five column-grouped sparse
                # products A^k A at 792 each + one dense 81 x 81 product at 2,000; 512 flop
                # each, zeros inside the tiles included) plus ~0.03 M flop of DFMA fringe;
                # the dense s = 3 build issued 5 x 2 x 81^3
                build_flops = B * (K4S_DMMAS * 512 + 2 * 81 * 161 + 2 * 80 * 80)
                # K3-T steps the trace-reduced map: 80 x 80 FMAs per traj-step (+ 3 butterfly DADDs / lane)
                step_flops = 2 * 80 ** 2
                exec_tf = (build_flops + B * S * step_flops) / (ms * 1e-3) / 1e12
                entry["roofline"] = {"bound": "fp64", "achieved": exec_tf, "peak": peak, "unit": "TFLOP/s",
                                     "frac": exec_tf / peak,
                                     "counted": "issued FP64 work: build 5,960 DMMA.8x8x4 (512 flop each) + DFMA "
                                                "fringe per trajectory (sparse-generator build, K4-S) + steps "
                                                "2 x 80^2 per traj-step (K3-T, the trace-reduced map)",
                                     "reference_form_8d4_frac": tf / peak}
                case.args[-1] = 0  # the build (K5 + K4) apart -> a steps = 0 pass
                tb, pb, _ = R.time_passes(case.run, 5, 1)
                build_ms = float(np.median(pb))
                step_ms = max(ms - build_ms, 1e-9)
                entry["build_ms"] = build_ms
                entry["build_executed_tflops"] = build_flops / (build_ms * 1e-3) / 1e12
                entry["steps_ms"] = step_ms
                entry["steps_executed_tflops"] = B * S * step_flops / (step_ms * 1e-3) / 1e12
                case = SweepCase(torch, lbg, R.dev, 0, B, B, mode="complex")
                total, per, _ = R.time_passes(case.run, 2, 1)
                entry["complex_mode_ms_per_pass"] = float(np.median(per))
            entry["cpu_reference"] = cpu_reference_entry(cfg, rate)
            out[f"c{cfg}"] = entry
        except Exception as e:  # noqa: BLE001
            out[f"c{cfg}"] = {"error": str(e)}
    for cfg in (1, 2, 3):
        try:
            out[f"c{cfg}_density"] = density_entry(torch, lbg, R, cfg, peak)
        except Exception as e:  # noqa: BLE001
            out[f"c{cfg}_density"] = {"error": str(e)}
    out["grape"] = grape_table(lbg)
    try:
        out["propagator_build"] = expm_table(torch, lbg, R)
    except Exception as e:  # noqa: BLE001
        out["propagator_build"] = {"error": str(e)}
    return out


K4S_DMMAS = 5 * 792 + 2000  # per trajectory at config 4: 72 k-steps x (5 + 6 m-tiles) per sparse product
EXTRA_REF_SAMPLE = {0: 1, 2: 4096, 3: 256, 4: 2048}  # ~1 s of host work each


def cpu_reference_entry(cfg, gpu_rate):
    """The reference (lb::evolve native-fast SoA; c4 with make_model +
    build_lindbladian + expm per trajectory) on the box's host threads."""
    threads = os.cpu_count() or 1
    sample = EXTRA_REF_SAMPLE[cfg]
    try:
        value, times = cpu_reference_rate(cfg, sample, threads, reps=1, warmup=0)
    except Exception as e:  # noqa: BLE001
        return {"unavailable": str(e)}
    d, _, S = CONFIGS[cfg]
    return {"value": value, "cores": threads, "kind": "reference",
            "sample": f"{sample} trajectories x {S} steps, {times[0]:.2f} s", "gpu_over_cpu": gpu_rate / value}


def density_entry(torch, lbg, R, cfg, peak):
    """Opt-in density-matrix mode (lbg_evolve_density_dev): the same propagation
    on the real coordinates of rho, P_R = T P T^-1 (2 d^4 executed flops per
    traj-step instead of 8 d^4)."""
    d, B, S = CONFIGS[cfg]
    _, rho0, pt, _, _ = R.shared_p_setup(cfg, 0, B)
    xt = torch.from_numpy(rho0).to(R.dev)
    work = torch.empty(lbg.density_workspace(d * d, B), dtype=torch.uint8, device=R.dev)
    total, per, launches = R.time_passes(lambda: lbg.evolve_density_dev(pt, xt, S, work, stream=R.stream), 3, 1)
    ms = total / len(per)
    rate = B * S / (ms * 1e-3)
    executed = rate * 2 * d ** 4 / 1e12
    return {"value": rate, "ms_per_pass": ms, "gpu_launches_per_pass": launches // len(per),
            "roofline": {"executed_tflops": executed, "frac": executed / peak}}


def expm_table(torch, lbg, R):
    """the propagator build (K5 assembly + K4 expm) on device
    buffers vs the reference's lb::build_lindbladian + lb::expm (Pade-13) on one
    host core; batched state validation (K6) over the c1 batch."""
    rows = {}
    try:
        from oracle.bindings import Reference
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        ref = None
        rows["reference"] = f"unavailable: {e}"
    T, dev = torch, R.dev
    for cfg, d in ((1, 3), (2, 9), (3, 27)):
        h, ops = lbg.config_model(cfg)
        n = d * d
        hd = T.from_numpy(np.ascontiguousarray(h)).to(dev)
        od = T.from_numpy(np.ascontiguousarray(ops)).to(dev)
        Ld = T.empty((n, n), dtype=T.complex128, device=dev)
        Pd = T.empty((n, n), dtype=T.complex128, device=dev)
        wk = T.empty(lbg.lib().lbg_expm_workspace(n), dtype=T.uint8, device=dev)
        L = lbg.lib()

        def build():
            lbg._check(L.lbg_build_lindbladian_dev(d, lbg._tp(hd), ops.shape[0], lbg._tp(od), lbg._tp(Ld),
                                                   lbg._sp(R.stream)), "build")
            lbg._check(L.lbg_expm_dev(lbg._tp(Ld), n, 0.1, lbg._tp(Pd), lbg._tp(wk), lbg._sp(R.stream)), "expm")
        total, per, launches = R.time_passes(build, 5, 2)
        row = {"gpu_ms": total / len(per)}
        if ref is not None:
            t0 = time.perf_counter()
            ref.expm(ref.build_lindbladian(h, ops), 0.1)
            row["ref_ms"] = (time.perf_counter() - t0) * 1e3
            row["speedup"] = row["ref_ms"] / row["gpu_ms"]
        rows[f"d{d}"] = row
    d, B, _ = CONFIGS[1]
    rho = lbg.ginibre_batch(1, 0, B, d)
    xd = T.from_numpy(rho).to(dev)
    o3 = T.empty(3, dtype=T.float64, device=dev)
    total, per, _ = R.time_passes(lambda: lbg.check_state_batched_dev(xd, d, o3, stream=R.stream), 5, 2)
    rows["check_state"] = {"states": B, "gpu_ms": total / len(per)}
    return rows


def grape_table(lbg):
    """GRAPE piecewise-constant chain (Table IV shapes: d=3/100, d=9/50,
    d=27/20 segments x 32 steps) on cmd_grape's seeded inputs; the reference's
    lb::grape_chain timed beside it (single-threaded, as the reference is)."""
    rows = {}
    try:
        from oracle.bindings import Reference
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        return {"error": f"reference unavailable: {e}"}
    for d, seg in ((3, 100), (9, 50), (27, 20)):
        h0, hc, op, amps, dt, rho0 = ref.grape_inputs(d, seg)
        for _ in range(3):
            lbg.grape_chain(h0, hc, amps, 32, dt, op, rho0)
        runs = sorted((lbg.grape_chain(h0, hc, amps, 32, dt, op, rho0)[1] for _ in range(5)),
                      key=lambda t: t["build_ms"] + t["chain_ms"])
        t = runs[len(runs) // 2]
        row = {"gpu_points_per_s": t["points_per_s"], "gpu_build_ms": t["build_ms"], "gpu_chain_ms": t["chain_ms"]}
        if d < 27:
            _, b, c = ref.grape_chain(h0, hc, amps, 32, dt, op, rho0)
            row["ref_points_per_s"] = 1000.0 / (b + c)
        rows[f"d{d}"] = row
    return rows


def summary_text(line) -> str:
    """One short human line ahead of the JSON (keeps the per-config numbers in a
    truncated log tail)."""
    parts = [f"headline {line['value'] / 1e9:.2f} G traj-steps/s, {line['ms_per_step']:.2f} ms/pass, "
             f"frac {line['roofline']['frac']:.3f}, e2e {line['e2e']['value'] / 1e9:.2f} G"]
    if "pageable" in line["e2e"]:
        parts.append(f"e2e pageable {line['e2e']['pageable']['value'] / 1e9:.2f} G")
    cb = line.get("cpu_baseline", {})
    if cb.get("value"):
        parts.append(f"cpu {cb['value'] / 1e6:.0f} M ({line['value'] / cb['value']:.0f}x)")
    for k, e in line.get("configs", {}).items():
        if k in ("c0", "c2", "c3", "c4") and "ms_per_pass" in e:
            s = f"{k} {e['ms_per_pass']:.3f} ms"
            if "roofline" in e:
                s += f" frac {e['roofline']['frac']:.2f}"
            if "ns_per_step" in e:
                s += f" {e['ns_per_step']:.1f} ns/step"
            cr = e.get("cpu_reference", {})
            if cr.get("gpu_over_cpu"):
                s += f" {cr['gpu_over_cpu']:.1f}x cpu"
            parts.append(s)
    pj = line.get("strong_scaling_projection")
    if pj:
        parts.append("8-GPU projection " + " ".join(f"{k} {v['speedup']['8']:.2f}x"
                                                    for k, v in pj.items() if k.startswith("c")))
    return "bench summary: " + " | ".join(parts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the config's global batch split over the ranks (default); weak: B per rank")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs and the projection")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
