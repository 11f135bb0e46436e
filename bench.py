#!/usr/bin/env python
"""bench.py — B200 Lindblad propagation engine benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

Headline workload (BASELINE.json configs[1], "c1"): d = 3 transmon with
leakage, ONE shared P = exp(L dt) (9x9 complex128), 2^20 independent
trajectories per GPU, 1,000 propagation steps per pass. One bench "step" = one
pass of the hot path (vec(rho_b) <- P vec(rho_b), 1,000 times, for every
trajectory). metric = trajectory-steps/s (whole job), FP64 GFLOP/s counted as
8 d^4 = 648 flops per trajectory-step. Multi-GPU: trajectories shard with no
data-path collective (weak scaling: each rank owns 2^20 trajectories with
global ids rank*2^20 + b, so inputs are independent of N).

value: inputs resident in HBM (151 MB state > 126 MB L2, so no L2 flush is
needed), CUDA events on the launching stream, barrier + synchronize around
exactly K passes, max over ranks. e2e: the same metric through the host-buffer
C-ABI call lbg_evolve_shared_p (H2D of rho0 from pinned memory, rho0
validation, the steps, D2H of the final states) timed per call.
roofline: FP64 pipe bound; peak = FP64 DMMA/DFMA throughput measured live by
lbg_fp64_peak() (MEASURED_PEAKS.json has no FP64 figure). cpu_baseline: the
reference (oracle/_ref/libref.so, compiled from /root/reference sources with
its native-fast flags) on a bounded sample, all host threads.
Extra key "configs": the other BASELINE configs (c0 latency, c2 d=9, c3 d=27,
c4 per-trajectory sweep) measured the same way at N=1.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # cfg: (d, batch per GPU, steps)
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


# ---------------------------------------------------- GPU roofline placement ---
# B200 re-targeting of the reference's CPU model (proj/src/roofline.cpp:62-99:
# characterize -> place -> classify). Levels are where P lives while stepping;
# bandwidths are MEASURED (profiles/r01_fp64_peaks.json, MEASURED_PEAKS.json),
# capacities per the hardware (per-SM for the on-chip levels, since every SM
# needs its own copy of a shared P).
B200_PROFILE = {
    "levels": ["regs/const", "smem", "l2", "hbm"],
    "capacity_bytes": [None, 227 * 1024, 126 * 2 ** 20, 180 * 10 ** 9],
    "bw_gbs": [None, 36895.5, 15363.8, 6465.2],
}


def roofline_place(d: int, batch: int, shared_p: bool, peak_tflops: float, tile: int = 32) -> dict:
    """characterize (8 d^4 flops per trajectory-step; roofline.cpp:62-74), place P
    on the B200 ladder (roofline.cpp:76-87) and classify (roofline.cpp:93-99):
    bytes are what one step must pull from P's level for the whole batch."""
    n = d * d
    p_bytes = 16 * n * n
    flops = 8 * d ** 4 * batch
    prof = B200_PROFILE
    if shared_p:
        if d == 3:
            level, bytes_ = 0, 0  # 9x9 P in the constant bank / uniform registers
        elif p_bytes <= prof["capacity_bytes"][1]:
            # each SM re-reads P from SMEM once per step for its tile of trajectories
            sms = min(148, -(-batch // tile))
            level, bytes_ = 1, p_bytes * sms
        elif p_bytes <= prof["capacity_bytes"][2]:
            # GEMM tiles (tile x tile complex) stream P and the state from L2
            level, bytes_ = 2, flops / (8 * tile * tile / (16 * 2 * tile))
        else:
            level, bytes_ = 3, p_bytes + 32 * n * batch
    else:
        level, bytes_ = (0, 0) if n <= 81 else (3, (n * n * 16 + 32 * n) * batch)  # per-trajectory P
    ai = flops / bytes_ if bytes_ else float("inf")
    bw = prof["bw_gbs"][level]
    attainable = peak_tflops if bw is None else min(peak_tflops, ai * bw / 1e3)
    ridge = None if bw is None else peak_tflops * 1e3 / bw
    return {"level": prof["levels"][level], "flops_per_step": flops, "bytes_per_step": bytes_,
            "ai_flop_per_byte": ai, "ridge_flop_per_byte": ridge, "attainable_tflops": attainable,
            "bound": "compute" if (ridge is None or ai >= ridge) else "memory"}


def reference_model(lbg, mprof, d: int) -> dict:
    """The reference's own roofline (roofline.cpp:62-99: characterize -> place
    -> classify, per single matvec) evaluated on the measured B200 profile."""
    k = lbg.place(lbg.characterize(d), mprof)
    c = lbg.classify(k, mprof)
    return {"flops": k.flops, "bytes": k.bytes, "ai": k.ai, "placement": lbg.LEVELS[k.placement],
            "ridge": lbg.ridge_point(mprof, k.placement), **c}


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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Ginibre rho0, counter-based RNG seed 42)",
        "gflops": value * flops_per_traj_step(d) / 1e9,
        "config": {"workload": WORKLOAD[cfg], "d": d, "batch_per_gpu": B, "steps_per_pass": S,
                   "sample_trajectories_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "traj-steps/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample} trajectories x {S} steps per bench step through lb::evolve "
                                   f"(native-fast SoA), {threads} std::threads"},
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

    def shared_p_setup(self, cfg, B):
        d, _, S = CONFIGS[cfg]
        T = self.torch
        P = self.propagator(cfg)
        if cfg == 0:
            rho0 = np.zeros((1, 3, 3), complex)
            rho0[0, 0, 0] = 1.0
        else:
            rho0 = self.lbg.ginibre_batch(cfg, self.rank * B, B, d)
        pt = T.from_numpy(P).to(self.dev)
        xt = T.from_numpy(rho0.reshape(B, d * d)).to(self.dev)
        ws = self.lbg.evolve_workspace(d * d, B)
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
    d, B, S = CONFIGS[cfg]
    K, W = args.steps, args.warmup
    dmma_peak, dfma_peak = lbg.fp64_peak()
    peak = max(dmma_peak, dfma_peak)
    # the B200 ladder measured live (lbg_measure_machine_profile): SMEM, L2, HBM,
    # host-over-PCIe bandwidths feed the placement model below
    mprof = lbg.measure_machine_profile()
    bw = list(mprof.bandwidth_gbs)
    B200_PROFILE["bw_gbs"] = [None, bw[0], bw[1], bw[2]]
    B200_PROFILE["capacity_bytes"] = [None, int(mprof.capacity_bytes[0]), int(mprof.capacity_bytes[1]),
                                      int(mprof.capacity_bytes[2])]
    traffic = load_traffic()

    # ---- device-resident timed region -----------------------------------
    if cfg == 4:
        sweep = SweepCase(torch, lbg, dev, rank, B)
        fn = sweep.run
    else:
        P, rho0, pt, xt, work = R.shared_p_setup(cfg, B)
        fn = lambda: lbg.evolve_batch_dev(pt, xt, S, work=work, stream=R.stream)  # noqa: E731
    with Clocks(local) as clk:
        total_ms, per_ms, launches = R.time_passes(fn, K, W)
    total_ms = max_over_ranks(torch, total_ms)
    units = world * B * S * K
    value = units / (total_ms * 1e-3)
    ms_step = total_ms / K
    kernel_ms = float(np.mean(per_ms))
    achieved = flops_per_traj_step(d) * B * S / (kernel_ms * 1e-3) / 1e12

    # ---- end to end through the host-buffer C-ABI call ---------------------
    e2e = None
    if cfg != 4:
        pin = torch.empty(B * d * d * 2, dtype=torch.float64).pin_memory()
        host_in = pin.numpy().view(np.complex128).reshape(B, d, d)
        host_in[...] = rho0
        pin_out = torch.empty_like(pin).pin_memory()
        host_out = pin_out.numpy().view(np.complex128).reshape(B, d, d)
        import ctypes as C
        L = lbg.lib()
        dp = C.POINTER(C.c_double)
        Pc = np.ascontiguousarray(P)

        def call():
            rc = L.lbg_evolve_shared_p(Pc.ctypes.data_as(dp), d, host_in.ctypes.data_as(dp), B, S,
                                       host_out.ctypes.data_as(dp), 0)
            assert rc == 0, L.lbg_last_error()
        call()
        reps = 11  # median of 11: host-buffer calls on a shared box show occasional 2-3x outliers
        if torch.distributed.is_initialized():
            torch.distributed.barrier()
        calls = []
        with Clocks(local) as eclk:  # clocks during the host-buffer calls too
            for _ in range(reps):
                t0 = time.perf_counter()
                call()
                calls.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(torch, float(np.median(calls)))
        e2e = {"value": world * B * S / e2e_s, "unit": "traj-steps/s",
               "h2d_bytes_per_step": int(host_in.nbytes + Pc.nbytes), "d2h_bytes_per_step": int(host_out.nbytes),
               "ms_per_call": e2e_s * 1e3, "ms_per_call_all": [c * 1e3 for c in calls],
               "call": "lbg_evolve_shared_p (host buffers, synchronous); median of the calls",
               "clocks": eclk.summary()}
    else:
        e2e = sweep.e2e(reps=2)
        e2e["value"] = e2e["value"] * world

    line = {
        "metric": "trajectory-steps/s", "value": value, "unit": "traj-steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded Ginibre rho0 (counter-based RNG, seed 42), BASELINE config models",
        "gflops": value * flops_per_traj_step(d) / 1e9,
        "config": {"workload": WORKLOAD[cfg], "d": d, "batch_per_gpu": B, "global_batch": B * world,
                   "steps_per_pass": S, "parallelism": f"trajectories sharded over {world} GPU(s), no collective"
                   if cfg != 4 else f"trajectories sharded over {world} GPU(s), ensemble allreduce",
                   "l2": "state larger than L2; no flush needed" if cfg == 1 else "working set L2/SMEM resident"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic.get(KERNEL[cfg]),
                     "kernel": KERNEL[cfg],
                     "peak_source": f"measured live by lbg_fp64_peak(): DMMA {dmma_peak:.2f}, DFMA {dfma_peak:.2f} TF/s "
                                    "(MEASURED_PEAKS.json has no FP64 entry)",
                     "flops_per_launch": flops_per_traj_step(d) * B * S, "launch_ms": kernel_ms},
        "e2e": e2e,
        "placement": roofline_place(d, B, cfg != 4, peak),
        "machine_profile": dict(mprof.as_dict(), levels=["smem/SM", "l2", "hbm", "host(pcie)"],
                                source="lbg_measure_machine_profile (measured now); file format of "
                                       "lb::write_profile"),
        "reference_roofline": reference_model(lbg, mprof, d),
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        try:
            sample = REF_SAMPLE[cfg]
            cv, times = cpu_reference_rate(cfg, sample, threads, reps=1, warmup=0)
            line["cpu_baseline"] = {"value": cv, "unit": "traj-steps/s", "cores": threads, "kind": "reference",
                                    "sample": f"{sample} trajectories x {S} steps through lb::evolve "
                                              f"(native-fast SoA), {threads} std::threads, {times[0]:.2f} s"}
            # the reference's own methodology is single-core
            s1 = max(1, sample // 16)
            c1, t1 = cpu_reference_rate(cfg, s1, 1, reps=1, warmup=0)
            line["cpu_baseline"]["value_1core"] = c1
            line["cpu_baseline"]["sample_1core"] = f"{s1} trajectories x {S} steps, 1 thread, {t1[0]:.2f} s"
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "traj-steps/s", "cores": threads, "kind": "reference",
                                    "sample": f"unavailable: {e}"}

    if rank == 0 and world == 1 and not args.no_extra and args.config == 1:
        line["configs"] = extra_configs(torch, lbg, R, peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    return 0


class SweepCase:
    """Config 4 through lbg_evolve_sweep_dev (+ NCCL allreduce of the ensemble sum)."""

    def __init__(self, torch, lbg, dev, rank, B, mode="auto"):
        self.torch, self.lbg, self.dev, self.B, self.mode = torch, lbg, dev, B, mode
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        h0, hd, hs = lbg.config_sweep_terms()
        _, ops = lbg.config_model(4)
        delta, scale = lbg.sweep_params(rank * B, B)
        rho0 = np.zeros((9, 9), complex)
        rho0[0, 0] = 1.0
        self.host = (h0, hd, hs, ops, delta, scale, rho0)
        self.args = [T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(rho0), CONFIGS[4][2]]
        self.pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
        self.ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
        self.work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)

    def run(self):
        self.lbg.evolve_sweep_dev(*self.args, self.pops, self.ens, self.work, mode=self.mode)
        dist = self.torch.distributed
        if dist.is_initialized():  # the engine's only collective: ensemble sum
            if dist.get_backend() == "nccl":
                dist.all_reduce(self.ens)
            else:
                host = self.ens.cpu()
                dist.all_reduce(host)
                self.ens.copy_(host)

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


def extra_configs(torch, lbg, R, peak):
    out = {}
    for cfg in (0, 2, 3, 4):
        d, B, S = CONFIGS[cfg]
        try:
            if cfg == 4:
                case = SweepCase(torch, lbg, R.dev, 0, B)
                total, per, launches = R.time_passes(case.run, 3, 1)
            else:
                _, _, pt, xt, work = R.shared_p_setup(cfg, B)
                total, per, launches = R.time_passes(
                    lambda: lbg.evolve_batch_dev(pt, xt, S, work=work, stream=R.stream), 3 if cfg else 5, 1)
            ms = total / len(per)
            rate = B * S / (ms * 1e-3)
            tf = rate * flops_per_traj_step(d) / 1e12
            entry = {"workload": WORKLOAD[cfg], "value": rate, "unit": "traj-steps/s", "ms_per_pass": ms,
                     "gflops": tf * 1e3, "kernel": KERNEL[cfg], "gpu_launches_per_pass": launches // len(per)}
            if cfg == 0:
                entry["ns_per_step"] = ms * 1e6 / S
                entry["bound"] = ("latency: one dependent chain; per step >= 6 dependent FP64 ops x 23 cycles "
                                  "+ a shared-memory round trip (profiles/r01_latency_probe.json)")
            else:
                entry["roofline"] = {"bound": "fp64", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                                     "frac": tf / peak}
                entry["placement"] = roofline_place(d, B, cfg != 4, peak)
            if cfg == 4:
                entry["note"] = ("real transfer-matrix mode (L_R = T L T^-1, 4x fewer executed flops than "
                                 "8 d^4); includes per-trajectory GPU assembly + expm (not counted in flops)")
                # the real form executes 2 d^4 flops per traj-step (+ the build), so
                # the reference-form 8 d^4 count would put frac above 1: the
                # roofline is the EXECUTED rate over the whole pass
                build_flops = B * 5 * 2 * 81 ** 3  # Taylor-12 PS: 5 real 81 x 81 products
                exec_tf = (build_flops + B * S * 2 * 81 ** 2) / (ms * 1e-3) / 1e12
                entry["roofline"] = {"bound": "fp64", "achieved": exec_tf, "peak": peak, "unit": "TFLOP/s",
                                     "frac": exec_tf / peak,
                                     "counted": ("executed real-form flops: build 5 x 2 x 81^3 per trajectory + "
                                                 "steps 2 x 81^2 per traj-step"),
                                     "reference_form_8d4_tflops": tf,
                                     "reference_form_8d4_frac": tf / peak}
                # report the build (K5 + K4) separately -> a steps=0 pass
                case.args[-1] = 0
                tb, pb, _ = R.time_passes(case.run, 3, 1)
                build_ms = tb / len(pb)
                step_ms = max(ms - build_ms, 1e-9)
                step_rate = B * S / (step_ms * 1e-3)
                smem_bw = B200_PROFILE["bw_gbs"][1]
                entry["build"] = {
                    "ms": build_ms, "kernels": "ptm_expm_kernel (+ ptm_terms_kernel, once)",
                    "executed_tflops": build_flops / (build_ms * 1e-3) / 1e12,
                    "note": ("per trajectory: A = dt L_R from three precomputed affine terms, Taylor-12 "
                             "Paterson-Stockmeyer, 5 real 81x81 matmuls (10x10 DMMA tiles on k < 80 + DFMA "
                             "fringe for row / column 80, 8 warps in 5x3 / 5x2 blocks)")}
                entry["stepping"] = {
                    "ms": step_ms, "traj_steps_per_s": step_rate, "kernel": "ptm_step_kernel",
                    "executed_tflops": step_rate * 2 * 81 ** 2 / 1e12,
                    "paper_bytes_per_s": step_rate * 107568,
                    "note": ("SURVEY 8(d) accounting: 16 (d^4 + 2 d^2) = 107,568 B per traj-step at the level P "
                             "is served from; P_R is register-resident (52 KB real per trajectory), so the "
                             f"SMEM bound ({smem_bw:.0f} GB/s x AI 0.488) does not apply"),
                    "smem_roofline_traj_steps_per_s": smem_bw * 1e9 / 107568}
                case = SweepCase(torch, lbg, R.dev, 0, B, mode="complex")
                total, per, _ = R.time_passes(case.run, 2, 1)
                msc = total / len(per)
                entry["complex_mode"] = {"value": B * S / (msc * 1e-3), "ms_per_pass": msc,
                                         "note": "reference-form complex d^2 x d^2 matrices (k_sweep.cu)"}
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


EXTRA_REF_SAMPLE = {0: 1, 2: 4096, 3: 128, 4: 512}


def cpu_reference_entry(cfg, gpu_rate):
    """The reference (lb::evolve native-fast SoA; c4 with make_model +
    build_lindbladian + expm per trajectory) on the box's host threads, beside
    each extra config; c4 also reports build and steps apart."""
    threads = os.cpu_count() or 1
    sample = EXTRA_REF_SAMPLE[cfg]
    try:
        value, times = cpu_reference_rate(cfg, sample, threads, reps=1, warmup=0)
    except Exception as e:  # noqa: BLE001
        return {"unavailable": str(e)}
    d, _, S = CONFIGS[cfg]
    out = {"value": value, "unit": "traj-steps/s", "cores": threads, "kind": "reference",
           "sample": f"{sample} trajectories x {S} steps, {threads} std::threads, {times[0]:.2f} s",
           "gpu_over_cpu": gpu_rate / value}
    if cfg == 4:
        from oracle.bindings import Oracle, Reference
        o, r = Oracle(), Reference()
        dl = np.array([o.sweep_params(42, b)[0] for b in range(sample)])
        sc = np.array([o.sweep_params(42, b)[1] for b in range(sample)])
        _, _, build_s = r.sweep_batch(dl, sc, steps=0, threads=threads)
        out["build_s"], out["steps_s"] = build_s, max(times[0] - build_s, 0.0)
    return out


def density_entry(torch, lbg, R, cfg, peak):
    """Opt-in density-matrix mode (lbg_evolve_density_dev): the same propagation
    on the real coordinates of rho, P_R = T P T^-1 (2 d^4 executed flops per
    traj-step instead of 8 d^4). Reported beside the complex headline."""
    d, B, S = CONFIGS[cfg]
    _, rho0, pt, _, _ = R.shared_p_setup(cfg, B)
    xt = torch.from_numpy(rho0).to(R.dev)
    work = torch.empty(lbg.density_workspace(d * d, B), dtype=torch.uint8, device=R.dev)
    total, per, launches = R.time_passes(lambda: lbg.evolve_density_dev(pt, xt, S, work, stream=R.stream), 3, 1)
    ms = total / len(per)
    rate = B * S / (ms * 1e-3)
    executed = rate * 2 * d ** 4 / 1e12
    # end to end through the host-buffer call lbg_evolve_density (pinned buffers)
    import ctypes as C
    pin = torch.empty(B * d * d * 2, dtype=torch.float64).pin_memory()
    pin_out = torch.empty_like(pin).pin_memory()
    host_in = pin.numpy().view(np.complex128).reshape(B, d, d)
    host_out = pin_out.numpy().view(np.complex128).reshape(B, d, d)
    host_in[...] = rho0
    Pc = np.ascontiguousarray(R.propagator(cfg))
    dp = C.POINTER(C.c_double)
    L = lbg.lib()

    def call():
        rc = L.lbg_evolve_density(Pc.ctypes.data_as(dp), d, host_in.ctypes.data_as(dp), B, S,
                                  host_out.ctypes.data_as(dp))
        assert rc == 0, L.lbg_last_error()
    call()
    calls = []
    for _ in range(9):
        t0 = time.perf_counter()
        call()
        calls.append(time.perf_counter() - t0)
    e2e_s = float(np.median(calls))
    return {"workload": WORKLOAD[cfg] + " (density-matrix mode)", "value": rate, "unit": "traj-steps/s",
            "e2e": {"value": B * S / e2e_s, "unit": "traj-steps/s", "ms_per_call": e2e_s * 1e3,
                    "h2d_bytes_per_step": int(host_in.nbytes + Pc.nbytes), "d2h_bytes_per_step": int(host_out.nbytes),
                    "call": "lbg_evolve_density (host buffers, synchronous); median of 9"},
            "ms_per_pass": ms, "gpu_launches_per_pass": launches // len(per),
            "kernel": ("dfma9r_kernel" if d * d == 9 else
                       "tiled_evolve_kernel<real>" if d * d > 84 else "smem_real_kernel"),
            "roofline": {"bound": "fp64", "executed_tflops": executed, "peak": peak, "unit": "TFLOP/s",
                         "frac": executed / peak},
            "note": "real coordinates of the Hermitian rho (2 d^4 flops per traj-step); the headline "
                    "keeps the reference's complex 8 d^4 arithmetic"}


def expm_table(torch, lbg, R):
    """the propagator build (K5 assembly + K4 expm) on device
    buffers, CUDA events, vs the reference's lb::build_lindbladian + lb::expm
    (Pade-13) on one host core; and batched state validation (K6) over the c1
    batch vs lb::check_state on a host sample."""
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
        row = {"gpu_ms": total / len(per), "gpu_launches": launches // len(per)}
        if ref is not None:
            t0 = time.perf_counter()
            ref.expm(ref.build_lindbladian(h, ops), 0.1)
            row["ref_ms"] = (time.perf_counter() - t0) * 1e3
            row["speedup"] = row["ref_ms"] / row["gpu_ms"]
        rows[f"d{d}"] = row
    # K6: check_state over the whole c1 batch
    d, B, _ = CONFIGS[1]
    rho = lbg.ginibre_batch(1, 0, B, d)
    xd = T.from_numpy(rho).to(dev)
    o3 = T.empty(3, dtype=T.float64, device=dev)
    total, per, _ = R.time_passes(lambda: lbg.check_state_batched_dev(xd, d, o3, stream=R.stream), 5, 2)
    val = {"states": B, "gpu_ms": total / len(per), "states_per_s": B / (total / len(per) * 1e-3)}
    if ref is not None:
        sample = 65536
        t0 = time.perf_counter()
        for b in range(sample):
            ref.check_state(rho[b])
        dt = time.perf_counter() - t0
        val["ref_states_per_s_sample"] = sample / dt
        val["ref_note"] = f"lb::check_state on {sample} states through ctypes (one call per state)"
    rows["check_state"] = val
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
        for _ in range(3):  # warm-up (clocks, caches, one-time attributes)
            lbg.grape_chain(h0, hc, amps, 32, dt, op, rho0)
        runs = sorted((lbg.grape_chain(h0, hc, amps, 32, dt, op, rho0)[1] for _ in range(5)),
                      key=lambda t: t["build_ms"] + t["chain_ms"])
        t = runs[len(runs) // 2]  # median call
        row = {"segments": seg, "steps_per_segment": 32, "gpu_build_ms": t["build_ms"],
               "gpu_chain_ms": t["chain_ms"], "gpu_points_per_s": t["points_per_s"]}
        if d < 27:
            _, b, c = ref.grape_chain(h0, hc, amps, 32, dt, op, rho0)
            row.update(ref_build_ms=b, ref_chain_ms=c, ref_points_per_s=1000.0 / (b + c))
        rows[f"d{d}"] = row
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
