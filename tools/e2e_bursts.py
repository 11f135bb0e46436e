"""e2e call times of lbg_evolve_shared_p with and without an nvidia-smi -lms 50 sampler
(measurement tooling): python tools/e2e_bursts.py"""
import os, sys, time, subprocess
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench, paper_2603_18052_b200 as lbg
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
cfg = 1
P, rho0, pt, xt, work = R.shared_p_setup(cfg, 0, bench.CONFIGS[1][1])
S = bench.CONFIGS[1][2]
import ctypes as C
B, d = rho0.shape[0], rho0.shape[1]
pin = torch.empty(B * d * d * 2, dtype=torch.float64).pin_memory()
pin_out = torch.empty_like(pin).pin_memory()
host_in = pin.numpy().view(np.complex128).reshape(B, d, d); host_in[...] = rho0
host_out = pin_out.numpy().view(np.complex128).reshape(B, d, d)
L = lbg.lib(); dp = C.POINTER(C.c_double); Pc = np.ascontiguousarray(P)
def call():
    assert L.lbg_evolve_shared_p(Pc.ctypes.data_as(dp), d, host_in.ctypes.data_as(dp), B, S, host_out.ctypes.data_as(dp), 0) == 0
for _ in range(3): call()
for smi in (False, True, False, True):
    proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "50"], stdout=subprocess.DEVNULL) if smi else None
    if smi: time.sleep(1.5)
    ts = []
    for _ in range(40):
        t0 = time.perf_counter(); call(); ts.append((time.perf_counter() - t0) * 1e3)
    if proc: proc.terminate(); proc.wait()
    ts = np.array(ts)
    print("smi" if smi else "no-smi", "median %.2f min %.2f max %.2f n>25ms %d" % (np.median(ts), ts.min(), ts.max(), (ts > 25).sum()), flush=True)
