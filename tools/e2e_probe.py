"""Break down the end-to-end host-buffer call (lbg_evolve_shared_p) for config 1:
per-call wall times, and the raw pinned H2D / D2H bandwidth of the same bytes.
Usage (GPU box): python tools/e2e_probe.py [cfg]"""
import ctypes as C
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_18052_b200 as lbg  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d, B, S = CONFIGS[cfg]
h, ops = lbg.config_model(cfg)
P = np.ascontiguousarray(lbg.expm(lbg.build_lindbladian(h, ops), 0.1))
rho0 = lbg.ginibre_batch(cfg, 0, B, d)
pin = torch.empty(B * d * d * 2, dtype=torch.float64).pin_memory()
pin_out = torch.empty_like(pin).pin_memory()
host_in = pin.numpy().view(np.complex128).reshape(B, d, d)
host_out = pin_out.numpy().view(np.complex128).reshape(B, d, d)
host_in[...] = rho0
L = lbg.lib()
dp = C.POINTER(C.c_double)
out = {"cfg": cfg, "bytes": host_in.nbytes, "is_pinned": bool(pin.is_pinned())}


def call():
    rc = L.lbg_evolve_shared_p(P.ctypes.data_as(dp), d, host_in.ctypes.data_as(dp), B, S,
                               host_out.ctypes.data_as(dp), 0)
    assert rc == 0, L.lbg_last_error()


times = []
for _ in range(8):
    t0 = time.perf_counter()
    call()
    times.append((time.perf_counter() - t0) * 1e3)
out["call_ms"] = times
dev = torch.empty(B * d * d * 2, dtype=torch.float64, device="cuda")
h2d, d2h = [], []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    h2d.append(host_in.nbytes / (time.perf_counter() - t0) / 1e9)
    t0 = time.perf_counter()
    pin_out.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    d2h.append(host_in.nbytes / (time.perf_counter() - t0) / 1e9)
out["h2d_GBps"] = h2d
out["d2h_GBps"] = d2h
print(json.dumps(out))
