"""Time lbg_evolve_shared_p at c1 from pinned host buffers (measurement only).
LBG_PIPELINE_TIMING=1 adds the per-chunk device timeline; argv[1] = calls."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_18052_b200 as lbg  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 4
h, ops = lbg.config_model(1)
P = np.ascontiguousarray(lbg.expm(lbg.build_lindbladian(h, ops), 0.1))
B = 1 << 20
rho0 = lbg.ginibre_batch(1, 0, B, 3)
pin = torch.empty(B * 18, dtype=torch.float64).pin_memory()
po = torch.empty_like(pin).pin_memory()
hin = pin.numpy().view(np.complex128).reshape(B, 3, 3)
hout = po.numpy().view(np.complex128).reshape(B, 3, 3)
hin[...] = rho0
L = lbg.lib()
dp = C.POINTER(C.c_double)
ms = []
for i in range(calls):
    t0 = time.perf_counter()
    rc = L.lbg_evolve_shared_p(P.ctypes.data_as(dp), 3, hin.ctypes.data_as(dp), B, 1000, hout.ctypes.data_as(dp), 0)
    ms.append((time.perf_counter() - t0) * 1e3)
    assert rc == 0
print("calls (ms):", " ".join(f"{m:.2f}" for m in ms), "median", f"{sorted(ms)[len(ms) // 2]:.2f}")
