"""c0 latency probe: one trajectory, d = 3, 10^4 steps on the chain kernel;
ns/step (median of 20 passes) and the final state (measurement tooling)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_18052_b200 as lbg  # noqa: E402

dev = torch.device("cuda", 0)
h, ops = lbg.config_model(0)
P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
rho0 = lbg.ginibre_batch(0, 0, 1, 3)
pt = torch.from_numpy(P).to(dev)
x0 = torch.from_numpy(rho0.reshape(1, 9).copy()).to(dev)
S = 10000
ms = []
for it in range(23):
    x = x0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lbg.evolve_batch_dev(pt, x, S, algo="chain")
    e1.record()
    torch.cuda.synchronize()
    if it >= 3:
        ms.append(e0.elapsed_time(e1))
ms.sort()
out = x.cpu().numpy()
ref = rho0.reshape(9)
for _ in range(S):
    ref = P @ ref
print(f"shfl={os.environ.get('LBG_CHAIN_SHFL') is not None} ns/step median {ms[len(ms) // 2] * 1e6 / S:.2f} "
      f"min {ms[0] * 1e6 / S:.2f}  max|d| vs numpy {np.abs(out.reshape(9) - ref).max():.2e}")
