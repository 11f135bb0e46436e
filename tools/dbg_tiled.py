"""Run the tiled stepper on one shape: python tools/dbg_tiled.py N BATCH STEPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_18052_b200 as lbg  # noqa: E402

n, B, S = (int(a) for a in sys.argv[1:4])
rng = np.random.default_rng(0)
P = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / n
x = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
dev = torch.device("cuda")
pt, xt = torch.from_numpy(P).to(dev), torch.from_numpy(x).to(dev)
ws = torch.empty(lbg.evolve_workspace(n, B, "tiled"), dtype=torch.uint8, device=dev)
lbg.evolve_batch_dev(pt, xt, S, algo="tiled", work=ws)
torch.cuda.synchronize()
want = x
for _ in range(S):
    want = want @ P.T
err = np.abs(xt.cpu().numpy() - want).max() / np.abs(want).max()
print(f"n={n} B={B} S={S} rel_err={err:.2e}", flush=True)
