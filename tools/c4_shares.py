"""Time config 4 (65,536 per-trajectory propagators x 500 steps) at its global
batch and per-rank shares (measurement tooling): python tools/c4_shares.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
_, B, S = bench.CONFIGS[4]
row = {}
for W in (1, 2, 4, 8):
    case = bench.SweepCase(torch, lbg, dev, 0, B // W, B // W)
    _, per, _ = R.time_passes(case.run, 7, 2)
    row[W] = float(np.median(per))
print(" | ".join(f"{B // W}: {row[W]:.3f} ms" for W in row), "| 8x:", round(row[1] / row[8], 3))
