"""Median c4 pass time by CUDA events, populations / ensemble sum saved for an
A/B between builds: python tools/c4_time.py OUT.npz [PASSES]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

passes = int(sys.argv[2]) if len(sys.argv) > 2 else 9
_, B, S = bench.CONFIGS[4]
case = bench.SweepCase(torch, lbg, torch.device("cuda", 0), 0, B, B)
for _ in range(2):
    case.run()
torch.cuda.synchronize()
ms = []
for _ in range(passes):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    case.run()
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
print(lbg.__file__, "c4 pass median ms", round(sorted(ms)[len(ms) // 2], 3), "min", round(min(ms), 3))
np.savez(sys.argv[1], pops=case.pops.cpu().numpy(), ens=case.ens.cpu().numpy())
