"""A/B one c4 stepping variant (LBG_PTM_STEP env): time passes, save outputs.
python tools/ab_c4.py OUT.npz [PASSES]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

out = sys.argv[1]
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
_, B, S = bench.CONFIGS[4]
case = bench.SweepCase(torch, lbg, dev, 0, B, B)
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
np.savez(out, pops=case.pops.cpu().numpy(), ens=case.ens.cpu().numpy())
print(f"variant={os.environ.get('LBG_PTM_EXPM', 'default')} c4 ms/pass median {sorted(ms)[len(ms) // 2]:.3f} all {['%.2f' % m for m in ms]}")
