"""One config-4 sweep call (for ncu captures): python tools/c4_one.py [B] [STEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
S = int(sys.argv[2]) if len(sys.argv) > 2 else bench.CONFIGS[4][2]
case = bench.SweepCase(torch, lbg, torch.device("cuda", 0), 0, B, B)
case.args[-1] = S
case.run()
torch.cuda.synchronize()
print("ok", B, S)
