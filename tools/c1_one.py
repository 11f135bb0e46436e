"""One config-1 pass (for ncu captures): python tools/c1_one.py [B] [STEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

_, B0, S0 = bench.CONFIGS[1]
B = int(sys.argv[1]) if len(sys.argv) > 1 else B0
S = int(sys.argv[2]) if len(sys.argv) > 2 else S0
R = bench.Runner(torch, lbg, torch.device("cuda", 0), 0)
_, _, pt, xt, work = R.shared_p_setup(1, 0, B)
lbg.evolve_batch_dev(pt, xt, S, work=work, stream=R.stream)
torch.cuda.synchronize()
print("ok", B, S)
