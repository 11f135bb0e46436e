"""Run config 2 once at a given batch on a given algorithm (for ncu captures).
python tools/c2_one_share.py BATCH [ALGO] [STEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

b = int(sys.argv[1])
algo = sys.argv[2] if len(sys.argv) > 2 else "auto"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
_, _, pt, xt, work = R.shared_p_setup(2, 0, b)
lbg.evolve_batch_dev(pt, xt, steps, algo=algo, work=work, stream=R.stream)
torch.cuda.synchronize()
print("ok")
