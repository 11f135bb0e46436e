"""c3 (d = 27) pass time at the global batch and the 8-GPU shares (measurement tooling; LBG_TILED_NO_EXACT_FIT=1 for the default tiles):
python tools/c3_shares.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, bench, paper_2603_18052_b200 as lbg
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
d, B, S = bench.CONFIGS[3]
for b in (B, 128, 100, 97):
    _, _, pt, xt, work = R.shared_p_setup(3, 0, b)
    _, per, _ = R.time_passes(lambda: lbg.evolve_batch_dev(pt, xt, S, work=work, stream=R.stream), 5, 2)
    print(b, "ms", round(float(np.median(per)), 3), flush=True)
