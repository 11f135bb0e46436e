"""Time config 2 (d = 9, 1,000 steps) at its per-rank shares 4,096 / 2,048 /
1,024 / 512 on a given algorithm (measurement tooling).
python tools/c2_shares.py [ALGO]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

algo = sys.argv[1] if len(sys.argv) > 1 else "auto"
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
d, B, S = bench.CONFIGS[2]
row = []
for W in (1, 2, 4, 8):
    _, _, pt, xt, work = R.shared_p_setup(2, 0, B // W)
    tot, per, _ = R.time_passes(lambda: lbg.evolve_batch_dev(pt, xt, S, algo=algo, work=work, stream=R.stream), 5, 2)
    row.append(f"{B // W}: {sorted(per)[len(per) // 2]:.3f} ms")
print(algo, " | ".join(row))
