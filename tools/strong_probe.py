"""Strong-scaling projection on ONE GPU: time each batched config at its global
batch B and at the per-rank share B/W (W = 2, 4, 8); stepping has no inter-GPU
traffic, so T(B)/T(B/W) is the projected W-GPU speed-up."""
import json
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_18052_b200 as lbg
import bench

algo = sys.argv[1] if len(sys.argv) > 1 else "auto"
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
out = {}
for cfg in (1, 2, 3, 4):
    d, B, S = bench.CONFIGS[cfg]
    row = {}
    for W in (1, 2, 4, 8):
        b = B // W
        if cfg == 4:
            case = bench.SweepCase(torch, lbg, dev, 0, b, b)
            tot, per, _ = R.time_passes(case.run, 3, 1)
        else:
            _, _, pt, xt, work = R.shared_p_setup(cfg, 0, b)
            tot, per, _ = R.time_passes(lambda: lbg.evolve_batch_dev(pt, xt, S, algo=algo, work=work,
                                                                     stream=R.stream), 3, 1)
        row[W] = tot / len(per)
    row["speedup"] = {W: row[1] / row[W] for W in (2, 4, 8)}
    out[f"c{cfg}"] = row
    print(cfg, json.dumps(row), flush=True)
print(json.dumps(out))
