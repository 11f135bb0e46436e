"""A/B the c4 build: sparse s = 6 (default) vs dense s = 3 (LBG_PTM_DENSE=1).
Times full c4 passes and build-only (steps = 0) passes for each mode and
compares populations / ensemble sums between the modes.
python tools/ab_build.py [PASSES]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

passes = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
_, B, S = bench.CONFIGS[4]


def timed(case, n):
    for _ in range(2):
        case.run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        case.run()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return sorted(ms)[len(ms) // 2]


res = {}
for mode in ("dense", "sparse"):
    if mode == "dense":
        os.environ["LBG_PTM_DENSE"] = "1"
    else:
        os.environ.pop("LBG_PTM_DENSE", None)
    case = bench.SweepCase(torch, lbg, dev, 0, B, B)
    full = timed(case, passes)
    pops, ens = case.pops.cpu().numpy().copy(), case.ens.cpu().numpy().copy()
    case.args[-1] = 0
    build = timed(case, passes)
    res[mode] = (full, build, pops, ens)
    print(f"{mode}: c4 pass {full:.3f} ms, build-only pass {build:.3f} ms", flush=True)
dp = float(np.abs(res["dense"][2] - res["sparse"][2]).max())
de = float(np.abs(res["dense"][3] - res["sparse"][3]).max() / B)
print(f"max |dpops| {dp:.3e}, max |dens|/B {de:.3e}")
