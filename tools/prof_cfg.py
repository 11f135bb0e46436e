"""Run one config's hot path a few times (for ncu captures):
python tools/prof_cfg.py CFG [PASSES] [density]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

cfg = int(sys.argv[1])
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
d, B, S = bench.CONFIGS[cfg]
if cfg == 4:
    case = bench.SweepCase(torch, lbg, dev, 0, B, B)
    fn = case.run
elif len(sys.argv) > 3 and sys.argv[3] == "density":
    _, rho0, pt, _, _ = R.shared_p_setup(cfg, 0, B)
    xt = torch.from_numpy(rho0).to(dev)
    work = torch.empty(lbg.density_workspace(d * d, B), dtype=torch.uint8, device=dev)

    def fn():
        lbg.evolve_density_dev(pt, xt, S, work)
else:
    _, _, pt, xt, work = R.shared_p_setup(cfg, 0, B)

    def fn():
        lbg.evolve_batch_dev(pt, xt, S, work=work)
for _ in range(passes):
    fn()
torch.cuda.synchronize()
print("ok", cfg)
