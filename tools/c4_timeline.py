"""Kernel timeline of config-4 passes through torch.profiler (CUPTI activity, no
kernel serialisation): per-kernel time, idle gaps between kernels, and the pass
time by CUDA events (measurement tooling): python tools/c4_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_18052_b200 as lbg  # noqa: E402

dev = torch.device("cuda", 0)
_, B, S = bench.CONFIGS[4]
case = bench.SweepCase(torch, lbg, dev, 0, B, B)
for _ in range(2):
    case.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0.record()
    case.run()
    e1.record()
    torch.cuda.synchronize()
print("pass (events) ms", round(e0.elapsed_time(e1), 3))
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
tot, last_end, gaps = {}, None, 0.0
for e in evs:
    tot[e.name[:60]] = tot.get(e.name[:60], 0.0) + (e.time_range.end - e.time_range.start) / 1e3
    if last_end is not None and e.time_range.start > last_end:
        gap = (e.time_range.start - last_end) / 1e3
        gaps += gap
        if gap > 0.005:
            print(f"gap {gap:.3f} ms before {e.name[:50]}")
    last_end = max(last_end or 0, e.time_range.end)
span = (evs[-1].time_range.end - evs[0].time_range.start) / 1e3
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
    print(f"{v:9.3f} ms  {k}")
print(f"span {span:.3f} ms, idle gaps {gaps:.3f} ms, kernels/copies {len(evs)}")
