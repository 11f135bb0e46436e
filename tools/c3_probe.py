"""c3 stepping time at batch B (argv[1], comma list) through the tiled engine;
argv[2] = steps per pass (default 200); prints ms/pass."""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2603_18052_b200 as lbg
import bench
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
S = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
res = {}
for B in [int(b) for b in sys.argv[1].split(",")]:
    _, _, pt, xt, work = R.shared_p_setup(3, 0, B)
    tot, per, _ = R.time_passes(lambda: lbg.evolve_batch_dev(pt, xt, S, algo="tiled", work=work, stream=R.stream),
                                reps, 1)
    res[B] = tot / len(per)
print(json.dumps(res))
