"""One c2-shaped pass (B = argv[1] trajectories, S = argv[2] steps, algo argv[3]) for profilers."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_18052_b200 as lbg
import bench
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
B, S = int(sys.argv[1]), int(sys.argv[2])
algo = sys.argv[3] if len(sys.argv) > 3 else "auto"
_, _, pt, xt, work = R.shared_p_setup(2, 0, B)
lbg.evolve_batch_dev(pt, xt, S, algo=algo, work=work, stream=R.stream)
torch.cuda.synchronize()
