"""c2 stepping time per pass at batches B (argv[1], comma list) for algo argv[2]."""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2603_18052_b200 as lbg
import bench
dev = torch.device("cuda", 0)
R = bench.Runner(torch, lbg, dev, 0)
algo = sys.argv[2] if len(sys.argv) > 2 else "auto"
res = {}
for B in [int(b) for b in sys.argv[1].split(",")]:
    _, _, pt, xt, work = R.shared_p_setup(2, 0, B)
    tot, per, _ = R.time_passes(lambda: lbg.evolve_batch_dev(pt, xt, 1000, algo=algo, work=work, stream=R.stream), 3, 1)
    res[B] = tot / len(per)
print(algo, json.dumps(res))
