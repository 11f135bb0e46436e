"""Small invocations of every kernel path (launch lists, quick regression checks):
    python tools/all_paths.py [all|shared|density|model|sweep|grape|bench]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_18052_b200 as lbg  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def shared_p(n, B, steps, algo):
    P = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / (2 * n)
    x = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    pt, xt = T(P), T(x)
    ws = lbg.evolve_workspace(n, B, algo)
    work = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
    lbg.evolve_batch_dev(pt, xt, steps, algo=algo, work=work)


if which in ("all", "shared"):
    for n, B, algo in ((9, 5, "chain"), (9, 300, "dfma9"), (81, 40, "smem"), (50, 3, "cta"),
                       (130, 2, "rowsplit"), (97, 40, "tiled"), (200, 70, "tiled")):
        shared_p(n, B, 3, algo)
if which in ("all", "density"):
    for d, B in ((3, 700), (9, 40), (5, 9)):
        P = np.eye(d * d, dtype=complex)
        x = rng.standard_normal((B, d, d)) + 1j * rng.standard_normal((B, d, d))
        xt = T(x)
        work = torch.empty(lbg.density_workspace(d * d, B), dtype=torch.uint8, device=dev)
        lbg.evolve_density_dev(T(P), xt, 3, work, mode="auto")
if which in ("all", "model"):
    for cfg in (0, 2, 3):
        h, ops = lbg.config_model(cfg)
        lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
if which in ("all", "sweep"):
    B = 8
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(0, B)
    r0 = np.zeros((9, 9), complex)
    r0[0, 0] = 1
    pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    for mode in ("real", "complex"):
        lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(r0), 5, pops, ens, work,
                             mode=mode)
if which in ("all", "grape"):
    for d in (3, 9):
        h = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        h = (h + h.conj().T) / 2
        hc = np.diag(np.arange(d)).astype(complex)
        op = np.diag(np.sqrt(np.arange(1, d)), 1).astype(complex) * 0.1
        rho = np.zeros((d, d), complex)
        rho[0, 0] = 1
        lbg.grape_chain(h, hc, [0.1, 0.2, 0.3], 4, 0.05, [op], rho)
if which in ("all", "bench"):
    lbg.run_bench(lbg.bench_config(3, "aos", 50, 2))
    lbg.run_bench(lbg.bench_config(27, "soa", 5, 1))
torch.cuda.synchronize()
print("paths ok", which)
