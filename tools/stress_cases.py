"""Small-shape runs of every kernel family (the barrier / DSMEM / TMA-ring /
split-K machinery exercised as at full size), each checked against a plain
torch fp64 reference or the invariants:

    python tools/stress_cases.py [names]

Written for compute-sanitizer (racecheck / synccheck); this GPU pool refuses
compute-sanitizer (profiles/r02_sanitizer.txt), so tests/test_gpu_races.py
runs the same shapes repeatedly and demands bitwise-identical results."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_18052_b200 as lbg  # noqa: E402

dev = torch.device("cuda", 0)


def rand_p(n, seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(n, n, dtype=torch.complex128, generator=g) / (2 * n)).to(dev)


def shared_case(n, B, steps, algo, seed=0):
    P = rand_p(n, seed)
    g = torch.Generator().manual_seed(seed + 1)
    x0 = torch.randn(B, n, dtype=torch.complex128, generator=g).to(dev)
    x = x0.clone()
    ws = torch.empty(max(lbg.evolve_workspace(n, B, algo), 1), dtype=torch.uint8, device=dev)
    lbg.evolve_batch_dev(P, x, steps, algo=algo, work=ws)
    want = x0
    for _ in range(steps):
        want = want @ P.T
    torch.cuda.synchronize()
    err = ((x - want).abs().max() / want.abs().max()).item()
    assert err < 1e-12, (n, B, algo, err)


def density_case(cfg, B, steps):
    d = lbg.config_dims(cfg)[0]
    h, ops = lbg.config_model(cfg)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(cfg, 0, B, d)
    want = lbg.evolve_batch(P, rho0, steps)
    got = lbg.evolve_batch(P, rho0, steps, algo="density")
    assert np.abs(got - want).max() < 1e-12


def sweep_case(B, steps, mode):
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(0, B)
    r0 = np.zeros((9, 9), complex)
    r0[0, 0] = 1.0
    pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(r0), steps, pops, ens, work,
                         mode=mode)
    torch.cuda.synchronize()
    assert abs(pops.sum().item() - B) < 1e-9


def pipeline_case(B, steps):
    """lbg_evolve_shared_p with >= 10 chunks (two compute streams, dfma9 constant
    slots reused across chunks), pageable buffers (host staging pool)."""
    h, ops = lbg.config_model(1)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(1, 0, B, 3)
    out = lbg.evolve_batch(P, rho0, steps)
    assert np.abs(np.trace(out, axis1=1, axis2=2) - 1).max() < 1e-12
    first = lbg.evolve_batch(P, rho0[:1000], steps)
    assert np.array_equal(first, out[:1000])


def grape_case(d, segments):
    from itertools import count  # noqa: F401
    h, ops = lbg.config_model(0 if d == 3 else 2 if d == 9 else 3)
    hc = np.zeros((d, d), complex)
    hc[0, 1] = hc[1, 0] = 0.02
    rho = np.zeros((d, d), complex)
    rho[0, 0] = 1.0
    got, _ = lbg.grape_chain(h, hc, np.linspace(-1, 1, segments), 4, 0.1, ops, rho)
    assert abs(np.trace(got) - 1) < 1e-12


CASES = {
    "dfma9": lambda: shared_case(9, 300, 4, "dfma9"),
    "chain": lambda: shared_case(9, 3, 6, "chain"),
    "smem": lambda: shared_case(81, 40, 3, "smem"),
    "cluster": lambda: shared_case(81, 120, 3, "cluster"),
    "ksplit": lambda: shared_case(81, 40, 3, "ksplit") or shared_case(81, 300, 3, "ksplit"),
    "cta": lambda: shared_case(81, 3, 3, "cta"),
    "rowsplit": lambda: shared_case(200, 2, 3, "rowsplit"),
    "tiled": lambda: shared_case(200, 40, 3, "tiled"),
    "tiled_multiway": lambda: shared_case(729, 64, 2, "tiled"),
    "density": lambda: density_case(1, 300, 3) or density_case(2, 40, 3) or density_case(3, 8, 2),
    "sweep_real": lambda: sweep_case(12, 5, "real"),
    "sweep_complex": lambda: sweep_case(4, 3, "complex"),
    "pipeline": lambda: pipeline_case(340000, 2),
    "grape": lambda: grape_case(3, 4) or grape_case(9, 3) or grape_case(27, 2),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        CASES[name]()
        print("ok", name, flush=True)
