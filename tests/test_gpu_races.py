"""Race / synchronisation stress for every kernel that synchronises across
warps, CTAs or clusters (mbarrier rings, DSMEM st.async exchanges, split-K
fixups, grid barriers, the multi-stream host pipeline). compute-sanitizer
racecheck / synccheck is closed on this GPU pool (profiles/r02_sanitizer.txt),
so the evidence is: each kernel runs the same input many times — with the
other kernels interleaved, so warps and CTAs are scheduled differently — and
every run must be bitwise identical and match a plain torch fp64 reference.
A missing barrier, a parity slip in an mbarrier phase or a split tile read
before its partial landed shows up as run-to-run differences. Anchor: the
reference's no-aliasing contract for the step kernels (propagate.cpp:14-28)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPS = 12


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


# (n, batch, steps, algo): small shapes of each synchronising kernel; the
# multi-way stream-K cases have fewer tiles than resident CTAs
SHAPES = [
    (81, 120, 7, "cluster"),      # K1b-C: DSMEM st.async + mbarrier per step parity
    (81, 40, 7, "ksplit"),        # K1b-K: K-split partials through DSMEM, G = 1
    (81, 1000, 5, "ksplit"),      # K1b-K, G = 2
    (81, 2100, 3, "ksplit"),      # K1b-K, G = 4, ragged last n-tile
    (200, 40, 5, "tiled"),        # K1c: TMA ring, 2-way stream-K, grid barrier
    (729, 64, 3, "tiled"),        # K1c: several-way stream-K (HEAD + MIDDLE + TAIL)
    (729, 100, 2, "tiled"),       # ragged columns, several-way
    (300, 2, 6, "rowsplit"),      # K2c: P rows over all SMs, grid barrier per step
    (81, 3, 9, "cta"),            # K2b
    (81, 2000, 4, "smem"),        # K1b, 2 n-tiles per CTA (12 warps, two m-tile counts)
    (81, 1000, 4, "smem"),        # K1b, 1 n-tile per CTA
]


def _run(lbg, torch, P, x0, steps, algo, ws):
    x = x0.clone()
    lbg.evolve_batch_dev(P, x, steps, algo=algo, work=ws)
    return x


def test_synchronising_kernels_bitwise_repeatable(lbg, torch):
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(11)
    cases = []
    for n, B, S, algo in SHAPES:
        P = (torch.randn(n, n, dtype=torch.complex128, generator=g) / (2 * n)).to(dev)
        x0 = torch.randn(B, n, dtype=torch.complex128, generator=g).to(dev)
        ws = torch.empty(max(lbg.evolve_workspace(n, B, algo), 1), dtype=torch.uint8, device=dev)
        want = x0
        for _ in range(S):
            want = want @ P.T
        cases.append((n, B, S, algo, P, x0, ws, want, []))
    for _ in range(REPS):  # interleaved: each case's runs see different neighbours
        for n, B, S, algo, P, x0, ws, want, outs in cases:
            outs.append(_run(lbg, torch, P, x0, S, algo, ws))
    torch.cuda.synchronize()
    for n, B, S, algo, P, x0, ws, want, outs in cases:
        first = outs[0]
        err = ((first - want).abs().max() / want.abs().max()).item()
        assert err <= 1e-12, (n, B, algo, err)
        for k, o in enumerate(outs[1:], 1):
            assert torch.equal(o, first), (n, B, algo, "run", k)


def test_density_and_grape_barriers_bitwise_repeatable(lbg, torch):
    """The real tile engine (density mode beyond n = 84), the real GRAPE chain
    (grid barrier per step) and the d = 9 PTM chain, repeated."""
    dev = torch.device("cuda")
    h, ops = lbg.config_model(3)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(3, 0, 64, 27)
    pt = torch.from_numpy(P).to(dev)
    outs = []
    for _ in range(6):
        x = torch.from_numpy(rho0.copy()).to(dev)
        work = torch.empty(lbg.density_workspace(729, 64), dtype=torch.uint8, device=dev)
        lbg.evolve_density_dev(pt, x, 5, work)
        outs.append(x.cpu().numpy())
    assert all(np.array_equal(o, outs[0]) for o in outs)
    want = lbg.evolve_batch(P, rho0, 5, algo="tiled")
    assert np.abs(outs[0] - want).max() <= 1e-12
    for d, cfg in ((9, 2), (27, 3)):
        h, ops = lbg.config_model(cfg)
        hc = np.zeros((d, d), complex)
        hc[0, 1] = hc[1, 0] = 0.02
        r = np.zeros((d, d), complex)
        r[0, 0] = 1.0
        runs = [lbg.grape_chain(h, hc, np.linspace(-1, 1, 5), 6, 0.1, ops, r)[0] for _ in range(5)]
        assert all(np.array_equal(x, runs[0]) for x in runs), d


def test_host_pipeline_slot_reuse_bitwise_repeatable(lbg, torch):
    """lbg_evolve_shared_p at 10 chunks (two compute streams, the dfma9
    constant-bank slots rotated across chunks, the high-priority check stream,
    pageable staging): repeated calls are bitwise identical to each other and
    to the single-stream device path."""
    h, ops = lbg.config_model(1)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    B, S = 400_000, 20
    rho0 = lbg.ginibre_batch(1, 0, B, 3)
    runs = [lbg.evolve_batch(P, rho0, S) for _ in range(4)]
    assert all(np.array_equal(r, runs[0]) for r in runs)
    dev = torch.device("cuda")
    x = torch.from_numpy(rho0.reshape(B, 9).copy()).to(dev)
    lbg.evolve_batch_dev(torch.from_numpy(P).to(dev), x, S, algo="dfma9")
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy().reshape(B, 3, 3), runs[0])
