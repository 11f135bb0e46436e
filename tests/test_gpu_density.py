"""GPU parity of the density-matrix mode (include/lbg.h lbg_evolve_density_dev):
the same shared-P propagation as lb::evolve (propagate.cpp:75-109), computed on
the real coordinates of rho with P_R = T P T^-1 (k_density.cu).

Same bar as the complex path (BASELINE.json north_star): max |rho_gpu -
rho_ref| <= 1e-10 against the reference's golden outputs and the oracle, trace
and Hermiticity <= 1e-12 on GPU outputs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_RHO = 1e-10
TOL_INV = 1e-12


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


def invariants(rho):
    tr = np.abs(np.trace(rho, axis1=-2, axis2=-1) - 1.0).max()
    herm = np.abs(rho - np.conj(np.swapaxes(rho, -1, -2))).max()
    return tr, herm


def run_density(lbg, torch, P, rho0, steps, mode="hermitian"):
    dev = torch.device("cuda")
    B, d = rho0.shape[0], rho0.shape[-1]
    pt = torch.from_numpy(np.ascontiguousarray(P)).to(dev)
    xt = torch.from_numpy(np.ascontiguousarray(rho0)).to(dev)
    work = torch.empty(max(lbg.density_workspace(d * d, B), 1), dtype=torch.uint8, device=dev)
    lbg.evolve_density_dev(pt, xt, steps, work, mode=mode)
    torch.cuda.synchronize()
    return xt.cpu().numpy()


@pytest.mark.parametrize("cfg", [0, 1, 2])
@pytest.mark.parametrize("mode", ["hermitian", "general", "auto"])
def test_density_vs_reference_goldens(lbg, golden, cfg, mode, torch):
    g, m = golden["evolve"], golden["models"]
    P = m[f"c{cfg}_P"]
    rho0, want, steps = g[f"c{cfg}_rho0"], g[f"c{cfg}_out"], int(g[f"c{cfg}_steps"])
    got = run_density(lbg, torch, P, rho0, steps, mode)
    assert np.abs(got - want).max() <= TOL_RHO
    tr, herm = invariants(got)
    assert tr <= TOL_INV and herm <= TOL_INV, (tr, herm)


@pytest.mark.parametrize("cfg,B,S", [(1, 1 << 20, 1000), (2, 4096, 1000)])
def test_density_full_size_vs_oracle(lbg, torch, oracle, cfg, B, S):
    d, _ = lbg.config_dims(cfg)
    h, ops = lbg.config_model(cfg)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(cfg, 0, B, d)
    out = run_density(lbg, torch, P, rho0, S)
    tr, herm = invariants(out)
    assert tr <= TOL_INV and herm <= TOL_INV, (tr, herm)
    rng = np.random.default_rng(cfg)
    for b in list(rng.integers(0, B, 24)) + [B - 1]:
        assert np.abs(out[b] - oracle.evolve(P, rho0[b], S)).max() <= TOL_RHO, b


@pytest.mark.parametrize("d,B", [(1, 5), (2, 33), (3, 130), (5, 70), (7, 31), (9, 1)])
def test_density_general_matrices_match_complex_path(lbg, torch, d, B):
    """Any Hermiticity-preserving P (P = sum_k c_k A_k (x) conj(A_k), c_k real:
    vec(A rho A^dag) in the row-major vec of lindblad.cpp:37-59) applied to any
    complex rho (not Hermitian, not unit trace): anti_hermitian=True is the same
    linear map as the complex kernels; ragged n and batch."""
    rng = np.random.default_rng(d * 100 + B)
    n = d * d
    P = np.zeros((n, n), np.complex128)
    for c in rng.standard_normal(4):
        A = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / (2 * d)
        P += c * np.kron(A, np.conj(A))
    x = rng.standard_normal((B, d, d)) + 1j * rng.standard_normal((B, d, d))
    want = x.reshape(B, n).T
    for _ in range(7):
        want = P @ want
    want = want.T.reshape(B, d, d)
    for mode in ("general", "auto"):
        got = run_density(lbg, torch, P, x, 7, mode)
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max()), mode


def test_density_zero_steps_and_empty(lbg, torch):
    """general / auto modes split rho = H + i H' (one rounding per entry)."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((9, 3, 3)) + 1j * rng.standard_normal((9, 3, 3))
    P = np.eye(9, dtype=np.complex128)
    for mode in ("general", "auto"):
        assert np.abs(run_density(lbg, torch, P, x, 0, mode) - x).max() <= 1e-15 * np.abs(x).max()
    h = x + np.conj(np.swapaxes(x, 1, 2))  # exactly Hermitian: the single-vector path is lossless
    assert np.array_equal(run_density(lbg, torch, P, h, 0), h)
    assert np.array_equal(run_density(lbg, torch, P, h, 3), h)  # identity P
    assert np.array_equal(run_density(lbg, torch, P, h, 3, "auto"), h)
    empty = np.zeros((0, 3, 3), np.complex128)
    assert run_density(lbg, torch, P, empty, 5).shape == (0, 3, 3)


def test_density_rejects_bad_mode(lbg, torch):
    dev = torch.device("cuda")
    work = torch.empty(lbg.density_workspace(9, 2), dtype=torch.uint8, device=dev)
    P9 = torch.eye(9, dtype=torch.complex128, device=dev)
    x3 = torch.zeros((2, 3, 3), dtype=torch.complex128, device=dev)
    with pytest.raises(ValueError):
        from paper_2603_18052_b200 import _check, _tp  # bad mode through the C-ABI
        _check(lbg.lib().lbg_evolve_density_dev(_tp(P9), 3, _tp(x3), 2, 1, 7, _tp(work), None), "mode")


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_density_host_api_vs_reference_goldens(lbg, golden, cfg):
    """lbg_evolve_density: host buffers, rho0 validation, chunked pipeline."""
    g, m = golden["evolve"], golden["models"]
    rho0, want, steps = g[f"c{cfg}_rho0"], g[f"c{cfg}_out"], int(g[f"c{cfg}_steps"])
    got = lbg.evolve_batch(m[f"c{cfg}_P"], rho0, steps, algo="density")
    assert np.abs(got - want).max() <= TOL_RHO
    bad = rho0.copy()
    bad[0, 0, 0] += 0.5  # trace error: propagate.cpp:79 rejects it
    with pytest.raises(ValueError):
        lbg.evolve_batch(m[f"c{cfg}_P"], bad, steps, algo="density")


def test_density_host_api_pipelined_full_size(lbg, oracle):
    """c1 at full size through the host API (8 chunks on 2 streams)."""
    B, S = 1 << 20, 1000
    h, ops = lbg.config_model(1)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(1, 0, B, 3)
    out = lbg.evolve_batch(P, rho0, S, algo="density")
    tr, herm = invariants(out)
    assert tr <= TOL_INV and herm <= TOL_INV
    for b in (0, 1, 131071, 131072, 524288, B - 1):  # chunk boundaries
        assert np.abs(out[b] - oracle.evolve(P, rho0[b], S)).max() <= TOL_RHO, b


@pytest.mark.parametrize("d,B", [(10, 7), (11, 40), (27, 6)])
def test_density_real_tile_engine_matches_complex(lbg, torch, oracle, d, B):
    """n > 84: the real-arithmetic K1c tile engine (odd n: even-stride copy of P_R)"""
    rng = np.random.default_rng(d)
    n = d * d
    if d == 27:
        h, ops = lbg.config_model(3)
        P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
        x = lbg.ginibre_batch(3, 0, B, d)
        steps = 20
    else:
        P = np.zeros((n, n), np.complex128)
        for c in rng.standard_normal(3):
            A = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / (2 * d)
            P += c * np.kron(A, np.conj(A))
        x = rng.standard_normal((B, d, d)) + 1j * rng.standard_normal((B, d, d))
        steps = 5
    want = lbg.evolve_batch(P, x, steps) if d == 27 else None
    if want is None:
        want = x.reshape(B, n).T
        for _ in range(steps):
            want = P @ want
        want = want.T.reshape(B, d, d)
    for mode in (("hermitian", "auto") if d == 27 else ("general", "auto")):
        got = run_density(lbg, torch, P, x, steps, mode)
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max()), mode
    if d == 27:
        assert np.abs(got[0] - oracle.evolve(P, x[0], steps)).max() <= TOL_RHO
