"""GPU parity: every kernel path through the C-ABI (liblbg.so) against the
pinned CPU oracle (oracle/lbo.c) and the reference's golden vectors.

Tolerances (BASELINE.json north_star): max |rho_gpu - rho_cpu| <= 1e-10 after
the full step count; |Tr rho - 1| <= 1e-12 and max |rho - rho^dag| <= 1e-12 on
GPU outputs. The GPU propagator uses Taylor-16/Paterson-Stockmeyer instead of
the reference's Pade-13 (both accurate to unit roundoff), so P itself is
compared at 1e-13 relative; the generator L is compared bit for bit.
"""
import ctypes

import numpy as np
import pytest

C_SZ = ctypes.c_size_t

pytestmark = pytest.mark.gpu

TOL_RHO = 1e-10
TOL_INV = 1e-12
ALGOS_FOR = {  # which kernel paths can run a given n
    4: ("chain", "smem", "tiled", "cta", "rowsplit"),
    9: ("chain", "dfma9", "smem", "tiled", "cta", "rowsplit"),
    81: ("smem", "cluster", "ksplit", "tiled", "cta", "rowsplit"),
    729: ("tiled", "rowsplit"),
}


def algos(n, batch):
    """kernel paths applicable to (n, batch): rowsplit takes at most 4 trajectories"""
    return tuple(a for a in ALGOS_FOR[n] if a != "rowsplit" or batch <= 4)


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


def invariants(rho):
    tr = np.abs(np.trace(rho, axis1=-2, axis2=-1) - 1.0).max()
    herm = np.abs(rho - np.conj(np.swapaxes(rho, -1, -2))).max()
    return tr, herm


# ------------------------------------------------------------ assembly / P ---
def test_lindbladian_bitwise_vs_reference(lbg, golden, oracle):
    g = golden["models"]
    for cfg in range(3):
        L = lbg.build_lindbladian(g[f"c{cfg}_h"], g[f"c{cfg}_ops"])
        assert np.array_equal(L, g[f"c{cfg}_L"]), cfg
    h, ops = lbg.config_model(3)
    assert np.array_equal(lbg.build_lindbladian(h, ops), oracle.build_lindbladian(h, ops))
    k = golden["kat"]
    h2 = np.zeros((2, 2), complex)
    l2 = np.zeros((1, 2, 2), complex)
    l2[0, 0, 1] = np.sqrt(0.7)
    assert np.array_equal(lbg.build_lindbladian(h2, l2), k["ad_L"])


def test_non_hermitian_rejected(lbg):
    h = np.zeros((2, 2), complex)
    h[0, 1] = 1.0
    with pytest.raises(ValueError):
        lbg.build_lindbladian(h, np.zeros((0, 2, 2), complex))


def test_expm_vs_reference(lbg, golden):
    g, k = golden["models"], golden["kat"]
    for cfg in range(3):
        P = lbg.expm(g[f"c{cfg}_L"], 0.1)
        ref = g[f"c{cfg}_P"]
        assert np.abs(P - ref).max() <= 1e-13 * np.abs(ref).max(), cfg
        # trace preservation of the propagator: vec(I)^dag P = vec(I)^dag
        d = int(round(np.sqrt(P.shape[0])))
        idv = np.eye(d).reshape(-1)
        assert np.abs(idv @ P - idv).max() <= 1e-14
    for a, p in (("expm_a", "expm_p"), ("expm_big_a", "expm_big_p")):
        got = lbg.expm(k[a], 1.0)
        assert np.abs(got - k[p]).max() <= 1e-12 * np.abs(k[p]).max(), a
    assert np.abs(lbg.expm(np.zeros((3, 3)), 0.1) - np.eye(3)).max() == 0.0
    nil = np.zeros((2, 2), complex)
    nil[0, 1] = 1.0
    assert np.abs(lbg.expm(nil, 1.0) - np.array([[1, 1], [0, 1]])).max() <= 1e-15
    with pytest.raises(ValueError):
        lbg.expm(np.full((2, 2), np.nan), 1.0)


@pytest.mark.parametrize("n", [3, 16, 17, 40, 130])
def test_expm_properties(lbg, n):
    """test_expm.cpp:27-164 on every expm path (one-CTA n <= 16, tile GEMMs, the
    stream-K engine for n >= 128): diagonal, semigroup (1e-10), unitary (1e-11),
    and the scaling-and-squaring branch agreeing with direct evaluation."""
    rng = np.random.default_rng(n)
    dg = rng.normal(size=n) + 1j * rng.normal(size=n)
    got = lbg.expm(np.diag(dg), 0.7)
    want = np.diag(np.exp(dg * 0.7))
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
    a = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(n)
    s, t = 0.3, 0.45
    lhs = lbg.expm(a, s + t)
    rhs = lbg.expm(a, s) @ lbg.expm(a, t)
    assert np.abs(lhs - rhs).max() <= 1e-10 * np.abs(lhs).max()
    hm = (a + a.conj().T) / 2
    u = lbg.expm(-1j * hm, 2.0)
    assert np.abs(u @ u.conj().T - np.eye(n)).max() <= 1e-11
    big = lbg.expm(a, 9.0)  # ||a dt|| >> 0.79: several squarings
    half = lbg.expm(a, 4.5)
    assert np.abs(big - half @ half).max() <= 1e-10 * np.abs(big).max()


def test_expm_d27_vs_oracle(lbg, oracle):
    h, ops = lbg.config_model(3)
    L = lbg.build_lindbladian(h, ops)
    P = lbg.expm(L, 0.1)
    ref = oracle.expm(L, 0.1)
    assert np.abs(P - ref).max() <= 1e-13 * np.abs(ref).max()


# ----------------------------------------------------------- raw step shim ---
def test_step_shims_vs_oracle(lbg, oracle):
    rng = np.random.default_rng(11)
    for n in (1, 4, 9, 16, 81, 729):
        p = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        v = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        want = oracle.step_soa(p, v)
        scale = np.abs(want).max()
        assert np.abs(lbg.step_soa(p, v) - want).max() <= 1e-13 * scale
        assert np.abs(lbg.step_aos(p, v) - want).max() <= 1e-13 * scale
    v = rng.uniform(-1, 1, 9) + 1j * rng.uniform(-1, 1, 9)
    assert np.array_equal(lbg.step_soa(np.eye(9), v), v)  # identity bitwise
    assert lbg.step_aos(np.array([[2 + 1j]]), np.array([1 - 1j]))[0] == 3 - 1j


# ------------------------------------------------- golden config subsets ---
@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_config_subsets_vs_reference_goldens(lbg, golden, oracle, cfg):
    g, m = golden["evolve"], golden["models"]
    if cfg < 3:
        P = m[f"c{cfg}_P"]
    else:
        h, ops = lbg.config_model(3)
        P = oracle.expm(oracle.build_lindbladian(h, ops), 0.1)
    rho0, want, steps = g[f"c{cfg}_rho0"], g[f"c{cfg}_out"], int(g[f"c{cfg}_steps"])
    for algo in algos(P.shape[0], rho0.shape[0]):
        got = lbg.evolve_batch(P, rho0, steps, algo=algo)
        err = np.abs(got - want).max()
        assert err <= TOL_RHO, (algo, err)
        tr, herm = invariants(got)
        assert tr <= TOL_INV and herm <= TOL_INV, (algo, tr, herm)
    # the full product path: GPU-built P
    hh, oo = lbg.config_model(cfg)
    Pg = lbg.expm(lbg.build_lindbladian(hh, oo), 0.1)
    got = lbg.evolve_batch(Pg, rho0, steps)
    assert np.abs(got - want).max() <= TOL_RHO


def test_closed_form_damping_every_path(lbg):
    gamma, dt, n = 0.7, 0.004, 500
    h = np.zeros((2, 2), complex)
    l = np.zeros((1, 2, 2), complex)
    l[0, 0, 1] = np.sqrt(gamma)
    P = lbg.expm(lbg.build_lindbladian(h, l), dt)
    rho0 = np.zeros((2, 2), complex)
    rho0[1, 1] = 1.0
    want = np.exp(-gamma * n * dt)
    for algo in algos(4, 1):
        rho = lbg.evolve(P, rho0, n, algo=algo)
        assert abs(rho[1, 1].real - want) < 1e-10
        assert abs(rho[0, 0].real - (1 - want)) < 1e-10
        assert abs(rho[0, 1]) < 1e-12
        assert lbg.check_state(rho)["passed"]


def test_evolve_contract(lbg, golden):
    P = golden["models"]["c1_P"]
    rho0 = golden["evolve"]["c1_rho0"][:5]
    for algo in algos(9, 5):
        assert np.array_equal(lbg.evolve_batch(P, rho0, 0, algo=algo), rho0)  # zero steps
        direct = lbg.evolve_batch(P, rho0, 10, algo=algo)
        stacked = lbg.evolve_batch(P, lbg.evolve_batch(P, rho0, 4, algo=algo), 6, algo=algo)
        assert np.array_equal(direct, stacked), algo  # composes bitwise
    zero_gen = lbg.expm(np.zeros((9, 9)), 0.1)
    assert np.abs(lbg.evolve_batch(zero_gen, rho0, 1000) - rho0).max() < 1e-12
    with pytest.raises(ValueError):
        lbg.evolve(P, np.eye(3), 1)  # trace 3
    bad = np.diag([1.0, 0, 0]).astype(complex)
    bad[0, 1] = 0.5
    with pytest.raises(ValueError):
        lbg.evolve(P, bad, 1)  # not Hermitian
    with pytest.raises(ValueError):
        lbg.evolve(np.eye(4), np.diag([1.0, 0, 0]), 1)  # shape mismatch


# ------------------------------------------------------------- full sizes ---
def _full_run(lbg, torch, cfg, B, S, algo, check_idx, oracle, P=None):
    d, _ = lbg.config_dims(cfg)
    if P is None:
        h, ops = lbg.config_model(cfg)
        P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(cfg, 0, B, d)
    dev = torch.device("cuda")
    pt = torch.from_numpy(P).to(dev)
    xt = torch.from_numpy(rho0.reshape(B, d * d)).to(dev)
    ws = lbg.evolve_workspace(d * d, B, algo)
    work = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
    lbg.evolve_batch_dev(pt, xt, S, algo=algo, work=work)
    torch.cuda.synchronize()
    out = xt.cpu().numpy().reshape(B, d, d)
    tr, herm = invariants(out)
    assert tr <= TOL_INV and herm <= TOL_INV, (cfg, tr, herm)
    for b in check_idx:
        want = oracle.evolve(P, rho0[b], S)
        assert np.abs(out[b] - want).max() <= TOL_RHO, (cfg, b)
    return out


def test_config1_full_size(lbg, torch, oracle):
    rng = np.random.default_rng(0)
    _full_run(lbg, torch, 1, 1 << 20, 1000, "dfma9", rng.integers(0, 1 << 20, 64), oracle)


@pytest.mark.parametrize("algo", ["smem", "cluster", "ksplit"])
def test_config2_full_size(lbg, torch, oracle, algo):
    rng = np.random.default_rng(1)
    _full_run(lbg, torch, 2, 4096, 1000, algo, list(rng.integers(0, 4096, 24)) + [4095], oracle)


@pytest.mark.parametrize("algo", ["cluster", "ksplit"])
@pytest.mark.parametrize("B", [1, 7, 8, 9, 55, 56, 57, 64, 100, 512, 600, 1000, 1024, 2048, 2500, 5000])
def test_cluster_batch_shapes_vs_smem(lbg, torch, B, algo):
    """every cluster plan against the single-CTA kernel, both layouts: K1b-C
    (k = 1..7 n-tiles per 2-CTA cluster, split and unsplit, ragged last cluster)
    and K1b-K (K split over the 2-CTA cluster, G = 1..4 n-tiles per cluster,
    ragged last n-tile, more clusters than SM pairs)"""
    rng = np.random.default_rng(B)
    n = 81
    P = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / (2 * n)
    x = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    dev = torch.device("cuda")
    pt = torch.from_numpy(P).to(dev)
    outs = {}
    for a in ("smem", algo):
        xt = torch.from_numpy(x.copy()).to(dev)
        lbg.evolve_batch_dev(pt, xt, 9, algo=a)
        outs[a] = xt.cpu().numpy()
    assert np.abs(outs[algo] - outs["smem"]).max() <= 1e-13 * max(1.0, np.abs(outs["smem"]).max())
    xr = torch.from_numpy(np.ascontiguousarray(x.real)).to(dev)
    xi = torch.from_numpy(np.ascontiguousarray(x.imag)).to(dev)
    L = lbg.lib()
    lbg._check(L.lbg_evolve_shared_p_soa_dev(lbg._tp(pt), n, lbg._tp(xr), lbg._tp(xi), B, 9, lbg.ALGO[algo],
                                             None, None), "soa")
    got = xr.cpu().numpy() + 1j * xi.cpu().numpy()
    assert np.abs(got - outs["smem"]).max() <= 1e-13 * max(1.0, np.abs(outs["smem"]).max())


@pytest.mark.parametrize("B", [1, 8, 9, 100, 1000, 1024, 1184, 1185, 1200, 2000, 2048, 2368, 2400, 4096])
def test_smem_n_tiles_per_cta_vs_torch(lbg, torch, B):
    """K1b at n = 81 picks 4, 2 or 1 n-tiles per CTA from the batch (2 / 1 for
    the 2,048 / 1,024 shares of config 2): every choice, ragged last CTA, more
    CTAs than SMs, AoS and SoA, against a plain torch complex128 reference."""
    rng = np.random.default_rng(300 + B)
    n, S = 81, 9
    P = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / (2 * n)
    x = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    dev = torch.device("cuda")
    pt = torch.from_numpy(P).to(dev)
    want = torch.from_numpy(x).to(dev)
    for _ in range(S):
        want = want @ pt.T
    want = want.cpu().numpy()
    tol = 1e-13 * max(1.0, np.abs(want).max())
    xt = torch.from_numpy(x.copy()).to(dev)
    lbg.evolve_batch_dev(pt, xt, S, algo="smem")
    assert np.abs(xt.cpu().numpy() - want).max() <= tol
    xr = torch.from_numpy(np.ascontiguousarray(x.real)).to(dev)
    xi = torch.from_numpy(np.ascontiguousarray(x.imag)).to(dev)
    L = lbg.lib()
    lbg._check(L.lbg_evolve_shared_p_soa_dev(lbg._tp(pt), n, lbg._tp(xr), lbg._tp(xi), B, S, lbg.ALGO["smem"],
                                             None, None), "soa")
    assert np.abs(xr.cpu().numpy() + 1j * xi.cpu().numpy() - want).max() <= tol


def test_config3_full_size(lbg, torch, oracle):
    _full_run(lbg, torch, 3, 1024, 200, "tiled", [0, 517, 1023], oracle)


def test_tiled_is_linear_at_scale(lbg, torch):
    """size-independent property at a large, non-physical, ragged shape."""
    dev = torch.device("cuda")
    n, B = 200, 333
    g = torch.Generator(device="cpu").manual_seed(3)
    P = (torch.randn(n, n, dtype=torch.complex128, generator=g) / n).to(dev)
    x = torch.randn(B, n, dtype=torch.complex128, generator=g).to(dev)
    y = torch.randn(B, n, dtype=torch.complex128, generator=g).to(dev)
    a = 0.3 - 1.2j
    ws = torch.empty(lbg.evolve_workspace(n, B, "tiled"), dtype=torch.uint8, device=dev)
    z = a * x + y
    for t in (x, y, z):
        lbg.evolve_batch_dev(P, t, 7, algo="tiled", work=ws)
    torch.cuda.synchronize()
    assert (z - (a * x + y)).abs().max().item() <= 1e-12 * (a * x + y).abs().max().item()
    ref = x.clone()
    # against torch fp64 matmuls (a plain fp64 reference of the same op)
    x0 = torch.randn(B, n, dtype=torch.complex128, generator=g).to(dev)
    x1 = x0.clone()
    lbg.evolve_batch_dev(P, x1, 3, algo="tiled", work=ws)
    want = x0
    for _ in range(3):
        want = want @ P.T
    torch.cuda.synchronize()
    assert (x1 - want).abs().max().item() <= 1e-12 * want.abs().max().item()
    del ref


# ----------------------------------------------------------- config 4 sweep ---
@pytest.mark.parametrize("mode", ["complex", "real"])
def test_sweep_vs_reference_goldens(lbg, torch, golden, mode):
    s = golden["sweep"]
    dev = torch.device("cuda")
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    B = s["delta"].shape[0]
    rho0 = np.zeros((9, 9), complex)
    rho0[0, 0] = 1.0
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(s["delta"]), T(s["scale"]), 0.1, T(rho0),
                         int(s["steps"]), pops, ens, work, mode=mode)
    torch.cuda.synchronize()
    assert np.abs(pops.cpu().numpy() - s["pops"]).max() <= TOL_RHO
    assert np.abs(ens.cpu().numpy() - s["ens_sum"]).max() <= TOL_RHO * B
    e = ens.cpu().numpy() / B
    tr, herm = invariants(e)
    assert tr <= TOL_INV and herm <= TOL_INV


@pytest.mark.parametrize("mode", ["complex", "real"])
def test_sweep_full_size_invariants(lbg, torch, mode):
    _sweep_full(lbg, torch, mode)


def _sweep_full(lbg, torch, mode):
    dev = torch.device("cuda")
    B = 65536
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(0, B)
    rho0 = np.zeros((9, 9), complex)
    rho0[0, 0] = 1.0
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(rho0), 500, pops, ens, work,
                         mode=mode)
    torch.cuda.synchronize()
    p = pops.cpu().numpy()
    assert np.abs(p.sum(axis=1) - 1.0).max() <= TOL_INV
    assert p.min() >= -TOL_INV
    e = ens.cpu().numpy() / B
    tr, herm = invariants(e)
    assert tr <= TOL_INV and herm <= TOL_INV
    assert np.abs(np.diag(e).real - p.mean(axis=0)).max() <= 1e-12
    return p, e


def test_sweep_modes_agree_at_full_size(lbg, torch):
    """real transfer-matrix path == complex path within the parity tolerance."""
    pr, er = _sweep_full(lbg, torch, "real")
    pc, ec = _sweep_full(lbg, torch, "complex")
    assert np.abs(pr - pc).max() <= TOL_RHO
    assert np.abs(er - ec).max() <= TOL_RHO


@pytest.mark.parametrize("B", [1, 2, 4, 1100, 16385])
def test_sweep_ensemble_sum_ragged_batches(lbg, torch, B):
    """The real path's ensemble sum is combined per CTA of 3 trajectories before
    its atomics: batches that leave a partial CTA (B % 3 != 0) or a 1-trajectory
    last chunk (16,385) must still sum every trajectory exactly once — against
    the complex path (one CTA per trajectory) and the populations."""
    dev = torch.device("cuda")
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(0, B)
    rho0 = np.zeros((9, 9), complex)
    rho0[0, 0] = 1.0
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    out = {}
    for mode in ("real", "complex"):
        pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
        ens = torch.full((9, 9), float("nan"), dtype=torch.complex128, device=dev)
        lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(rho0), 60, pops, ens, work,
                             mode=mode)
        torch.cuda.synchronize()
        out[mode] = pops.cpu().numpy(), ens.cpu().numpy()
    (pr, er), (pc, ec) = out["real"], out["complex"]
    assert np.isfinite(er).all()
    assert np.abs(pr - pc).max() <= TOL_RHO
    assert np.abs(er - ec).max() <= TOL_RHO * B
    assert np.abs(np.diag(er).real - pr.sum(axis=0)).max() <= 1e-12 * B
    assert abs(np.trace(er).real - B) <= 1e-11 * B


@pytest.mark.parametrize("dt", [0.07, 0.12, 0.6])
def test_sweep_real_expm_branches(lbg, torch, dt):
    """k_ptm.cu expm branches: ||A||_1 ~ 0.23 / 0.41 / 2.0 take Taylor degree 12,
    degree 14, and degree 14 with two squarings; a ragged batch (not a multiple
    of the 3 trajectories per step CTA) and a full Hermitian rho0. The real
    path must agree with the reference-form complex path."""
    dev = torch.device("cuda")
    B, S = 301, 40
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(7, B)
    rng = np.random.default_rng(5)
    g = rng.normal(size=(9, 9)) + 1j * rng.normal(size=(9, 9))
    rho0 = g @ g.conj().T
    rho0 = rho0 / np.trace(rho0).real
    rho0 = 0.5 * (rho0 + rho0.conj().T)  # exactly Hermitian
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    out = {}
    for mode in ("real", "complex"):
        pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
        ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
        work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
        lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), dt, T(rho0), S, pops, ens, work,
                             mode=mode)
        torch.cuda.synchronize()
        out[mode] = (pops.cpu().numpy(), ens.cpu().numpy())
    assert np.abs(out["real"][0] - out["complex"][0]).max() <= TOL_RHO
    assert np.abs(out["real"][1] - out["complex"][1]).max() <= TOL_RHO * B
    tr, herm = invariants(out["real"][1] / B)
    assert tr <= TOL_INV and herm <= TOL_INV


def _sweep_real(lbg, torch, h0, hd, hs, ops, delta, scale, dt, rho0, S, dense_build):
    import os
    dev = torch.device("cuda")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    B = len(delta)
    pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    if dense_build:
        os.environ["LBG_PTM_DENSE"] = "1"
    try:
        lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), dt, T(rho0), S, pops, ens, work,
                             mode="real")
        torch.cuda.synchronize()
    finally:
        os.environ.pop("LBG_PTM_DENSE", None)
    return pops.cpu().numpy(), ens.cpu().numpy()


@pytest.mark.parametrize("dt", [0.1, 0.12, 0.6])
def test_sweep_sparse_build_matches_dense_build(lbg, torch, dt):
    """K4-S (sparse generator: five column-grouped DMMA products A^k A and one
    dense product, Paterson-Stockmeyer s = 6) against the dense s = 3 build:
    ||A||_1 ~ 0.33 (no squaring), 0.41 (one squaring in the sparse form, degree
    14 in the dense one) and 2.0 (squarings in both); ragged batch, Hermitian
    rho0 with every entry populated. The batch is past the plan threshold
    (1,024) and not a multiple of the 3 trajectories per step CTA."""
    B, S = 1100, 40
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(11, B)
    rng = np.random.default_rng(9)
    g = rng.normal(size=(9, 9)) + 1j * rng.normal(size=(9, 9))
    rho0 = g @ g.conj().T
    rho0 = 0.5 * (rho0 + rho0.conj().T) / np.trace(rho0).real
    ps, es = _sweep_real(lbg, torch, h0, hd, hs, ops, delta, scale, dt, rho0, S, False)
    pd, ed = _sweep_real(lbg, torch, h0, hd, hs, ops, delta, scale, dt, rho0, S, True)
    assert np.abs(ps - pd).max() <= 1e-12
    assert np.abs(es - ed).max() <= 1e-12 * B
    assert (ps != pd).any()  # different rounding: the sparse path did run


def test_sweep_sparse_build_edge_patterns(lbg, torch):
    """K4-S plans on patterns other than config 4's: (a) the zero generator (every
    column group empty, P = I: populations of rho0 unchanged — bitwise but for rho_88,
    which the step kernel recovers from the trace); (b) a
    random sparse Hamiltonian with a single collapse operator (ragged union
    sizes, groups with empty columns) against the dense build."""
    B, S = 1040, 30
    z = np.zeros((9, 9), complex)
    delta, scale = lbg.sweep_params(3, B)
    rng = np.random.default_rng(21)
    g = rng.normal(size=(9, 9)) + 1j * rng.normal(size=(9, 9))
    rho0 = g @ g.conj().T
    rho0 = 0.5 * (rho0 + rho0.conj().T) / np.trace(rho0).real
    pz, _ = _sweep_real(lbg, torch, z, z, z, np.zeros((1, 9, 9), complex), delta, scale, 0.1, rho0, S, False)
    want = np.tile(np.diag(rho0).real, (B, 1))
    # P_R = I exactly: rho_00..rho_77 bitwise; rho_88 is recovered from the trace
    # by the trace-reduced step kernel (t - the other eight), one rounding per term
    assert np.array_equal(pz[:, :8], want[:, :8])
    assert np.abs(pz[:, 8] - want[:, 8]).max() <= 8 * np.finfo(float).eps
    h = np.zeros((9, 9), complex)
    for _ in range(6):
        i, j = rng.integers(0, 9, 2)
        v = rng.normal() + 1j * rng.normal()
        h[i, j] += v
        h[j, i] += np.conj(v)
    hd = np.diag(rng.normal(size=9)).astype(complex)
    hs = np.zeros((9, 9), complex)
    hs[0, 3] = hs[3, 0] = 0.4
    op = np.zeros((1, 9, 9), complex)
    op[0, 2, 5] = 0.3
    ps, es = _sweep_real(lbg, torch, h, hd, hs, op, delta, scale, 0.1, rho0, S, False)
    pd, ed = _sweep_real(lbg, torch, h, hd, hs, op, delta, scale, 0.1, rho0, S, True)
    assert np.abs(ps - pd).max() <= 1e-12
    assert np.abs(es - ed).max() <= 1e-12 * B


def test_sweep_dense_generator_falls_back_to_dense_build(lbg, torch):
    """A generator with no sparsity (dense random Hermitian h0) overflows the
    sparse plan's k-step capacity; the build must take the dense path on the
    device and still match the reference-form complex path."""
    dev = torch.device("cuda")
    B, S = 1030, 25
    rng = np.random.default_rng(3)
    a = rng.normal(size=(9, 9)) + 1j * rng.normal(size=(9, 9))
    h0 = 0.05 * (a + a.conj().T)
    _, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(0, B)
    rho0 = np.zeros((9, 9), complex)
    rho0[0, 0] = 1.0
    pr, er = _sweep_real(lbg, torch, h0, hd, hs, ops, delta, scale, 0.1, rho0, S, False)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(rho0), S, pops, ens, work,
                         mode="complex")
    torch.cuda.synchronize()
    assert np.abs(pr - pops.cpu().numpy()).max() <= TOL_RHO
    assert np.abs(er - ens.cpu().numpy()).max() <= TOL_RHO * B


def test_sweep_real_mode_rejects_non_hermitian(lbg, torch):
    dev = torch.device("cuda")
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rho0 = np.zeros((9, 9), complex)
    rho0[0, 0] = 1.0
    rho0[0, 1] = 1e-3
    pops = torch.zeros(1, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, 1), dtype=torch.uint8, device=dev)
    with pytest.raises(ValueError):
        lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(np.zeros(1)), T(np.ones(1)), 0.1, T(rho0), 5,
                             pops, ens, work, mode="real")


# ------------------------------------------------------- drop-in boundary ---
def test_reference_evolve_drives_the_gpu_kernel():
    """tests/cpp/dropin_gate: the reference's own lb::evolve / grape_chain with
    KernelProfile{"b200", lbg_step_aos, lbg_step_soa} (kernels.hpp:29-33)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "_bin", "dropin_gate")
    if not os.path.exists(exe):
        pytest.skip("dropin_gate not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all criteria passed" in r.stdout


def test_nccl_allreduce_single_rank(lbg, torch):
    """lbg_nccl_* + lbg_allreduce_sum_dev (the engine's one collective) on a
    1-rank communicator: the sum over one rank is the identity."""
    import ctypes as C
    L = lbg.lib()
    uid = C.create_string_buffer(128)
    assert L.lbg_nccl_unique_id(C.cast(uid, C.c_void_p)) == 0, L.lbg_last_error()
    comm = C.c_void_p()
    assert L.lbg_nccl_comm_init(C.byref(comm), 1, C.cast(uid, C.c_void_p), 0) == 0, L.lbg_last_error()
    buf = torch.arange(162, dtype=torch.float64, device="cuda")
    want = buf.clone()
    assert L.lbg_allreduce_sum_dev(C.c_void_p(buf.data_ptr()), 162, comm, None) == 0, L.lbg_last_error()
    torch.cuda.synchronize()
    assert torch.equal(buf, want)
    assert L.lbg_nccl_comm_destroy(comm) == 0


def test_ensemble_mean_through_the_engine_comm(lbg, torch):
    """bench.py's config-4 collective: NcclComm (unique id -> broadcast -> init)
    and lbg_ensemble_mean_dev (allreduce, then / global batch) on one rank; and
    the no-communicator form."""
    comm = lbg.NcclComm(0, 1, lambda raw: raw)
    ens = (torch.arange(81, dtype=torch.float64, device="cuda").reshape(9, 9) * (1 + 2j)).to(torch.complex128)
    want = ens / 7
    lbg.ensemble_mean_dev(ens, 7, comm)
    torch.cuda.synchronize()
    assert torch.allclose(ens, want, rtol=1e-15, atol=0)
    comm.close()
    x = torch.full((162,), 3.0, dtype=torch.float64, device="cuda")
    lbg.ensemble_mean_dev(x, 3, None)
    torch.cuda.synchronize()
    assert torch.equal(x, torch.ones_like(x))
    with pytest.raises(ValueError):
        lbg.ensemble_mean_dev(x, 0, None)


# ------------------------------------------------------------ GRAPE chain ---
@pytest.mark.parametrize("d,segments", [(3, 100), (9, 20), (27, 3)])
def test_grape_chain_vs_reference(lbg, reference, d, segments):
    """lbg_grape_chain vs the reference's own lb::grape_chain on cmd_grape's
    seeded inputs (commands.cpp:123-159; Table IV shapes, fewer segments at d=27)."""
    h0, hc, op, amps, dt, rho0 = reference.grape_inputs(d, segments)
    want, _, _ = reference.grape_chain(h0, hc, amps, 32, dt, op, rho0)
    got, t = lbg.grape_chain(h0, hc, amps, 32, dt, op, rho0)
    assert np.abs(got - want).max() <= TOL_RHO
    tr, herm = invariants(got)
    assert tr <= TOL_INV and herm <= TOL_INV
    assert t["build_ms"] > 0 and t["chain_ms"] > 0 and t["segments"] == segments


def test_grape_constant_pulse_equals_evolve(lbg):
    """test_propagate.cpp:216-241: a constant pulse is plain evolution."""
    rng = np.random.default_rng(31)
    r = rng.uniform(-1, 1, (3, 3)) + 1j * rng.uniform(-1, 1, (3, 3))
    h0 = 0.5 * (r + r.conj().T)
    r = rng.uniform(-1, 1, (3, 3)) + 1j * rng.uniform(-1, 1, (3, 3))
    hc = 0.5 * (r + r.conj().T)
    a = np.diag(np.sqrt([1.0, 2.0]), 1).astype(complex)
    dis = [0.2 * a]
    rho0 = np.zeros((3, 3), complex)
    rho0[2, 2] = 1.0
    amp, dt, sps, seg = 0.8, 0.002, 8, 5
    got, t = lbg.grape_chain(h0, hc, [amp] * seg, sps, dt, dis, rho0)
    P = lbg.expm(lbg.build_lindbladian(h0 + amp * hc, dis), dt)
    want = lbg.evolve(P, rho0, seg * sps)
    assert np.abs(got - want).max() <= 1e-13
    assert t["steps_per_segment"] == sps
    with pytest.raises(ValueError):
        lbg.grape_chain(h0, hc, [], 4, 0.01, dis, rho0)
    with pytest.raises(ValueError):
        lbg.grape_chain(h0, np.zeros((2, 2)), [0.5], 4, 0.01, dis, rho0)


@pytest.mark.parametrize("d", [9, 11, 27])
def test_grape_real_form_matches_complex(lbg, reference, d):
    """d = 9 (k_ptm.cu launch_ptm_grape) and n > 96 (k_grape_real.cu, odd n = 121
    exercises the padded leading dimension): an exactly Hermitian rho0 takes the
    real transfer-matrix path; a
    rho0 off Hermitian by one ulp takes the complex path. Both agree with each
    other and with the constant-pulse evolve route."""
    rng = np.random.default_rng(d)
    if d in (9, 27):
        h0, hc, op, amps, dt, rho0 = reference.grape_inputs(d, 3)
    else:
        r = rng.uniform(-1, 1, (d, d)) + 1j * rng.uniform(-1, 1, (d, d))
        h0 = 0.5 * (r + r.conj().T)
        r = rng.uniform(-1, 1, (d, d)) + 1j * rng.uniform(-1, 1, (d, d))
        hc = 0.5 * (r + r.conj().T)
        op = [0.3 * np.diag(np.sqrt(np.arange(1, d)), 1).astype(complex)]
        amps, dt = list(rng.uniform(-1, 1, 4)), 0.01
        rho0 = np.zeros((d, d), complex)
        rho0[d - 1, d - 1] = 1.0
    amps = list(amps)
    got_r, _ = lbg.grape_chain(h0, hc, amps, 8, dt, op, rho0)
    r2 = np.array(rho0, dtype=complex)
    r2[0, 1] += 1e-15
    got_c, _ = lbg.grape_chain(h0, hc, amps, 8, dt, op, r2)
    assert np.abs(got_r - got_c).max() <= TOL_RHO
    tr, herm = invariants(got_r)
    assert tr <= TOL_INV and herm <= TOL_INV
    # constant pulse: the real chain equals expm + evolve of the one generator
    got, _ = lbg.grape_chain(h0, hc, [amps[0]] * 3, 5, dt, op, rho0)
    P = lbg.expm(lbg.build_lindbladian(h0 + amps[0] * hc, op), dt)
    assert np.abs(got - lbg.evolve(P, rho0, 15)).max() <= TOL_RHO


@pytest.mark.parametrize("dt", [0.002, 0.05, 0.4])
def test_grape_real_squarings(lbg, dt):
    """k_grape_real.cu: the squaring count is decided on the device under a host
    bound (conditional products that copy past the device count). dt spans no
    squaring with bound > 0, and several squarings; the real path must match the
    complex one (rho0 off Hermitian by one ulp) and the expm + evolve route."""
    d = 10
    rng = np.random.default_rng(int(dt * 1000))
    r = rng.uniform(-1, 1, (d, d)) + 1j * rng.uniform(-1, 1, (d, d))
    h0 = 3.0 * (r + r.conj().T)
    r = rng.uniform(-1, 1, (d, d)) + 1j * rng.uniform(-1, 1, (d, d))
    hc = r + r.conj().T
    ops = [0.5 * np.diag(np.sqrt(np.arange(1, d)), 1).astype(complex), 0.2 * np.diag(np.arange(d)).astype(complex)]
    amps = list(rng.uniform(-1, 1, 5))
    rho0 = np.zeros((d, d), complex)
    rho0[d - 1, d - 1] = 0.6
    rho0[0, 0] = 0.4
    got_r, _ = lbg.grape_chain(h0, hc, amps, 6, dt, ops, rho0)
    r2 = rho0.copy()
    r2[0, 1] += 1e-15
    got_c, _ = lbg.grape_chain(h0, hc, amps, 6, dt, ops, r2)
    assert np.abs(got_r - got_c).max() <= TOL_RHO
    got1, _ = lbg.grape_chain(h0, hc, [amps[0]], 6, dt, ops, rho0)
    P = lbg.expm(lbg.build_lindbladian(h0 + amps[0] * hc, ops), dt)
    assert np.abs(got1 - lbg.evolve(P, rho0, 6)).max() <= TOL_RHO


@pytest.mark.parametrize("n,B", [(17, 16), (33, 5), (81, 8), (97, 40), (130, 333), (729, 128), (729, 100), (729, 97),
                                 (700, 128), (729, 96), (500, 200)])
def test_tiled_ragged_shapes_vs_torch(lbg, torch, n, B):
    """Regression: odd n (ragged last K chunk and last M tile) through the TMA /
    mbarrier tile engine, against torch fp64 matmuls (a plain fp64 reference).
    (729, 128), (729, 100), (729, 97), (700, 128): the exact-fit geometry (37 x 4 = 148 tiles,
    35 x 4 = 140 at n = 700
    of 20 rows x 32 trajectories, warp pairs splitting k by parity, ragged last
    row tile and trajectory tile); (729, 96), (500, 200): fewer tiles than
    resident CTAs on the default tiles, split several ways (stream-K HEAD +
    MIDDLE + TAIL parts)."""
    dev = torch.device("cuda")
    g = torch.Generator(device="cpu").manual_seed(n)
    P = (torch.randn(n, n, dtype=torch.complex128, generator=g) / n).to(dev)
    x0 = torch.randn(B, n, dtype=torch.complex128, generator=g).to(dev)
    x = x0.clone()
    ws = torch.empty(max(lbg.evolve_workspace(n, B, "tiled"), 1), dtype=torch.uint8, device=dev)
    lbg.evolve_batch_dev(P, x, 3, algo="tiled", work=ws)
    want = x0
    for _ in range(3):
        want = want @ P.T
    torch.cuda.synchronize()
    assert (x - want).abs().max().item() <= 1e-13 * want.abs().max().item()


@pytest.mark.parametrize("n,B", [(9, 3000), (81, 70), (81, 5), (729, 3), (729, 100)])
def test_all_soa_planes_entry_point(lbg, torch, n, B):
    """lbg_evolve_shared_p_planes_dev (P and the states as re / im planes, the
    reference's Variant::soa) equals the AoS path"""
    rng = np.random.default_rng(n + B)
    P = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / (2 * n)
    x = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    dev = torch.device("cuda")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    xa, pt = T(x), T(P)
    w0 = torch.empty(max(lbg.evolve_workspace(n, B), 1), dtype=torch.uint8, device=dev)
    lbg.evolve_batch_dev(pt, xa, 6, work=w0)
    xr, xi = T(x.real), T(x.imag)
    L = lbg.lib()
    L.lbg_evolve_planes_workspace.restype = C_SZ
    ws = L.lbg_evolve_planes_workspace(n, B, 0)
    work = torch.empty(ws, dtype=torch.uint8, device=dev)
    pr, pi = T(P.real), T(P.imag)  # keep the planes alive across the call
    lbg._check(L.lbg_evolve_shared_p_planes_dev(lbg._tp(pr), lbg._tp(pi), n, lbg._tp(xr), lbg._tp(xi),
                                                B, 6, 0, lbg._tp(work), None), "planes")
    torch.cuda.synchronize()
    got = xr.cpu().numpy() + 1j * xi.cpu().numpy()
    assert np.abs(got - xa.cpu().numpy()).max() <= 1e-13 * max(1.0, np.abs(got).max())


@pytest.mark.parametrize("d,B", [(2, 1000), (3, 65536), (3, 33)])
def test_small_d_sweep_real_vs_complex_and_oracle(lbg, torch, oracle, d, B):
    """per-trajectory P at d <= 3 (warp-per-trajectory build, thread-per-trajectory
    steps) against the complex path and, for sampled trajectories, the oracle"""
    rng = np.random.default_rng(d * 7 + B)
    dev = torch.device("cuda")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    if d == 3:
        h0, ops = lbg.config_model(0)
    else:
        h0 = np.array([[0.3, 0.1 - 0.05j], [0.1 + 0.05j, -0.2]], complex)
        ops = np.array([[[0, 0.05], [0, 0]]], complex)
    hd = np.diag(np.arange(d)).astype(complex)
    hs = np.zeros((d, d), complex)
    for i in range(d - 1):
        hs[i, i + 1] = hs[i + 1, i] = 0.02 * np.sqrt(i + 1)
    delta, scale = rng.uniform(-0.03, 0.03, B), rng.uniform(0.9, 1.1, B)
    r0 = np.zeros((d, d), complex)
    r0[0, 0] = 1.0
    S = 200
    outs = {}
    for mode in ("real", "complex"):
        pops = torch.zeros(B, d, dtype=torch.float64, device=dev)
        ens = torch.zeros(d, d, dtype=torch.complex128, device=dev)
        work = torch.empty(lbg.sweep_workspace(d, B), dtype=torch.uint8, device=dev)
        lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(r0), S, pops, ens, work,
                             mode=mode)
        torch.cuda.synchronize()
        outs[mode] = (pops.cpu().numpy(), ens.cpu().numpy())
    assert np.abs(outs["real"][0] - outs["complex"][0]).max() <= TOL_RHO
    assert np.abs(outs["real"][1] - outs["complex"][1]).max() <= TOL_RHO * B
    assert abs(np.trace(outs["real"][1]).real - B) <= 1e-9 * B
    for b in (0, B // 2, B - 1):
        P = oracle.expm(oracle.build_lindbladian(h0 + delta[b] * hd + scale[b] * hs, ops), 0.1)
        want = np.diag(oracle.evolve(P, r0, S)).real
        assert np.abs(outs["real"][0][b] - want).max() <= TOL_RHO, b


@pytest.mark.parametrize("d,B", [(3, 1000), (9, 257), (27, 33)])
def test_check_state_batched_vs_oracle(lbg, torch, oracle, d, B):
    """K6 (thread per state for d < 6, warp per state above) == the reference's
    check_state (validate.cpp:10-30) reduced over the batch, bit for bit."""
    rng = np.random.default_rng(d)
    g = rng.normal(size=(B, d, d)) + 1j * rng.normal(size=(B, d, d))
    rho = g @ np.conj(np.swapaxes(g, 1, 2))
    rho /= np.trace(rho, axis1=1, axis2=2)[:, None, None]
    rho[B // 2, 0, d - 1] += 3e-9  # one slightly non-Hermitian state
    rho[B // 3, 1, 1] -= 2e-9      # and one with a trace error
    x = torch.from_numpy(np.ascontiguousarray(rho.reshape(B, d * d))).cuda()
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    lbg.check_state_batched_dev(x, d, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    want = [oracle.check_state(r) for r in rho]
    assert got[0] == max(w["trace_error"] for w in want)
    assert got[1] == max(w["hermiticity_error"] for w in want)
    assert got[2] == min(w["min_diagonal"] for w in want)


def test_barrier_kernels_bitwise_deterministic(lbg, torch, reference):
    """The grid-barrier / stream-K kernels (K1c complex and real, the real GRAPE
    chain) reduce in a fixed order: two runs give identical bits. A broken
    release/acquire barrier shows up here as run-to-run differences."""
    d, B, S = 27, 256, 40
    h, ops = lbg.config_model(3)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(3, 0, B, d)
    a = lbg.evolve_batch(P, rho0, S, algo="tiled")
    b = lbg.evolve_batch(P, rho0, S, algo="tiled")
    assert np.array_equal(a, b)
    dev = torch.device("cuda")
    outs = []
    for _ in range(2):
        x = torch.from_numpy(rho0.copy()).to(dev)
        work = torch.empty(lbg.density_workspace(d * d, B), dtype=torch.uint8, device=dev)
        lbg.evolve_density_dev(torch.from_numpy(P).to(dev), x, S, work)
        torch.cuda.synchronize()
        outs.append(x.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    h0, hc, op, amps, dt, r0 = reference.grape_inputs(27, 4)
    g1, _ = lbg.grape_chain(h0, hc, amps, 16, dt, op, r0)
    g2, _ = lbg.grape_chain(h0, hc, amps, 16, dt, op, r0)
    assert np.array_equal(g1, g2)
