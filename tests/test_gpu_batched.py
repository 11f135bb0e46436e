"""Batched building blocks (include/lbg.h lbg_build_lindbladian_batched_dev,
lbg_expm_batched_dev): many independent models assembled and
exponentiated at once, as a per-parameter sweep over arbitrary models needs
(propagate.cpp:137-143 builds one model, L and P per point). Each batched
result against the single-model entry points and against the reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


def random_models(rng, B, d, n_ops):
    a = rng.normal(size=(B, d, d)) + 1j * rng.normal(size=(B, d, d))
    h = (a + np.conj(np.swapaxes(a, 1, 2))) / (2 * d)
    ops = (rng.normal(size=(B, n_ops, d, d)) + 1j * rng.normal(size=(B, n_ops, d, d))) * 0.1
    return h, ops


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


@pytest.mark.parametrize("d,n_ops", [(2, 1), (3, 2), (4, 0), (9, 4)])
def test_build_lindbladian_batched_bitwise(lbg, torch, reference, d, n_ops):
    rng = np.random.default_rng(10 * d + n_ops)
    B = 5
    h, ops = random_models(rng, B, d, n_ops)
    out = torch.empty((B, d * d, d * d), dtype=torch.complex128, device="cuda")
    lbg.build_lindbladian_batched_dev(dev(torch, h), dev(torch, ops) if n_ops else None, out)
    got = out.cpu().numpy()
    for b in range(B):
        assert np.array_equal(got[b], lbg.build_lindbladian(h[b], ops[b] if n_ops else []))
        if n_ops:
            assert np.array_equal(got[b], reference.build_lindbladian(h[b], ops[b]))


@pytest.mark.parametrize("d,scale", [(2, 1.0), (3, 1.0), (4, 1.0), (3, 40.0)])
def test_expm_batched_small_equals_single(lbg, torch, reference, d, scale):
    """n <= 16: one CTA per matrix with its own scaling — bit-identical to
    lbg_expm per matrix (scale 40 forces squarings that differ across the batch)."""
    rng = np.random.default_rng(d)
    B = 9
    h, ops = random_models(rng, B, d, 2)
    L = np.stack([reference.build_lindbladian(h[b], ops[b]) for b in range(B)]) * (scale * (1 + np.arange(B)))[:, None, None] / B
    n = d * d
    out = torch.empty((B, n, n), dtype=torch.complex128, device="cuda")
    work = torch.empty(lbg.expm_batched_workspace(n, B), dtype=torch.uint8, device="cuda")
    lbg.expm_batched_dev(dev(torch, L), 0.1, out, work)
    got = out.cpu().numpy()
    for b in range(B):
        assert np.array_equal(got[b], lbg.expm(L[b], 0.1)), b
        want = reference.expm(L[b], 0.1)
        assert np.abs(got[b] - want).max() <= 1e-13 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("n,scale", [(17, 1.0), (81, 1.0), (81, 25.0)])
def test_expm_batched_gemm_path(lbg, torch, reference, n, scale):
    """n > 16: batched DMMA GEMMs with the batch's largest squaring count;
    within 1e-13 of the per-matrix expm and of the reference's Pade-13."""
    rng = np.random.default_rng(n)
    B = 6
    a = (rng.normal(size=(B, n, n)) + 1j * rng.normal(size=(B, n, n))) / n * scale * (1 + np.arange(B))[:, None, None] / B
    out = torch.empty((B, n, n), dtype=torch.complex128, device="cuda")
    work = torch.empty(lbg.expm_batched_workspace(n, B), dtype=torch.uint8, device="cuda")
    lbg.expm_batched_dev(dev(torch, a), 0.1, out, work)
    got = out.cpu().numpy()
    for b in range(B):
        want = reference.expm(a[b], 0.1)
        tol = 1e-13 * max(1.0, np.abs(want).max())
        assert np.abs(got[b] - want).max() <= tol, b
        assert np.abs(got[b] - lbg.expm(a[b], 0.1)).max() <= tol, b


def test_expm_batched_beyond_grid_limit(lbg, torch):
    """66,000 matrices of n = 17: the GEMMs run in chunks of 65,535 along grid z."""
    g = torch.Generator(device="cuda").manual_seed(5)
    B, n = 66000, 17
    a = torch.complex(torch.randn(B, n, n, dtype=torch.float64, device="cuda", generator=g),
                      torch.randn(B, n, n, dtype=torch.float64, device="cuda", generator=g)) / (2 * n)
    out = torch.empty_like(a)
    work = torch.empty(lbg.expm_batched_workspace(n, B), dtype=torch.uint8, device="cuda")
    lbg.expm_batched_dev(a, 0.1, out, work)
    for b in (0, 65534, 65535, B - 1):
        want = lbg.expm(a[b].cpu().numpy(), 0.1)
        assert np.abs(out[b].cpu().numpy() - want).max() <= 1e-13 * max(1.0, np.abs(want).max()), b
    del a, out, work
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [9, 81])
def test_expm_rejects_non_finite_like_the_reference(lbg, torch, reference, n):
    """expm.cpp:110-112: a NaN / Inf anywhere raises std::invalid_argument —
    the batched entry point, and the single-matrix device entry point (a NaN
    column must not be dropped by the norm's max)."""
    rng = np.random.default_rng(n)
    B = 4
    a = (rng.normal(size=(B, n, n)) + 1j * rng.normal(size=(B, n, n))) / n
    work = torch.empty(lbg.expm_batched_workspace(n, B), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, n, n), dtype=torch.complex128, device="cuda")
    for bad in (np.nan, np.inf):
        x = a.copy()
        x[2, 3, 1] = bad
        with pytest.raises(ValueError, match="non-finite"):
            lbg.expm_batched_dev(dev(torch, x), 0.1, out, work)
        with pytest.raises(ValueError):
            reference.expm(x[2], 0.1)
        L = lbg.lib()
        w1 = torch.empty(L.lbg_expm_workspace(n), dtype=torch.uint8, device="cuda")
        o1 = torch.empty((n, n), dtype=torch.complex128, device="cuda")
        rc = L.lbg_expm_dev(lbg._tp(dev(torch, x[2])), n, 0.1, lbg._tp(o1), lbg._tp(w1), None)
        assert rc == 1 and b"non-finite" in L.lbg_last_error()
    lbg.expm_batched_dev(dev(torch, a), 0.1, out, work)  # usable afterwards


def test_batched_empty_and_errors(lbg, torch):
    L = lbg.lib()
    assert L.lbg_expm_batched_dev(None, 9, 0, 0.1, None, None, None) == 0  # batch 0: no-op
    assert L.lbg_build_lindbladian_batched_dev(3, None, 0, None, 0, None, None) == 0
    assert L.lbg_expm_batched_dev(None, 9, -1, 0.1, None, None, None) == 1
    assert L.lbg_expm_batched_dev(None, 0, 1, 0.1, None, None, None) == 1
    assert L.lbg_build_lindbladian_batched_dev(0, None, 0, None, 1, None, None) == 1


def test_sweep_rejects_non_finite_parameters(lbg, torch):
    """lb::expm rejects a non-finite generator (expm.cpp:110-112), so a sweep
    point with a NaN / Inf parameter or model term raises before any work."""
    T = lambda a: dev(torch, a)  # noqa: E731
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(0, 8)
    r0 = np.zeros((9, 9), complex)
    r0[0, 0] = 1.0
    pops = torch.zeros(8, 9, dtype=torch.float64, device="cuda")
    ens = torch.zeros(9, 9, dtype=torch.complex128, device="cuda")
    work = torch.empty(lbg.sweep_workspace(9, 8), dtype=torch.uint8, device="cuda")
    cases = []
    dd = delta.copy()
    dd[5] = np.nan
    cases.append((h0, hd, hs, dd, scale))
    ss = scale.copy()
    ss[7] = np.inf
    cases.append((h0, hd, hs, delta, ss))
    hh = h0.copy()
    hh[1, 2] = np.nan
    cases.append((hh, hd, hs, delta, scale))
    for a0, ad, as_, de, sc in cases:
        for mode in ("auto", "complex"):
            with pytest.raises(ValueError, match="non-finite"):
                lbg.evolve_sweep_dev(T(a0), T(ad), T(as_), T(ops), T(de), T(sc), 0.1, T(r0), 5, pops, ens, work,
                                     mode=mode)
    lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(r0), 5, pops, ens, work)


def test_grape_rejects_non_finite_like_the_reference(lbg, reference):
    """A NaN / Inf amplitude or operator entry: lb::grape_chain's per-segment
    expm throws std::invalid_argument (expm.cpp:110-112); so does the engine."""
    h0, hc, op, amps, dt, rho0 = reference.grape_inputs(3, 10)
    for what in ("amp", "h0", "op"):
        a, h, o = amps.copy(), h0.copy(), np.array(op, copy=True)
        if what == "amp":
            a[4] = np.nan
        elif what == "h0":
            h[0, 0] = np.inf
        else:
            o.reshape(-1)[3] = np.nan
        with pytest.raises(ValueError, match="non-finite"):
            lbg.grape_chain(h, hc, a, 4, dt, o, rho0)
        with pytest.raises(ValueError):
            reference.grape_chain(h, hc, a, 4, dt, o, rho0)
