"""The reference's invariant checks on the GPU (validate.cpp:10-45) against the
reference itself: lb::check_state through K6 with host buffers, and
lb::check_generator (trace annihilation) with the reference's own state
sequence (lb::random_density from lb::make_rng(42))."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_check_state_host_contract(lbg, reference):
    """test_validate.cpp-style cases: valid, trace-broken, non-Hermitian,
    negative diagonal, and the tolerance edge; GPU == lb::check_state."""
    cases = [np.diag([0.25, 0.75]).astype(complex), np.eye(2, dtype=complex)]
    r = np.diag([0.5, 0.5]).astype(complex)
    r[0, 1] = 3e-8
    cases.append(r)
    r = np.diag([1.0 + 2e-8, -2e-8]).astype(complex)
    cases.append(r)
    r = np.diag([0.6, 0.4]).astype(complex)
    r[0, 1], r[1, 0] = 0.1 + 0.2j, 0.1 - 0.2j + 5e-9
    cases.append(r)
    for rho in cases:
        got = lbg.check_state(rho)
        ok, te, he, md = reference.check_state(rho)
        assert got["passed"] == ok
        assert (got["trace_error"], got["hermiticity_error"], got["min_diagonal"]) == (te, he, md)
    with pytest.raises(ValueError):
        lbg.check_state(np.zeros((2, 3), complex))


def test_check_state_batch_equals_per_state(lbg, reference):
    rng = np.random.default_rng(5)
    g = rng.normal(size=(300, 9, 9)) + 1j * rng.normal(size=(300, 9, 9))
    rho = g @ np.conj(np.swapaxes(g, 1, 2))
    rho /= np.trace(rho, axis1=1, axis2=2)[:, None, None]
    rho[17, 2, 3] += 4e-9
    te, he, md = lbg.check_state_batch(rho)
    want = [reference.check_state(r)[1:] for r in rho]
    assert te == max(w[0] for w in want)
    assert he == max(w[1] for w in want)
    assert md == min(w[2] for w in want)


@pytest.mark.parametrize("cfg", [0, 2, 3])
def test_check_generator_config_models(lbg, reference, cfg):
    """Built generators annihilate the trace: same verdict as lb::check_generator,
    worst |Tr| at unit roundoff (the reference's own bound is 1e-10)."""
    h, ops = reference.config_model(cfg)
    d = h.shape[0]
    L = reference.build_lindbladian(h, ops)
    ok, worst = lbg.check_generator(L, d, 25)
    assert ok == reference.check_generator(L, d, 25) is True
    assert worst <= 1e-12
    # a tolerance below the achieved bound flips both the same way
    assert lbg.check_generator(L, d, 25, tol=0.0)[0] == reference.check_generator(L, d, 25, tol=0.0)


def test_check_generator_flags_trace_leak(lbg, reference):
    """test_validate.cpp:98-102: L(0, 0) += 1e-6 leaks trace."""
    h, ops = reference.config_model(0)
    L = reference.build_lindbladian(h, ops)
    L[0, 0] += 1e-6
    ok, worst = lbg.check_generator(L, 3, 10)
    assert not ok and not reference.check_generator(L, 3, 10)
    assert worst > 1e-10


def test_check_generator_zero_and_shapes(lbg, reference):
    """test_validate.cpp:84-86, 104-107: the zero generator passes; a matrix that
    is not dim^2 x dim^2 is rejected (std::invalid_argument -> ValueError)."""
    z = np.zeros((4, 4), complex)
    assert lbg.check_generator(z, 2, 10) == (True, 0.0)
    assert reference.check_generator(z, 2, 10)
    with pytest.raises(ValueError, match="dim\\^2"):
        lbg.check_generator(z, 3, 5)
    with pytest.raises(ValueError):
        reference.check_generator(z, 3, 5)
    assert lbg.check_generator(z, 2, 0) == (True, 0.0)


def test_non_finite_inputs_follow_the_reference(lbg, reference):
    """Non-finite states meet lb::check_state's own semantics (validate.cpp:10-30,
    std::max / std::min drop a NaN operand): an Inf anywhere, or a NaN on the
    diagonal (trace), fails it, so lb::evolve throws std::invalid_argument
    (propagate.cpp:79-80) and so does the engine; a NaN OFF the diagonal passes
    the reference's check (its hermiticity max ignores NaN) and the engine's K6
    reproduces that verdict and its three numbers. lb::expm rejects non-finite
    input (expm.cpp:110-112), as does the engine."""
    h, ops = lbg.config_model(1)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho = lbg.ginibre_batch(1, 0, 70000, 3)
    for pos, bad in (((1, 2), np.inf), ((1, 2), -np.inf), ((1, 1), np.nan), ((0, 0), np.inf), ((1, 2), np.nan)):
        r = rho.copy()
        r[69998][pos] = bad
        ok, te, he, md = reference.check_state(r[69998])
        got = lbg.check_state(r[69998])
        assert got["passed"] == ok, (pos, bad)
        for a, b in ((got["trace_error"], te), (got["hermiticity_error"], he), (got["min_diagonal"], md)):
            assert a == b or (np.isnan(a) and np.isnan(b)), (pos, bad, a, b)
        if ok:
            lbg.evolve_batch(P, r, 3)  # accepted, as lb::evolve accepts it
        else:
            with pytest.raises(ValueError, match="physical-state"):
                lbg.evolve_batch(P, r, 3)
    L = lbg.build_lindbladian(h, ops)
    L[3, 4] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        lbg.expm(L, 0.1)
    with pytest.raises(ValueError):
        reference.expm(L, 0.1)


def test_sweep_validates_rho0_like_evolve(lbg):
    """lbg_evolve_sweep_dev checks rho0 as lb::evolve does (propagate.cpp:79-80)
    before building any propagator; an unphysical rho0 raises in every mode."""
    import torch
    dev = torch.device("cuda")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    delta, scale = lbg.sweep_params(0, 4)
    pops = torch.zeros(4, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, 4), dtype=torch.uint8, device=dev)
    for bad in ("trace", "nan"):
        r0 = np.zeros((9, 9), complex)
        r0[0, 0] = 1.0
        if bad == "trace":
            r0[1, 1] = 0.5
        else:
            r0[0, 0] = np.nan
        for mode in ("auto", "real", "complex"):
            with pytest.raises(ValueError, match="physical-state"):
                lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(r0), 5, pops, ens, work,
                                     mode=mode)


def test_no_per_step_allocation(lbg):
    """test_propagate.cpp:200-214: evolve allocates nothing per step. Device
    memory in use is the same after 10 and after 2,000 steps, on the device
    entry point (caller's workspace) and on the pooled host-buffer call, and
    repeated host calls of one size do not grow it."""
    import torch
    dev = torch.device("cuda")
    h, ops = lbg.config_model(2)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(2, 0, 512, 9)
    pt = torch.from_numpy(P).to(dev)
    x = torch.from_numpy(rho0.reshape(512, 81).copy()).to(dev)
    work = torch.empty(max(lbg.evolve_workspace(81, 512, "auto"), 1), dtype=torch.uint8, device=dev)
    lbg.evolve_batch_dev(pt, x, 10, work=work)  # warm: module load, attributes
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for steps in (10, 2000):
        lbg.evolve_batch_dev(pt, x, steps, work=work)
        torch.cuda.synchronize()
        assert torch.cuda.mem_get_info()[0] == free0, steps
    hb = lbg.ginibre_batch(1, 0, 70000, 3)
    P1 = lbg.expm(lbg.build_lindbladian(*lbg.config_model(1)), 0.1)
    lbg.evolve_batch(P1, hb, 5)  # grows the pool once
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    for steps in (5, 1000, 5):
        lbg.evolve_batch(P1, hb, steps)
        torch.cuda.synchronize()
        assert torch.cuda.mem_get_info()[0] == free1, steps
