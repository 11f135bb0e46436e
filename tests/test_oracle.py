"""Pins the CPU oracle (oracle/lbo.c) before it is trusted as the checker.

(a) against golden vectors produced by the reference itself
    (tests/golden/*.npz, oracle/gen_golden.py over oracle/_ref/libref.so), and
(b) against the reference's own known-answer tests, restated:
    closed-form amplitude damping (proj/tests/test_propagate.cpp:156-176,
    acceptance.cpp:211-243), the hand-derived damping generator
    (proj/tests/oracles.hpp:97-104), generator vs term-by-term RHS
    (acceptance.cpp:132-160), trace annihilation (test_lindblad.cpp:84-99),
    expm vs a truncated-Taylor oracle (oracles.hpp:66-83, acceptance.cpp:198-206),
    matvec vs the naive oracle (test_propagate.cpp:77-91), check_state
    contract (validate.cpp:10-30).
CPU only.
"""
import numpy as np
import pytest


def taylor_expm(a, terms=30):
    """oracles.hpp:66-83 restated: own scaling to norm <= 1/2, 30 terms, squaring."""
    s, nrm = 0, np.abs(a).sum(axis=0).max()
    while nrm > 0.5:
        nrm /= 2.0
        s += 1
    m = a * 2.0 ** -s
    out = np.eye(a.shape[0], dtype=complex)
    term = np.eye(a.shape[0], dtype=complex)
    for k in range(1, terms):
        term = term @ m / k
        out = out + term
    for _ in range(s):
        out = out @ out
    return out


def rhs(h, ops, rho):
    """apply_rhs (lindblad.cpp:61-74): -i[H,rho] + sum L rho L^+ - 1/2{L^+L, rho}."""
    out = -1j * (h @ rho - rho @ h)
    for l in ops:
        ldl = l.conj().T @ l
        out += l @ rho @ l.conj().T - 0.5 * (ldl @ rho + rho @ ldl)
    return out


def test_config_models_match_reference_bitwise(oracle, golden):
    g = golden["models"]
    for cfg in range(4):
        h, ops = oracle.config_model(cfg)
        assert np.array_equal(h, g[f"c{cfg}_h"])
        assert np.array_equal(ops, g[f"c{cfg}_ops"])


def test_lindbladian_and_propagator_match_reference_bitwise(oracle, golden):
    g = golden["models"]
    for cfg in range(3):
        L = oracle.build_lindbladian(g[f"c{cfg}_h"], g[f"c{cfg}_ops"])
        assert np.array_equal(L, g[f"c{cfg}_L"])
        P = oracle.expm(L, 0.1)
        assert np.array_equal(P, g[f"c{cfg}_P"])


def test_evolve_matches_reference_subsets(oracle, golden):
    """Reference native-fast SoA reassociates (-ffast-math); agreement ~1e-15."""
    g, m = golden["evolve"], golden["models"]
    for cfg in range(3):
        P = m[f"c{cfg}_P"]
        for rho0, want in zip(g[f"c{cfg}_rho0"], g[f"c{cfg}_out"]):
            got = oracle.evolve(P, rho0, int(g[f"c{cfg}_steps"]))
            assert np.abs(got - want).max() <= 1e-13


def test_closed_form_amplitude_damping(oracle, golden):
    gamma, dt, n = 0.7, 0.004, 500
    k = golden["kat"]
    h = np.zeros((2, 2), complex)
    l = np.zeros((1, 2, 2), complex)
    l[0, 0, 1] = np.sqrt(gamma)
    L = oracle.build_lindbladian(h, l)
    want_L = np.zeros((4, 4), complex)  # oracles.hpp:97-104
    want_L[0, 3], want_L[1, 1], want_L[2, 2], want_L[3, 3] = gamma, -gamma / 2, -gamma / 2, -gamma
    assert np.abs(L - want_L).max() <= 2e-16  # sqrt(gamma)^2 rounding
    assert np.array_equal(L, k["ad_L"])
    P = oracle.expm(L, dt)
    assert np.array_equal(P, k["ad_P"])
    rho0 = np.zeros((2, 2), complex)
    rho0[1, 1] = 1.0
    rho = oracle.evolve(P, rho0, n)
    want = np.exp(-gamma * n * dt)
    assert abs(rho[1, 1].real - want) < 1e-10
    assert abs(rho[0, 0].real - (1 - want)) < 1e-10
    assert abs(rho[0, 1]) < 1e-12
    assert np.abs(rho - k["ad_out"]).max() <= 1e-14
    # acceptance.cpp:211-243: gamma = 1, dt = 1e-4, 10^4 steps
    l[0, 0, 1] = 1.0
    P = oracle.expm(oracle.build_lindbladian(h, l), 1e-4)
    rho = oracle.evolve(P, rho0, 10000)
    assert abs(rho[1, 1].real - np.exp(-1.0)) <= 1e-10


def test_generator_vs_rhs_and_trace_annihilation(oracle):
    rng = np.random.default_rng(42)
    for trial in range(30):
        d = (2, 3, 9)[trial % 3]
        r = rng.uniform(-1, 1, (d, d)) + 1j * rng.uniform(-1, 1, (d, d))
        h = 0.5 * (r + r.conj().T)
        ops = [rng.uniform(-1, 1, (d, d)) + 1j * rng.uniform(-1, 1, (d, d)) for _ in range(trial % 3)]
        L = oracle.build_lindbladian(h, np.array(ops).reshape(-1, d, d))
        rho = rng.uniform(-1, 1, (d, d)) + 1j * rng.uniform(-1, 1, (d, d))
        via = (L @ rho.reshape(-1)).reshape(d, d)
        want = rhs(h, ops, rho)
        assert np.abs(via - want).max() / np.abs(want).max() < 1e-12
        idv = np.eye(d).reshape(-1)
        assert np.abs(idv.conj() @ L).max() <= 1e-12


def test_non_hermitian_hamiltonian_rejected(oracle):
    h = np.zeros((2, 2), complex)
    h[0, 1] = 1.0
    with pytest.raises(ValueError):
        oracle.build_lindbladian(h, np.zeros((0, 2, 2), complex))


def test_expm_against_taylor_oracle_and_reference(oracle, golden):
    k = golden["kat"]
    assert np.array_equal(oracle.expm(k["expm_a"], 1.0), k["expm_p"])
    assert np.array_equal(oracle.expm(k["expm_big_a"], 1.0), k["expm_big_p"])  # squaring path
    rng = np.random.default_rng(1)
    worst = 0.0
    for t in range(20):
        a = rng.uniform(-1, 1, (9, 9)) + 1j * rng.uniform(-1, 1, (9, 9))
        a *= 2.0 * (t + 1) / 20 / np.abs(a).sum(axis=0).max()
        want = taylor_expm(a)
        worst = max(worst, np.abs(oracle.expm(a, 1.0) - want).max() / np.abs(want).max())
    assert worst < 1e-11
    # zero, diagonal, nilpotent (test_expm.cpp)
    assert np.abs(oracle.expm(np.zeros((3, 3), complex), 0.1) - np.eye(3)).max() <= 2e-16
    dg = np.diag([-1.0, 0.5 + 0.5j, 2j])
    assert np.abs(oracle.expm(dg, 1.0) - np.diag(np.exp(np.diag(dg)))).max() < 1e-13
    nil = np.zeros((2, 2), complex)
    nil[0, 1] = 1.0
    assert np.abs(oracle.expm(nil, 1.0) - np.array([[1, 1], [0, 1]])).max() <= 1e-15
    with pytest.raises(ValueError):
        oracle.expm(np.full((2, 2), np.nan, complex), 1.0)


def test_step_kernels_match_naive_matvec(oracle):
    rng = np.random.default_rng(3)
    for n in (1, 9, 16, 81):
        p = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        v = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        want = p @ v
        assert np.abs(oracle.step_soa(p, v) - want).max() < 1e-13 * np.abs(want).max()


def test_step_kernels_match_reference_profiles(oracle, reference):
    """acceptance.cpp:245-278 kernel equivalence, oracle vs every reference profile."""
    rng = np.random.default_rng(5)
    for n in (9, 81, 729):
        p = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        v = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        base = oracle.step_soa(p, v)
        assert np.array_equal(base, reference.step_soa(p, v, "baseline"))
        for prof in ("opt", "native", "native-fast"):
            got = reference.step_soa(p, v, prof)
            assert np.abs(got - base).max() / np.abs(base).max() < 1e-12


def test_check_state_contract(oracle):
    rho = np.diag([0.5, 0.5]).astype(complex)
    r = oracle.check_state(rho)
    assert r["passed"] and r["trace_error"] == 0.0
    assert not oracle.check_state(np.eye(2, dtype=complex))["passed"]  # trace 2
    bad = rho.copy()
    bad[0, 1] = 0.5
    assert not oracle.check_state(bad)["passed"]
    with pytest.raises(ValueError):
        oracle.evolve(np.eye(4, dtype=complex), np.eye(2, dtype=complex), 1)


def test_ginibre_states_are_physical(oracle):
    vals = []
    for b in range(200):
        rho = oracle.ginibre_rho(42, 1, b, 3)
        r = oracle.check_state(rho, 1e-14)
        assert r["passed"]
        assert np.linalg.eigvalsh(rho).min() > -1e-15
        vals.append(oracle.uniform(42, 1, b, 0))
    vals = np.array(vals)
    assert 0.0 < vals.min() and vals.max() < 1.0 and abs(vals.mean() - 0.5) < 0.1


def test_reference_evolve_subset_regenerates(reference, golden):
    """The committed fixtures are exactly what the reference produces here."""
    g, m = golden["evolve"], golden["models"]
    out, _ = reference.evolve_batch(m["c2_P"], g["c2_rho0"], int(g["c2_steps"]))
    assert np.array_equal(out, g["c2_out"])
