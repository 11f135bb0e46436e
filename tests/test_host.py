"""Host-side logic of the product (CPU only): config models, seeded inputs,
the C-ABI surface, and argument validation that happens before any GPU work."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "lbg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(lbg_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol(lbg):
    names = header_functions()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", lbg.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (lbg_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:  # and ctypes can bind them
        getattr(lbg.lib(), n)


def test_library_is_sm100a_only(lbg):
    out = subprocess.run(["cuobjdump", "--list-elf", lbg.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_config_models_match_oracle_bitwise(lbg, oracle):
    for cfg in range(5):
        args = (0.0123, 1.05) if cfg == 4 else (0.0, 1.0)
        h, ops = lbg.config_model(cfg, *args)
        h2, ops2 = oracle.config_model(cfg, *args)
        assert np.array_equal(h, h2), cfg
        assert np.array_equal(ops, ops2), cfg


def test_sweep_terms_are_the_affine_family(lbg, oracle):
    h0, hd, hs = lbg.config_sweep_terms()
    for delta, s in [(0.0, 1.0), (0.02, 0.93), (-0.031, 1.09)]:
        h, _ = oracle.config_model(4, delta, s)
        assert np.abs(h0 + delta * hd + s * hs - h).max() <= 4e-16 * np.abs(h).max()


def test_ginibre_and_sweep_params_match_oracle_bitwise(lbg, oracle):
    for cfg, d in ((1, 3), (2, 9), (3, 27)):
        got = lbg.ginibre_batch(cfg, 1000, 4, d, threads=2)
        for b in range(4):
            assert np.array_equal(got[b], oracle.ginibre_rho(42, cfg, 1000 + b, d))
    delta, scale = lbg.sweep_params(5, 10)
    for b in range(10):
        dd, ss = oracle.sweep_params(42, 5 + b)
        assert delta[b] == dd and scale[b] == ss
    assert np.all(np.abs(delta) <= 2 * np.pi * 0.005) and np.all((scale > 0.9) & (scale < 1.1))
    assert lbg.lib().lbg_uniform(42, 1, 7, 3) == oracle.uniform(42, 1, 7, 3)


def test_ginibre_batch_is_independent_of_sharding(lbg):
    whole = lbg.ginibre_batch(1, 0, 64, 3, threads=4)
    parts = np.concatenate([lbg.ginibre_batch(1, r * 16, 16, 3, threads=1) for r in range(4)])
    assert np.array_equal(whole, parts)


def test_python_validation_before_gpu(lbg):
    with pytest.raises(ValueError):
        lbg.evolve_batch(np.eye(9), np.zeros((2, 2, 2)), 1)  # dimension mismatch
    with pytest.raises(ValueError):
        lbg.evolve(np.eye(4), np.zeros((2, 3)), 1)
    with pytest.raises(ValueError):
        lbg.expm(np.zeros((2, 3)), 0.1)
    with pytest.raises(ValueError):
        lbg.config_dims(7)
    # lb::Variant::simd has no GPU counterpart: std::runtime_error like propagate.cpp:99-100
    assert not lbg.simd_available()
    with pytest.raises(RuntimeError):
        lbg.evolve(np.eye(4), np.diag([1.0, 0.0]).astype(complex), 1, layout="simd")
    with pytest.raises(RuntimeError):
        lbg.step_simd(np.eye(4), np.zeros(4))
    with pytest.raises(ValueError):
        lbg.evolve(np.eye(4), np.diag([1.0, 0.0]).astype(complex), 1, layout="avx512")


def test_random_density_sequence_matches_reference_bitwise(lbg):
    """lbg_random_density_batch reproduces lb::random_density(make_rng(seed), d)
    drawn in sequence (the states lb::check_generator uses), bit for bit."""
    from oracle.bindings import Reference
    ref = Reference()
    for seed, d, k in ((42, 2, 25), (42, 3, 10), (7, 9, 3)):
        got = lbg.random_density_batch(seed, d, k)
        want = ref.random_density(seed, d, k)
        assert np.array_equal(got.view(np.float64), want.view(np.float64)), (seed, d)


def test_kernel_sources_have_no_fallback_paths():
    """The product never routes through the oracle or a CPU step loop."""
    pkg = os.path.join(ROOT, "paper_2603_18052_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".hpp")):
                text = open(os.path.join(dirpath, f)).read()
                for token in ("oracle.bindings", "from oracle", "import oracle", "liblbo", "libref", "lbo_"):
                    assert token not in text, (f, token)
