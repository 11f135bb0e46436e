"""Full-output parity gate: EVERY trajectory of every BASELINE config, at full
size, against the reference itself (oracle/_ref/libref.so — the unmodified
reference compiled from its own sources — driving lb::evolve / the per-trajectory
make_model + build_lindbladian + expm + evolve of config 4 on all host threads),
in the exhaustive style of proj/tests/acceptance.cpp:245-278 (every case run,
the worst reported).

Paths covered: the device entry points (each applicable kernel), the host-buffer
call lbg_evolve_shared_p that bench.py's e2e times (chunked two-stream pipeline
with pinned and with pageable caller buffers), the per-rank shares of the
strong-scaling partition [floor(r B / W), floor((r + 1) B / W)) at W = 8, and
config 4 in both sweep modes.

Tolerances (BASELINE.json north_star): max |rho_gpu - rho_ref| <= 1e-10 after
the full step count; |Tr rho - 1| <= 1e-12 and max |rho - rho^dag| <= 1e-12 on
every GPU output.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_RHO = 1e-10
TOL_INV = 1e-12
THREADS = os.cpu_count() or 1
CFG = {1: (3, 1 << 20, 1000), 2: (9, 4096, 1000), 3: (27, 1024, 200)}
_cache = {}


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


def ref_case(lbg, reference, cfg):
    """(P_ref, rho0, reference final states) for the full config, computed once."""
    if cfg not in _cache:
        d, B, S = CFG[cfg]
        P = reference.config_propagator(cfg)
        rho0 = lbg.ginibre_batch(cfg, 0, B, d)
        out, _ = reference.evolve_batch(P, rho0, S, threads=THREADS)
        _cache[cfg] = (P, rho0, out)
    return _cache[cfg]


def assert_parity(got, want, what):
    err = float(np.abs(got - want).max())
    tr = float(np.abs(np.trace(got, axis1=-2, axis2=-1) - 1.0).max())
    herm = float(np.abs(got - np.conj(np.swapaxes(got, -1, -2))).max())
    assert err <= TOL_RHO, (what, "max|d rho|", err)
    assert tr <= TOL_INV and herm <= TOL_INV, (what, tr, herm)
    return err


def device_run(lbg, torch, P, rho0, S, algo):
    B, d = rho0.shape[0], rho0.shape[1]
    dev = torch.device("cuda")
    pt = torch.from_numpy(np.ascontiguousarray(P)).to(dev)
    xt = torch.from_numpy(rho0.reshape(B, d * d).copy()).to(dev)
    work = torch.empty(max(lbg.evolve_workspace(d * d, B, algo), 1), dtype=torch.uint8, device=dev)
    lbg.evolve_batch_dev(pt, xt, S, algo=algo, work=work)
    torch.cuda.synchronize()
    return xt.cpu().numpy().reshape(B, d, d)


def host_run(lbg, torch, P, rho0, S, pinned):
    """lbg_evolve_shared_p (the e2e call) with pinned or pageable caller buffers."""
    P = np.ascontiguousarray(P)
    if not pinned:
        return lbg.evolve_batch(P, rho0, S)
    B, d = rho0.shape[0], rho0.shape[1]
    pin_in = torch.empty(B * d * d * 2, dtype=torch.float64).pin_memory()
    pin_out = torch.empty(B * d * d * 2, dtype=torch.float64).pin_memory()
    hin = pin_in.numpy().view(np.complex128).reshape(B, d, d)
    hout = pin_out.numpy().view(np.complex128).reshape(B, d, d)
    hin[...] = rho0
    dp = C.POINTER(C.c_double)
    L = lbg.lib()
    rc = L.lbg_evolve_shared_p(P.ctypes.data_as(dp), d, hin.ctypes.data_as(dp), B, S, hout.ctypes.data_as(dp), 0)
    assert rc == 0, L.lbg_last_error()
    return hout.copy()


# ------------------------------------------------------------ shared P ---
@pytest.mark.parametrize("cfg,algo", [(1, "dfma9"), (2, "auto"), (2, "smem"), (2, "cluster"), (2, "ksplit"),
                                      (3, "tiled")])
def test_full_config_device_every_trajectory(lbg, torch, reference, cfg, algo):
    P, rho0, want = ref_case(lbg, reference, cfg)
    got = device_run(lbg, torch, P, rho0, CFG[cfg][2], algo)
    assert_parity(got, want, (cfg, algo))


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_full_config_host_pipeline_pinned_and_pageable(lbg, torch, reference, cfg):
    """The e2e call: the GPU-built P (K5 + K4, independent of the reference's
    Pade-13) and the chunked host pipeline, with pinned and pageable buffers;
    every trajectory against the reference, and the two buffer kinds agree
    bit for bit (same chunks, same kernels)."""
    d, B, S = CFG[cfg]
    _, rho0, want = ref_case(lbg, reference, cfg)
    h, ops = lbg.config_model(cfg)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    pinned = host_run(lbg, torch, P, rho0, S, pinned=True)
    pageable = host_run(lbg, torch, P, rho0, S, pinned=False)
    assert np.array_equal(pinned, pageable)
    assert_parity(pinned, want, (cfg, "host pipeline, GPU-built P"))


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_strong_scaling_shares_every_trajectory(lbg, torch, reference, cfg):
    """The per-rank shares of the global batch at W = 2, 4, 8 (rank r owns
    [floor(r B / W), floor((r + 1) B / W))) run on the small-batch kernels
    (K1a; K1b with 2 / 1 n-tiles per CTA and K1b-K for config 2; several-way
    stream-K K1c); each share against the reference's trajectories of the same
    global ids."""
    P, rho0, want = ref_case(lbg, reference, cfg)
    d, B, S = CFG[cfg]
    for W in (2, 4, 8):
        for r in sorted({0, W // 2, W - 1}):
            lo, hi = r * B // W, (r + 1) * B // W
            got = device_run(lbg, torch, P, rho0[lo:hi], S, "auto")
            assert_parity(got, want[lo:hi], (cfg, "share", W, r))


def test_pipeline_rejects_before_any_output(lbg, torch):
    """propagate.cpp:79-80: an unphysical rho0 raises before any result is
    produced — the caller's `out` is untouched (also when the bad state sits in
    the last chunk of the pipeline), pinned and pageable; the engine stays
    usable afterwards."""
    d, B, S = 3, 200_000, 50
    h, ops = lbg.config_model(1)
    P = lbg.expm(lbg.build_lindbladian(h, ops), 0.1)
    rho0 = lbg.ginibre_batch(1, 0, B, d)
    rho0[B - 5, 0, 0] += 0.5  # trace 1.5, in the last chunk
    L = lbg.lib()
    dp = C.POINTER(C.c_double)
    for pinned in (False, True):
        if pinned:
            pin_in = torch.empty(B * 18, dtype=torch.float64).pin_memory()
            pin_out = torch.empty(B * 18, dtype=torch.float64).pin_memory()
            hin = pin_in.numpy().view(np.complex128).reshape(B, d, d)
            out = pin_out.numpy().view(np.complex128).reshape(B, d, d)
            hin[...] = rho0
        else:
            hin, out = rho0, np.empty_like(rho0)
        out[...] = 7.0 + 7.0j
        rc = L.lbg_evolve_shared_p(np.ascontiguousarray(P).ctypes.data_as(dp), d, hin.ctypes.data_as(dp), B, S,
                                   out.ctypes.data_as(dp), 0)
        assert rc == 1, "LBG_EINVAL expected"
        assert b"physical-state" in L.lbg_last_error()
        assert np.all(out == 7.0 + 7.0j), "out was written before validation"
    good = lbg.evolve_batch(P, rho0[:1000], S)  # the pooled pipeline still works
    assert np.abs(np.trace(good, axis1=1, axis2=2) - 1).max() <= TOL_INV


# ------------------------------------------------------------ config 4 ---
@pytest.fixture(scope="module")
def c4_reference(lbg, reference):
    B, S = 65536, 500
    delta, scale = lbg.sweep_params(0, B)
    pops, ens, _ = reference.sweep_batch(delta, scale, steps=S, threads=THREADS)
    return delta, scale, pops, ens


@pytest.mark.parametrize("mode", ["real", "complex"])
def test_config4_every_trajectory(lbg, torch, c4_reference, mode):
    """All 65,536 per-trajectory propagators built on the GPU and stepped 500
    times; every trajectory's populations and the ensemble sum against the
    reference's make_model + build_lindbladian + expm (Pade-13) + evolve."""
    delta, scale, want_pops, want_ens = c4_reference
    B, S = delta.shape[0], 500
    dev = torch.device("cuda")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    h0, hd, hs = lbg.config_sweep_terms()
    _, ops = lbg.config_model(4)
    r0 = np.zeros((9, 9), complex)
    r0[0, 0] = 1.0
    pops = torch.zeros(B, 9, dtype=torch.float64, device=dev)
    ens = torch.zeros(9, 9, dtype=torch.complex128, device=dev)
    work = torch.empty(lbg.sweep_workspace(9, B), dtype=torch.uint8, device=dev)
    lbg.evolve_sweep_dev(T(h0), T(hd), T(hs), T(ops), T(delta), T(scale), 0.1, T(r0), S, pops, ens, work, mode=mode)
    torch.cuda.synchronize()
    got_pops, got_ens = pops.cpu().numpy(), ens.cpu().numpy()
    err = float(np.abs(got_pops - want_pops).max())
    assert err <= TOL_RHO, (mode, err)
    assert np.abs(got_pops.sum(axis=1) - 1.0).max() <= TOL_INV
    # the ensemble sum of 65,536 states: per-state tolerance scaled by B
    assert np.abs(got_ens - want_ens).max() <= TOL_RHO * B
    assert abs(np.trace(got_ens).real - B) <= TOL_INV * B
    assert np.abs(got_ens - got_ens.conj().T).max() <= TOL_INV * B


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 7, 9, 10, 12, 16])
def test_every_dimension_and_regime_against_the_reference(lbg, reference, d):
    """Random Lindblad models (random Hermitian H, two random collapse operators,
    built and exponentiated by the reference) at every d = 1..16 class, batches
    that select each automatic regime (chain / CTA / K1a / K1b / K1b-C / K1b-K /
    tiled / rowsplit), through the host-buffer call: every trajectory against
    lb::evolve."""
    rng = np.random.default_rng(100 + d)
    a = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    h = (a + a.conj().T) / (2 * d)
    ops = (rng.normal(size=(2, d, d)) + 1j * rng.normal(size=(2, d, d))) * 0.05
    P = reference.expm(reference.build_lindbladian(h, ops), 0.05)
    for B in (1, 3, 40, 300, 1100):
        g = rng.normal(size=(B, d, d)) + 1j * rng.normal(size=(B, d, d))
        rho0 = g @ np.conj(np.swapaxes(g, 1, 2))
        rho0 /= np.trace(rho0, axis1=1, axis2=2)[:, None, None]
        want, _ = reference.evolve_batch(P, rho0, 17, threads=THREADS)
        got = lbg.evolve_batch(P, rho0, 17)
        err = float(np.abs(got - want).max())
        assert err <= TOL_RHO, (d, B, err)
