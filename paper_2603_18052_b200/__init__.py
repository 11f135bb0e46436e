"""B200-native Lindblad propagation engine — Python mirror of the C-ABI.

The product is ``liblbg.so`` (hand-written sm_100a CUDA kernels + the C-ABI in
``include/lbg.h``). This module binds it with ctypes and mirrors the
reference's operator interface for the hot path (lindbench, /root/reference):

    build_lindbladian(h, ops)        lb::build_lindbladian  (lindblad.cpp:37-59)   -> GPU K5
    expm(a, dt)                      lb::expm               (expm.cpp:109-134)      -> GPU K4
    step_soa / step_aos              lb::StepSoAFn/StepAoSFn (kernels.hpp:22-24)    -> GPU shim
    evolve(p, rho0, n_steps)         lb::evolve             (propagate.cpp:75-109)  -> GPU K1/K2
    evolve_batch(p, rho0s, n_steps)  batched evolve over trajectories               -> GPU K1/K2
    evolve_sweep_dev(...)            per-trajectory build+expm+steps (config 4)     -> GPU K3-K5
    check_state(rho)                 lb::check_state        (validate.cpp:10-30)      -> GPU K6
    check_generator(l, dim, trials)  lb::check_generator    (validate.cpp:32-45)      -> GPU

Errors map like the reference: ValueError <- std::invalid_argument,
RuntimeError <- std::runtime_error. There is no CPU fallback: if the
extension is missing or no GPU is present, calls raise.

torch is used only as device-memory/stream plumbing for the ``*_dev`` entry
points (tensors' data pointers are passed through the C-ABI).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = [
    "lib", "LbgError", "ALGO", "config_dims", "config_model", "config_sweep_terms",
    "ginibre_batch", "sweep_params", "build_lindbladian", "expm", "step_soa", "step_aos",
    "evolve", "evolve_batch", "evolve_batch_dev", "evolve_workspace", "evolve_sweep_dev",
    "sweep_workspace", "check_state", "check_state_batch", "check_generator", "random_density_batch",
    "check_state_batched_dev", "launch_count",
    "reset_launch_count", "SEED",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblbg.so")
SEED = 42  # lb::kDefaultSeed (proj/include/lb/random.hpp:10)

ALGO = {"auto": 0, "chain": 1, "dfma9": 2, "smem": 3, "tiled": 4, "cta": 5, "rowsplit": 6, "cluster": 7, "ksplit": 8}
SWEEP_MODE = {"auto": 0, "complex": 1, "real": 2}

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_lib = None


class LbgError(RuntimeError):
    """CUDA / launch failure inside liblbg (LBG_ECUDA)."""


def lib() -> C.CDLL:
    """Load liblbg.so (built in-tree by paper_2603_18052_b200.build). Fails loudly."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2603_18052_b200.build`")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.lbg_last_error.restype = C.c_char_p
    L.lbg_version.restype = C.c_char_p
    L.lbg_launch_count.restype = C.c_int64
    L.lbg_step_soa.argtypes = [_dp] * 6 + [_sz]
    L.lbg_step_soa.restype = None
    L.lbg_step_aos.argtypes = [_dp, _dp, _dp, _sz]
    L.lbg_step_aos.restype = None
    L.lbg_build_lindbladian.argtypes = [_sz, _dp, _sz, _dp, _dp]
    L.lbg_build_lindbladian_dev.argtypes = [_sz, vp, _sz, vp, vp, vp]
    L.lbg_expm.argtypes = [_dp, _sz, C.c_double, _dp]
    L.lbg_expm_dev.argtypes = [vp, _sz, C.c_double, vp, vp, vp]
    L.lbg_expm_workspace.argtypes = [_sz]
    L.lbg_expm_workspace.restype = _sz
    L.lbg_build_lindbladian_batched_dev.argtypes = [_sz, vp, _sz, vp, C.c_int64, vp, vp]
    L.lbg_expm_batched_workspace.argtypes = [_sz, C.c_int64]
    L.lbg_expm_batched_workspace.restype = _sz
    L.lbg_expm_batched_dev.argtypes = [vp, _sz, C.c_int64, C.c_double, vp, vp, vp]
    L.lbg_evolve_workspace.argtypes = [_sz, C.c_int64, C.c_int]
    L.lbg_evolve_workspace.restype = _sz
    L.lbg_evolve_shared_p_soa_dev.argtypes = [vp, _sz, vp, vp, C.c_int64, C.c_int64, C.c_int, vp, vp]
    L.lbg_evolve_shared_p_aos_dev.argtypes = [vp, _sz, vp, C.c_int64, C.c_int64, C.c_int, vp, vp]
    L.lbg_evolve_shared_p.argtypes = [_dp, _sz, _dp, C.c_int64, C.c_int64, _dp, C.c_int]
    L.lbg_evolve_planes_workspace.argtypes = [_sz, C.c_int64, C.c_int]
    L.lbg_evolve_planes_workspace.restype = _sz
    L.lbg_evolve_shared_p_planes_dev.argtypes = [vp, vp, _sz, vp, vp, C.c_int64, C.c_int64, C.c_int, vp, vp]
    L.lbg_density_workspace.argtypes = [_sz, C.c_int64]
    L.lbg_density_workspace.restype = _sz
    L.lbg_evolve_density_dev.argtypes = [vp, _sz, vp, C.c_int64, C.c_int64, C.c_int, vp, vp]
    L.lbg_evolve_density.argtypes = [_dp, _sz, _dp, C.c_int64, C.c_int64, _dp]
    L.lbg_sweep_workspace.argtypes = [_sz, C.c_int64]
    L.lbg_sweep_workspace.restype = _sz
    L.lbg_evolve_sweep_dev.argtypes = [_sz, vp, vp, vp, _sz, vp, vp, vp, C.c_double, vp, C.c_int64,
                                       C.c_int64, vp, vp, C.c_int, vp, vp]
    L.lbg_check_state_batched_dev.argtypes = [vp, _sz, C.c_int64, vp, vp]
    L.lbg_allreduce_sum_dev.argtypes = [vp, _sz, vp, vp]
    L.lbg_ensemble_mean_dev.argtypes = [vp, _sz, C.c_int64, vp, vp]
    L.lbg_nccl_unique_id.argtypes = [vp]
    L.lbg_nccl_comm_init.argtypes = [C.POINTER(vp), C.c_int, vp, C.c_int]
    L.lbg_nccl_comm_destroy.argtypes = [vp]
    L.lbg_config_dims.argtypes = [C.c_int, C.POINTER(_sz), C.POINTER(_sz)]
    L.lbg_config_model.argtypes = [C.c_int, C.c_double, C.c_double, _dp, _dp]
    L.lbg_config_sweep_terms.argtypes = [_dp, _dp, _dp]
    L.lbg_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64]
    L.lbg_uniform.restype = C.c_double
    L.lbg_ginibre_batch.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int64, _sz, _dp, C.c_int]
    L.lbg_sweep_params_batch.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _dp, _dp]
    _lib = L
    return L


def _check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = f"{what}: {lib().lbg_last_error().decode()}"
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RuntimeError(msg)
    raise LbgError(msg)


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return a.ctypes.data_as(_dp)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _tp(t):
    """device pointer of a torch tensor (or None)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def _sp(stream):
    if stream is None:
        return None
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def fp64_peak() -> tuple[float, float]:
    """(DMMA, DFMA) FP64 TF/s measured live on the current device."""
    a, b = C.c_double(), C.c_double()
    L = lib()
    L.lbg_fp64_peak.argtypes = [_dp, _dp]
    _check(L.lbg_fp64_peak(C.byref(a), C.byref(b)), "fp64_peak")
    return a.value, b.value


def launch_count() -> int:
    return int(lib().lbg_launch_count())


def reset_launch_count() -> None:
    lib().lbg_reset_launch_count()


# ---------------------------------------------------------------- configs ---
def config_dims(cfg: int) -> tuple[int, int]:
    d, k = _sz(), _sz()
    _check(lib().lbg_config_dims(cfg, C.byref(d), C.byref(k)), "config_dims")
    return d.value, k.value


def config_model(cfg: int, delta: float = 0.0, s: float = 1.0):
    """(H, L_k) of BASELINE.json config `cfg`."""
    d, k = config_dims(cfg)
    h = np.zeros((d, d), np.complex128)
    ops = np.zeros((k, d, d), np.complex128)
    _check(lib().lbg_config_model(cfg, delta, s, _p(h), _p(ops)), "config_model")
    return h, ops


def config_sweep_terms():
    """Config 4: H(delta, s) = h0 + delta*hd + s*hs."""
    h0, hd, hs = (np.zeros((9, 9), np.complex128) for _ in range(3))
    _check(lib().lbg_config_sweep_terms(_p(h0), _p(hd), _p(hs)), "config_sweep_terms")
    return h0, hd, hs


def ginibre_batch(cfg: int, first: int, count: int, d: int, seed: int = SEED, threads: int | None = None):
    out = np.empty((count, d, d), np.complex128)
    threads = threads or os.cpu_count() or 1
    _check(lib().lbg_ginibre_batch(seed, cfg, first, count, d, _p(out), threads), "ginibre_batch")
    return out


def sweep_params(first: int, count: int, seed: int = SEED):
    delta, scale = np.empty(count), np.empty(count)
    _check(lib().lbg_sweep_params_batch(seed, first, count, _p(delta), _p(scale)), "sweep_params")
    return delta, scale


# ------------------------------------------------------ host (synchronous) ---
def build_lindbladian(h, ops):
    """Vectorised generator L (d^2 x d^2), assembled on the GPU (K5)."""
    h = _c128(h)
    d = h.shape[0]
    if h.ndim != 2 or h.shape[1] != d:
        raise ValueError("make_model: Hamiltonian must be square")
    ops = _c128(np.asarray(ops, np.complex128).reshape(-1, d, d)) if len(ops) else np.zeros((0, d, d), np.complex128)
    out = np.zeros((d * d, d * d), np.complex128)
    _check(lib().lbg_build_lindbladian(d, _p(h), ops.shape[0], _p(ops), _p(out)), "build_lindbladian")
    return out


def expm(a, dt: float):
    """P = exp(a*dt) on the GPU (K4: Taylor-16 / Paterson-Stockmeyer on DMMA)."""
    a = _c128(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("expm: matrix must be square")
    out = np.zeros_like(a)
    _check(lib().lbg_expm(_p(a), a.shape[0], float(dt), _p(out)), "expm")
    return out


def build_lindbladian_batched_dev(h, ops, out, stream=None):
    """Batched K5 on device tensors: h (B, d, d), ops (B, n_ops, d, d) complex128
    -> out (B, d^2, d^2); each out[b] bit-identical to build_lindbladian(h[b], ops[b])."""
    B, d = h.shape[0], h.shape[-1]
    n_ops = ops.shape[1] if ops is not None and ops.dim() == 4 else 0
    _check(lib().lbg_build_lindbladian_batched_dev(d, _tp(h), n_ops, _tp(ops) if n_ops else None, B, _tp(out),
                                                   _sp(stream)), "build_lindbladian_batched_dev")


def expm_batched_workspace(n: int, batch: int) -> int:
    return int(lib().lbg_expm_batched_workspace(n, batch))


def expm_batched_dev(a, dt: float, out, work, stream=None):
    """Batched P_b = exp(a_b dt) on device tensors a, out (B, n, n) complex128."""
    B, n = a.shape[0], a.shape[-1]
    _check(lib().lbg_expm_batched_dev(_tp(a), n, B, float(dt), _tp(out), _tp(work), _sp(stream)),
           "expm_batched_dev")


def step_soa(p, v):
    """One raw step through the lb::StepSoAFn-compatible shim."""
    p, v = _c128(p), _c128(v)
    n = v.shape[0]
    pr, pi = np.ascontiguousarray(p.real), np.ascontiguousarray(p.imag)
    vr, vi = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)
    orr, oi = np.zeros(n), np.zeros(n)
    lib().lbg_step_soa(_p(pr), _p(pi), _p(vr), _p(vi), _p(orr), _p(oi), n)
    return orr + 1j * oi


def step_aos(p, v):
    p, v = _c128(p), _c128(v)
    out = np.zeros_like(v)
    lib().lbg_step_aos(_p(p), _p(v), _p(out), v.shape[0])
    return out


def simd_available() -> bool:
    """lb::simd_available (kernels.hpp): the reference's AVX2 path has no GPU
    counterpart; the GPU kernels serve the aos and soa variants."""
    return False


def step_simd(p, v):
    """lb::step_simd (propagate.hpp:26-28): throws like the reference on a
    platform without the SIMD path (std::runtime_error)."""
    raise RuntimeError("step_simd: SIMD variant unavailable on this platform")


def _layout_check(layout: str) -> None:
    # lb::Variant (kernels.hpp:15); evolve throws std::runtime_error for an
    # unavailable variant (propagate.cpp:99-100)
    if layout == "simd":
        raise RuntimeError("evolve: SIMD variant unavailable on this platform")
    if layout not in ("aos", "soa"):
        raise ValueError(f"evolve: unknown layout {layout!r}")


def evolve_batch(p, rho0, n_steps: int, algo: str = "auto", layout: str = "soa"):
    """rho0: (B, d, d) complex -> final states (B, d, d). Host buffers, end-to-end.
    algo "density": the density-matrix mode (lbg_evolve_density, d*d <= 84).
    layout: the reference's Variant; both "aos" and "soa" run the GPU kernels
    (the device layout is the engine's choice), "simd" raises like lb::evolve."""
    _layout_check(layout)
    p, rho0 = _c128(p), _c128(rho0)
    if rho0.ndim != 3 or rho0.shape[1] != rho0.shape[2]:
        raise ValueError("evolve: states must be (B, d, d)")
    B, d = rho0.shape[0], rho0.shape[1]
    if p.shape != (d * d, d * d):
        raise ValueError("evolve: state dimension does not match propagator")
    out = np.empty_like(rho0)
    if algo == "density":
        _check(lib().lbg_evolve_density(_p(p), d, _p(rho0), B, int(n_steps), _p(out)), "evolve")
        return out
    _check(lib().lbg_evolve_shared_p(_p(p), d, _p(rho0), B, int(n_steps), _p(out), ALGO[algo]), "evolve")
    return out


def evolve(p, rho0, n_steps: int, layout: str = "soa", algo: str = "auto"):
    """lb::evolve(prop, rho0, n_steps, layout) for one trajectory
    (propagate.hpp:33-34, propagate.cpp:75-109), on the GPU."""
    _layout_check(layout)
    rho0 = _c128(rho0)
    if rho0.ndim != 2 or rho0.shape[0] != rho0.shape[1]:
        raise ValueError("evolve: state must be square")
    return evolve_batch(p, rho0[None], n_steps, algo, layout)[0]


def grape_chain(h0, hc, amplitudes, steps_per_segment: int, dt: float, dissipators, rho0):
    """lb::grape_chain (propagate.cpp:111-168) on the GPU: all segment propagators
    in one batched build, then the chain. Returns (final rho, timings dict)."""
    h0, hc, rho0 = _c128(h0), _c128(hc), _c128(rho0)
    d = h0.shape[0]
    if h0.ndim != 2 or h0.shape != hc.shape or h0.shape != rho0.shape:
        raise ValueError("grape_chain: operator shapes do not conform")
    amps = np.ascontiguousarray(amplitudes, np.float64)
    if amps.size == 0:
        raise ValueError("grape_chain: amplitudes are empty")
    ops = _c128(np.asarray(dissipators, np.complex128).reshape(-1, d, d)) if len(dissipators) else \
        np.zeros((0, d, d), np.complex128)
    out = np.empty_like(rho0)
    b, c = C.c_double(), C.c_double()
    L = lib()
    L.lbg_grape_chain.argtypes = [_sz, _dp, _dp, _dp, C.c_int64, C.c_int64, C.c_double, _sz, _dp, _dp, _dp,
                                  _dp, _dp]
    _check(L.lbg_grape_chain(d, _p(h0), _p(hc), _p(amps), amps.size, int(steps_per_segment), float(dt),
                             ops.shape[0], _p(ops) if ops.size else None, _p(rho0), _p(out), C.byref(b),
                             C.byref(c)), "grape_chain")
    bm, cm = b.value, c.value
    return out, dict(build_ms=bm, chain_ms=cm, segments=int(amps.size),
                     steps_per_segment=int(steps_per_segment), points_per_s=1000.0 / (bm + cm))


def _vcheck(rc: int, what: str) -> None:
    if rc == 0:
        return
    L = lib()
    L.lbg_validate_last_error.restype = C.c_char_p
    msg = f"{what}: {L.lbg_validate_last_error().decode()}"
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RuntimeError(msg)
    raise LbgError(msg)


def check_state_batch(rho) -> tuple[float, float, float]:
    """lb::check_state (validate.cpp:10-30) over a batch (B, d, d) on the GPU (K6):
    (max |Tr rho - 1|, max |rho_ij - conj rho_ji|, min Re rho_ii)."""
    rho = _c128(rho)
    if rho.ndim != 3 or rho.shape[1] != rho.shape[2]:
        raise ValueError("check_state: states must be (B, d, d)")
    out = np.zeros(3)
    L = lib()
    L.lbg_check_state.argtypes = [_dp, _sz, C.c_int64, _dp]
    _vcheck(L.lbg_check_state(_p(rho), rho.shape[1], rho.shape[0], _p(out)), "check_state")
    return float(out[0]), float(out[1]), float(out[2])


def check_state(rho, tol: float = 1e-8) -> dict:
    """lb::check_state (validate.cpp:10-30) for one d x d density matrix, on the GPU (K6)."""
    rho = _c128(rho)
    if rho.ndim != 2 or rho.shape[0] != rho.shape[1]:
        raise ValueError("check_state: state must be square")
    te, herm, mind = check_state_batch(rho[None])
    return dict(trace_error=te, hermiticity_error=herm, min_diagonal=mind,
                passed=te <= tol and herm <= tol and mind >= -tol)


def check_generator(l, dim: int, trials: int, tol: float = 1e-10) -> tuple[bool, float]:
    """lb::check_generator (validate.cpp:32-45): trace annihilation of the generator
    l (dim^2 x dim^2) on lb::random_density states from the reference's fixed seed;
    the traces are summed on the GPU. Returns (passed, worst |Tr|)."""
    l = _c128(np.atleast_2d(l))
    ok, worst = C.c_int(), C.c_double()
    L = lib()
    L.lbg_check_generator.argtypes = [_sz, _dp, _sz, _sz, _sz, C.c_double, C.POINTER(C.c_int), _dp]
    _vcheck(L.lbg_check_generator(dim, _p(l), l.shape[0], l.shape[1], trials, tol, C.byref(ok), C.byref(worst)),
            "check_generator")
    return bool(ok.value), worst.value


def random_density_batch(seed: int, d: int, count: int):
    """lb::random_density drawn count times from lb::make_rng(seed) (random.hpp:12-37)."""
    out = np.zeros((count, d, d), np.complex128)
    L = lib()
    L.lbg_random_density_batch.argtypes = [C.c_uint64, _sz, C.c_int64, _dp]
    _vcheck(L.lbg_random_density_batch(seed, d, count, _p(out)), "random_density_batch")
    return out


# -------------------------------------------------- device (stream-ordered) ---
def evolve_workspace(n: int, batch: int, algo: str = "auto") -> int:
    return int(lib().lbg_evolve_workspace(n, batch, ALGO[algo]))


def evolve_batch_dev(p, x, n_steps: int, algo: str = "auto", work=None, stream=None):
    """In-place on device tensors: p (n, n) complex128, x (B, n) complex128."""
    n = p.shape[0]
    B = x.shape[0]
    _check(lib().lbg_evolve_shared_p_aos_dev(_tp(p), n, _tp(x), B, int(n_steps), ALGO[algo], _tp(work),
                                             _sp(stream)), "evolve_shared_p_aos_dev")


def density_workspace(n: int, batch: int) -> int:
    return int(lib().lbg_density_workspace(n, batch))


DENSITY_MODE = {"hermitian": 0, "general": 1, "auto": 2}


def evolve_density_dev(p, rho, n_steps: int, work, mode: str = "auto", stream=None):
    """Density-matrix mode (include/lbg.h lbg_evolve_density_dev): rho (B, d, d)
    complex128 on the device, propagated in place through the real coordinates
    with P_R = T P T^-1. mode "hermitian" asserts rho is stored exactly
    Hermitian (its anti-Hermitian part is dropped), "general" propagates the
    anti-Hermitian part too, "auto" does so only when it is non-zero."""
    d = rho.shape[-1]
    _check(lib().lbg_evolve_density_dev(_tp(p), d, _tp(rho), rho.shape[0], int(n_steps),
                                        DENSITY_MODE[mode], _tp(work), _sp(stream)),
           "evolve_density_dev")


def sweep_workspace(d: int, batch: int) -> int:
    return int(lib().lbg_sweep_workspace(d, batch))


def evolve_sweep_dev(h0, hd, hs, ops, delta, scale, dt, rho0, n_steps, pops, ens_sum, work, stream=None,
                     mode: str = "auto"):
    """Config-4 sweep on device tensors (see include/lbg.h lbg_evolve_sweep_dev).

    mode "real": real d^2 x d^2 representation of the same generator (4x fewer
    flops); "complex": the reference's complex matrices; "auto": real when rho0
    is exactly Hermitian and d == 9."""
    d = h0.shape[0]
    _check(lib().lbg_evolve_sweep_dev(d, _tp(h0), _tp(hd), _tp(hs), ops.shape[0], _tp(ops), _tp(delta),
                                      _tp(scale), float(dt), _tp(rho0), delta.shape[0], int(n_steps),
                                      _tp(pops), _tp(ens_sum), SWEEP_MODE[mode], _tp(work), _sp(stream)),
           "evolve_sweep_dev")


class NcclComm:
    """The engine's NCCL communicator (include/lbg.h lbg_nccl_*): rank 0 makes the
    unique id, the caller's process group broadcasts its 128 bytes, every rank
    joins on its own device. Used only for the config-4 ensemble mean."""

    def __init__(self, rank: int, world: int, broadcast):
        L = lib()
        idb = (C.c_char * 128)()
        if rank == 0:
            _check(L.lbg_nccl_unique_id(C.cast(idb, C.c_void_p)), "nccl_unique_id")
        raw = broadcast(bytes(idb))
        C.memmove(idb, raw, 128)
        self.comm = C.c_void_p()
        _check(L.lbg_nccl_comm_init(C.byref(self.comm), world, C.cast(idb, C.c_void_p), rank), "nccl_comm_init")

    def close(self):
        if self.comm:
            _check(lib().lbg_nccl_comm_destroy(self.comm), "nccl_comm_destroy")
            self.comm = C.c_void_p()


def ensemble_mean_dev(buf, global_batch: int, comm=None, stream=None):
    """In place: buf (a device tensor of partial sums) -> sum over ranks / global_batch."""
    _check(lib().lbg_ensemble_mean_dev(_tp(buf), buf.numel() * buf.element_size() // 8, int(global_batch),
                                       comm.comm if comm is not None else None, _sp(stream)), "ensemble_mean_dev")


def check_state_batched_dev(x, d: int, out3, stream=None):
    _check(lib().lbg_check_state_batched_dev(_tp(x), d, x.shape[0], _tp(out3), _sp(stream)),
           "check_state_batched_dev")


# ------------------------------------------------------- text formats (host) ---
def _io_check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = f"{what}: {lib().lbg_io_last_error().decode()}"
    raise ValueError(msg) if rc == 1 else RuntimeError(msg)


def write_matrix(a) -> str:
    """lb::write_matrix (complex_matrix.cpp:166-177): 17-digit interchange text."""
    a = _c128(np.atleast_2d(a))
    L = lib()
    L.lbg_io_last_error.restype = C.c_char_p
    L.lbg_write_matrix.argtypes = [_dp, _sz, _sz, C.c_char_p, _sz, C.POINTER(_sz)]
    n = _sz()
    _io_check(L.lbg_write_matrix(_p(a), a.shape[0], a.shape[1], None, 0, C.byref(n)), "write_matrix")
    buf = C.create_string_buffer(n.value + 1)
    _io_check(L.lbg_write_matrix(_p(a), a.shape[0], a.shape[1], buf, n.value + 1, C.byref(n)), "write_matrix")
    return buf.value.decode()


def read_matrix(text: str):
    """lb::read_matrix (complex_matrix.cpp:179-188)."""
    L = lib()
    L.lbg_io_last_error.restype = C.c_char_p
    L.lbg_read_matrix.argtypes = [C.c_char_p, C.POINTER(_sz), C.POINTER(_sz), _dp, _sz]
    r, c = _sz(), _sz()
    raw = text.encode()
    _io_check(L.lbg_read_matrix(raw, C.byref(r), C.byref(c), None, 0), "read_matrix")
    out = np.zeros((r.value, c.value), np.complex128)
    _io_check(L.lbg_read_matrix(raw, C.byref(r), C.byref(c), _p(out), out.size), "read_matrix")
    return out


def read_model(text: str):
    """lb::read_model (model_io.cpp:37-109): returns (H, collapse ops)."""
    L = lib()
    L.lbg_io_last_error.restype = C.c_char_p
    L.lbg_read_model.argtypes = [C.c_char_p, C.POINTER(_sz), C.POINTER(_sz), _dp, _dp, _sz]
    d, k = _sz(), _sz()
    raw = text.encode()
    _io_check(L.lbg_read_model(raw, C.byref(d), C.byref(k), None, None, 0), "read_model")
    h = np.zeros((d.value, d.value), np.complex128)
    ops = np.zeros((max(k.value, 1), d.value, d.value), np.complex128)
    _io_check(L.lbg_read_model(raw, C.byref(d), C.byref(k), _p(h), _p(ops), k.value), "read_model")
    return h, ops[: k.value]


def read_model_file(path: str):
    with open(path) as f:
        return read_model(f.read())


# ---------------------------------------------------- benchmark harness ---
class BenchConfig(C.Structure):
    """lbg_bench_config (include/lbg.h) — lb::BenchConfig (bench.hpp:14-21) + batch."""
    _fields_ = [("dim", C.c_size_t), ("variant", C.c_int), ("reps", C.c_int64), ("warmup", C.c_int64),
                ("seed", C.c_uint64), ("batch", C.c_int64)]


class BenchResult(C.Structure):
    """lbg_bench_result — lb::BenchResult (bench.hpp:23-32) + the GPU columns."""
    _fields_ = [("ns_per_step", C.c_double), ("gflops", C.c_double), ("gbs", C.c_double),
                ("checksum_re", C.c_double), ("checksum_im", C.c_double), ("traj_steps_per_s", C.c_double),
                ("algo", C.c_int), ("failed", C.c_int), ("error", C.c_char * 224)]


VARIANT = {"aos": 0, "soa": 1, "simd": 2}


def bench_config(dim: int, variant: str = "soa", reps: int = 50000, warmup: int = 10, seed: int = SEED,
                 batch: int = 1) -> BenchConfig:
    return BenchConfig(dim, VARIANT[variant], reps, warmup, seed, batch)


def bench_inputs(dim: int, seed: int = SEED):
    """(P, v0) of lb::run_bench (bench.cpp:81-86), bit-identical to the reference."""
    n = dim * dim
    p = np.zeros((n, n), np.complex128)
    v = np.zeros(n, np.complex128)
    L = lib()
    L.lbg_bench_inputs.argtypes = [_sz, C.c_uint64, _dp, _dp]
    L.lbg_bench_last_error.restype = C.c_char_p
    rc = L.lbg_bench_inputs(dim, seed, _p(p), _p(v))
    if rc:
        raise ValueError(L.lbg_bench_last_error().decode())
    return p, v


def run_bench(cfg: BenchConfig, raise_on_error: bool = True) -> BenchResult:
    """lb::run_bench on the GPU (lbg_run_bench): a timed chain of cfg.reps steps."""
    L = lib()
    L.lbg_run_bench.argtypes = [C.POINTER(BenchConfig), C.POINTER(BenchResult)]
    res = BenchResult()
    rc = L.lbg_run_bench(C.byref(cfg), C.byref(res))
    if rc and raise_on_error:
        _check(rc, "run_bench")
    return res


def run_matrix(dims, variants, reps: int, warmup: int, seed: int = SEED, batch: int = 1):
    """lb::run_matrix (bench.cpp:160-185): every (dim, variant); failures kept as rows."""
    cfgs = [bench_config(d, v, reps, warmup, seed, batch) for d in dims for v in variants]
    return cfgs, [run_bench(c, raise_on_error=False) for c in cfgs]


def _write_bench(fn_name: str, cfgs, results, machine: str) -> str:
    L = lib()
    fn = getattr(L, fn_name)
    fn.argtypes = [C.POINTER(BenchConfig), C.POINTER(BenchResult), _sz, C.c_char_p, C.c_char_p, _sz,
                   C.POINTER(_sz)]
    L.lbg_bench_last_error.restype = C.c_char_p
    n = len(cfgs)
    ca = (BenchConfig * max(n, 1))(*cfgs)
    ra = (BenchResult * max(n, 1))(*results)
    ln = _sz()
    if fn(ca, ra, n, machine.encode(), None, 0, C.byref(ln)):
        raise ValueError(L.lbg_bench_last_error().decode())
    buf = C.create_string_buffer(ln.value + 1)
    if fn(ca, ra, n, machine.encode(), buf, ln.value + 1, C.byref(ln)):
        raise ValueError(L.lbg_bench_last_error().decode())
    return buf.value.decode()


def write_bench_csv(cfgs, results, machine: str) -> str:
    """lb::write_csv (bench.cpp:202-221) + GPU columns."""
    return _write_bench("lbg_write_bench_csv", cfgs, results, machine)


def write_bench_json(cfgs, results, machine: str) -> str:
    """lb::write_json (bench.cpp:223-246) + GPU keys."""
    return _write_bench("lbg_write_bench_json", cfgs, results, machine)


# ------------------------------------------------------------- roofline ---
class MachineProfile(C.Structure):
    """lbg_machine_profile — lb::MachineProfile (roofline.hpp:27-36) on the B200
    ladder: L1 = shared memory per SM, L2 = L2, L3 = HBM, DRAM = host over PCIe."""
    _fields_ = [("name", C.c_char * 64), ("peak_gflops", C.c_double), ("bandwidth_gbs", C.c_double * 4),
                ("capacity_bytes", C.c_uint64 * 3)]

    def as_dict(self):
        return dict(name=self.name.decode(), peak_gflops=self.peak_gflops, bandwidth_gbs=list(self.bandwidth_gbs),
                    capacity_bytes=list(self.capacity_bytes))


class KernelCharacter(C.Structure):
    """lbg_kernel_character — lb::KernelCharacter (roofline.hpp:16-24)."""
    _fields_ = [("dim", C.c_size_t), ("flops", C.c_uint64), ("bytes", C.c_uint64), ("ai", C.c_double),
                ("working_set_bytes", C.c_uint64), ("placement", C.c_int)]


LEVELS = ("L1", "L2", "L3", "DRAM")


def _roof(rc: int, what: str) -> None:
    if rc == 0:
        return
    L = lib()
    L.lbg_roofline_last_error.restype = C.c_char_p
    msg = f"{what}: {L.lbg_roofline_last_error().decode()}"
    raise ValueError(msg) if rc == 1 else RuntimeError(msg)


def machine_profile(name: str, peak_gflops: float, bandwidth_gbs, capacity_bytes) -> MachineProfile:
    return MachineProfile(name.encode()[:63], peak_gflops, (C.c_double * 4)(*bandwidth_gbs),
                          (C.c_uint64 * 3)(*capacity_bytes))


def measure_machine_profile() -> MachineProfile:
    """Every figure of the B200 ladder measured on the current device."""
    L = lib()
    L.lbg_measure_machine_profile.argtypes = [C.POINTER(MachineProfile)]
    m = MachineProfile()
    _check(L.lbg_measure_machine_profile(C.byref(m)), "measure_machine_profile")
    return m


def characterize(d: int) -> KernelCharacter:
    L = lib()
    L.lbg_characterize.argtypes = [_sz, C.POINTER(KernelCharacter)]
    k = KernelCharacter()
    _roof(L.lbg_characterize(d, C.byref(k)), "characterize")
    return k


def place(k: KernelCharacter, m: MachineProfile) -> KernelCharacter:
    L = lib()
    L.lbg_place.argtypes = [C.POINTER(KernelCharacter), C.POINTER(MachineProfile)]
    out = KernelCharacter.from_buffer_copy(k)
    _roof(L.lbg_place(C.byref(out), C.byref(m)), "place")
    return out


def ridge_point(m: MachineProfile, level: int) -> float:
    L = lib()
    L.lbg_ridge_point.argtypes = [C.POINTER(MachineProfile), C.c_int, _dp]
    r = C.c_double()
    _roof(L.lbg_ridge_point(C.byref(m), level, C.byref(r)), "ridge_point")
    return r.value


def classify(k: KernelCharacter, m: MachineProfile) -> dict:
    L = lib()
    L.lbg_classify.argtypes = [C.POINTER(KernelCharacter), C.POINTER(MachineProfile), C.POINTER(C.c_int), _dp]
    b, a = C.c_int(), C.c_double()
    _roof(L.lbg_classify(C.byref(k), C.byref(m), C.byref(b), C.byref(a)), "classify")
    return dict(bound="memory_bound" if b.value == 0 else "compute_bound", attainable_gflops=a.value)


def write_machine_profile(m: MachineProfile) -> str:
    L = lib()
    L.lbg_write_machine_profile.argtypes = [C.POINTER(MachineProfile), C.c_char_p, _sz, C.POINTER(_sz)]
    ln = _sz()
    _roof(L.lbg_write_machine_profile(C.byref(m), None, 0, C.byref(ln)), "write_profile")
    buf = C.create_string_buffer(ln.value + 1)
    _roof(L.lbg_write_machine_profile(C.byref(m), buf, ln.value + 1, C.byref(ln)), "write_profile")
    return buf.value.decode()


def read_machine_profile(text: str, name: str = "") -> MachineProfile:
    L = lib()
    L.lbg_read_machine_profile.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(MachineProfile)]
    m = MachineProfile()
    _roof(L.lbg_read_machine_profile(text.encode(), name.encode(), C.byref(m)), "read_profile")
    return m
