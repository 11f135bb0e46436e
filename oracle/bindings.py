"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

- ``Oracle``: oracle/liblbo.so, the plain-C restatement of the reference path
  (oracle/lbo.c; each function cites the reference file:line it follows).
- ``Reference``: oracle/_ref/libref.so, the unmodified reference library
  compiled from /root/reference/proj/src by oracle/Makefile, driven through
  its own C++ API by oracle/ref_driver.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the CPU baseline. The product path (paper_2603_18052_b200) never does.
Complex matrices are numpy complex128, row-major (interleaved re/im in memory,
like lb::MatrixAoS).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


class _Report(C.Structure):
    _fields_ = [("trace_error", C.c_double), ("hermiticity_error", C.c_double),
                ("min_diagonal", C.c_double), ("passed", C.c_int)]


class Oracle:
    """The C restatement (oracle/lbo.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liblbo.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        sz = C.c_size_t
        L.lbo_kron.argtypes = [_dp, sz, sz, _dp, sz, sz, _dp]
        L.lbo_matmul.argtypes = [_dp, sz, sz, _dp, sz, _dp]
        L.lbo_one_norm.argtypes = [_dp, sz, sz]
        L.lbo_one_norm.restype = C.c_double
        L.lbo_build_lindbladian.argtypes = [sz, _dp, sz, _dp, _dp]
        L.lbo_expm.argtypes = [_dp, sz, C.c_double, _dp]
        L.lbo_step_soa.argtypes = [_dp] * 6 + [sz]
        L.lbo_step_aos.argtypes = [_dp, _dp, _dp, sz]
        L.lbo_evolve.argtypes = [_dp, sz, _dp, sz, _dp]
        L.lbo_check_state.argtypes = [_dp, sz, C.c_double]
        L.lbo_check_state.restype = _Report
        L.lbo_config_dim.argtypes = [C.c_int]
        L.lbo_config_dim.restype = sz
        L.lbo_config_nops.argtypes = [C.c_int]
        L.lbo_config_nops.restype = sz
        L.lbo_config_model.argtypes = [C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.lbo_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64]
        L.lbo_uniform.restype = C.c_double
        L.lbo_ginibre_rho.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, sz, _dp]
        L.lbo_ginibre_batch.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, sz, _dp]
        L.lbo_sweep_params.argtypes = [C.c_uint64, C.c_uint64, _dp, _dp]

    def kron(self, a, b):
        a = np.ascontiguousarray(a, np.complex128)
        b = np.ascontiguousarray(b, np.complex128)
        out = np.zeros((a.shape[0] * b.shape[0], a.shape[1] * b.shape[1]), np.complex128)
        self.lib.lbo_kron(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[0], b.shape[1], _ptr(out))
        return out

    def matmul(self, a, b):
        a = np.ascontiguousarray(a, np.complex128)
        b = np.ascontiguousarray(b, np.complex128)
        out = np.zeros((a.shape[0], b.shape[1]), np.complex128)
        self.lib.lbo_matmul(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(out))
        return out

    def one_norm(self, a):
        a = np.ascontiguousarray(a, np.complex128)
        return self.lib.lbo_one_norm(_ptr(a), a.shape[0], a.shape[1])

    def build_lindbladian(self, h, ops):
        h = np.ascontiguousarray(h, np.complex128)
        d = h.shape[0]
        ops = np.ascontiguousarray(np.asarray(ops, np.complex128).reshape(-1, d, d))
        out = np.zeros((d * d, d * d), np.complex128)
        rc = self.lib.lbo_build_lindbladian(d, _ptr(h), ops.shape[0], _ptr(ops), _ptr(out))
        if rc:
            raise ValueError("lbo_build_lindbladian: invalid argument")
        return out

    def expm(self, a, dt):
        a = np.ascontiguousarray(a, np.complex128)
        out = np.zeros_like(a)
        rc = self.lib.lbo_expm(_ptr(a), a.shape[0], dt, _ptr(out))
        if rc == 1:
            raise ValueError("lbo_expm: invalid argument")
        if rc == 2:
            raise RuntimeError("lbo_expm: runtime error")
        return out

    def step_soa(self, p, v):
        p = np.asarray(p, np.complex128)
        v = np.asarray(v, np.complex128)
        n = v.shape[0]
        pr, pi = np.ascontiguousarray(p.real), np.ascontiguousarray(p.imag)
        vr, vi = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)
        orr, oi = np.zeros(n), np.zeros(n)
        self.lib.lbo_step_soa(_ptr(pr), _ptr(pi), _ptr(vr), _ptr(vi), _ptr(orr), _ptr(oi), n)
        return orr + 1j * oi

    def evolve(self, p, rho0, steps):
        p = np.ascontiguousarray(p, np.complex128)
        rho0 = np.ascontiguousarray(rho0, np.complex128)
        out = np.zeros_like(rho0)
        rc = self.lib.lbo_evolve(_ptr(p), rho0.shape[0], _ptr(rho0), steps, _ptr(out))
        if rc:
            raise ValueError("lbo_evolve: initial state fails physical-state checks")
        return out

    def check_state(self, rho, tol=1e-8):
        rho = np.ascontiguousarray(rho, np.complex128)
        r = self.lib.lbo_check_state(_ptr(rho), rho.shape[0], tol)
        return dict(trace_error=r.trace_error, hermiticity_error=r.hermiticity_error,
                    min_diagonal=r.min_diagonal, passed=bool(r.passed))

    def config_model(self, cfg, delta=0.0, s=1.0):
        d = self.lib.lbo_config_dim(cfg)
        k = self.lib.lbo_config_nops(cfg)
        h = np.zeros((d, d), np.complex128)
        ops = np.zeros((k, d, d), np.complex128)
        self.lib.lbo_config_model(cfg, delta, s, _ptr(h), _ptr(ops))
        return h, ops

    def uniform(self, seed, cfg, traj, k):
        return self.lib.lbo_uniform(seed, cfg, traj, k)

    def ginibre_rho(self, seed, cfg, traj, d):
        out = np.zeros((d, d), np.complex128)
        self.lib.lbo_ginibre_rho(seed, cfg, traj, d, _ptr(out))
        return out

    def ginibre_batch(self, seed, cfg, first, count, d):
        out = np.zeros((count, d, d), np.complex128)
        self.lib.lbo_ginibre_batch(seed, cfg, first, count, d, _ptr(out))
        return out

    def sweep_params(self, seed, traj):
        a, b = C.c_double(), C.c_double()
        self.lib.lbo_sweep_params(seed, traj, C.byref(a), C.byref(b))
        return a.value, b.value


class Reference:
    """The reference library itself (oracle/_ref/libref.so)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        sz = C.c_size_t
        L.ref_last_error.restype = C.c_char_p
        L.ref_config_model.argtypes = [C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.ref_build_lindbladian.argtypes = [sz, _dp, sz, _dp, _dp]
        L.ref_expm.argtypes = [_dp, sz, C.c_double, _dp]
        L.ref_config_propagator.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.ref_step_soa.argtypes = [C.c_char_p] + [_dp] * 6 + [sz]
        L.ref_evolve_batch.argtypes = [_dp, sz, _dp, C.c_int64, sz, _dp, C.c_int, _dp]
        L.ref_sweep_batch.argtypes = [_dp, _dp, C.c_int64, sz, _dp, _dp, C.c_int, _dp]
        L.ref_check_state.argtypes = [_dp, sz, C.c_double, _dp, _dp, _dp]
        L.ref_check_generator.argtypes = [sz, _dp, sz, sz, sz, C.c_double, C.POINTER(C.c_int)]
        L.ref_random_density.argtypes = [C.c_uint64, sz, C.c_int64, _dp]

    def _rc(self, rc, what):
        if rc == 1:
            raise ValueError(f"{what}: {self.lib.ref_last_error().decode()}")
        if rc:
            raise RuntimeError(f"{what}: {self.lib.ref_last_error().decode()}")

    def hardware_threads(self):
        return self.lib.ref_hardware_threads()

    def config_model(self, cfg, delta=0.0, s=1.0):
        d = {0: 3, 1: 3, 2: 9, 3: 27, 4: 9}[cfg]
        k = {0: 2, 1: 2, 2: 4, 3: 6, 4: 4}[cfg]
        h = np.zeros((d, d), np.complex128)
        ops = np.zeros((k, d, d), np.complex128)
        self._rc(self.lib.ref_config_model(cfg, delta, s, _ptr(h), _ptr(ops)), "config_model")
        return h, ops

    def build_lindbladian(self, h, ops):
        h = np.ascontiguousarray(h, np.complex128)
        d = h.shape[0]
        ops = np.ascontiguousarray(np.asarray(ops, np.complex128).reshape(-1, d, d))
        out = np.zeros((d * d, d * d), np.complex128)
        self._rc(self.lib.ref_build_lindbladian(d, _ptr(h), ops.shape[0], _ptr(ops), _ptr(out)),
                 "build_lindbladian")
        return out

    def expm(self, a, dt):
        a = np.ascontiguousarray(a, np.complex128)
        out = np.zeros_like(a)
        self._rc(self.lib.ref_expm(_ptr(a), a.shape[0], dt, _ptr(out)), "expm")
        return out

    def config_propagator(self, cfg, delta=0.0, s=1.0):
        d = {0: 3, 1: 3, 2: 9, 3: 27, 4: 9}[cfg]
        out = np.zeros((d * d, d * d), np.complex128)
        self._rc(self.lib.ref_config_propagator(cfg, delta, s, _ptr(out)), "config_propagator")
        return out

    def step_soa(self, p, v, profile="native-fast"):
        p = np.asarray(p, np.complex128)
        v = np.asarray(v, np.complex128)
        n = v.shape[0]
        pr, pi = np.ascontiguousarray(p.real), np.ascontiguousarray(p.imag)
        vr, vi = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)
        orr, oi = np.zeros(n), np.zeros(n)
        self._rc(self.lib.ref_step_soa(profile.encode(), _ptr(pr), _ptr(pi), _ptr(vr), _ptr(vi),
                                       _ptr(orr), _ptr(oi), n), "step_soa")
        return orr + 1j * oi

    def evolve_batch(self, p, rho0, steps, threads=1):
        """rho0: (B, d, d) complex. Returns (out, seconds)."""
        p = np.ascontiguousarray(p, np.complex128)
        rho0 = np.ascontiguousarray(rho0, np.complex128)
        out = np.zeros_like(rho0)
        secs = C.c_double()
        self._rc(self.lib.ref_evolve_batch(_ptr(p), rho0.shape[1], _ptr(rho0), rho0.shape[0], steps,
                                           _ptr(out), threads, C.byref(secs)), "evolve_batch")
        return out, secs.value

    def grape_inputs(self, d, segments, seed=42):
        """cmd_grape's seeded inputs (commands.cpp:123-159)."""
        L = self.lib
        L.ref_grape_inputs.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64] + [_dp] * 6
        h0 = np.zeros((d, d), np.complex128)
        hc = np.zeros((d, d), np.complex128)
        op = np.zeros((1, d, d), np.complex128)
        amps = np.zeros(segments)
        dt = C.c_double()
        rho0 = np.zeros((d, d), np.complex128)
        self._rc(L.ref_grape_inputs(d, segments, seed, _ptr(h0), _ptr(hc), _ptr(op), _ptr(amps), C.byref(dt),
                                    _ptr(rho0)), "grape_inputs")
        return h0, hc, op, amps, dt.value, rho0

    def grape_chain(self, h0, hc, amps, steps, dt, ops, rho0):
        """lb::grape_chain (propagate.cpp:111-168). Returns (final rho, build_ms, chain_ms)."""
        L = self.lib
        L.ref_grape_chain.argtypes = [C.c_size_t, _dp, _dp, _dp, C.c_size_t, C.c_size_t, C.c_double,
                                      C.c_size_t, _dp, _dp, _dp, _dp, _dp]
        h0, hc, rho0 = (np.ascontiguousarray(x, np.complex128) for x in (h0, hc, rho0))
        d = h0.shape[0]
        ops = np.ascontiguousarray(np.asarray(ops, np.complex128).reshape(-1, d, d))
        amps = np.ascontiguousarray(amps, np.float64)
        out = np.zeros_like(rho0)
        b, c = C.c_double(), C.c_double()
        self._rc(L.ref_grape_chain(d, _ptr(h0), _ptr(hc), _ptr(amps), amps.shape[0], steps, dt, ops.shape[0],
                                   _ptr(ops), _ptr(rho0), _ptr(out), C.byref(b), C.byref(c)), "grape_chain")
        return out, b.value, c.value

    def check_state(self, rho, tol=1e-8):
        """lb::check_state (validate.cpp:10-30). Returns (passed, trace_err, herm_err, min_diag)."""
        rho = np.ascontiguousarray(rho, np.complex128)
        te, he, md = C.c_double(), C.c_double(), C.c_double()
        rc = self.lib.ref_check_state(_ptr(rho), rho.shape[0], tol, C.byref(te), C.byref(he), C.byref(md))
        return rc == 0, te.value, he.value, md.value

    def check_generator(self, l, dim, trials, tol=1e-10):
        """lb::check_generator (validate.cpp:32-45) on the generator matrix l."""
        l = np.ascontiguousarray(l, np.complex128)
        ok = C.c_int()
        self._rc(self.lib.ref_check_generator(dim, _ptr(l), l.shape[0], l.shape[1], trials, tol, C.byref(ok)),
                 "check_generator")
        return bool(ok.value)

    def random_density(self, seed, d, count):
        """count states lb::random_density(make_rng(seed), d), drawn in sequence."""
        out = np.zeros((count, d, d), np.complex128)
        self._rc(self.lib.ref_random_density(seed, d, count, _ptr(out)), "random_density")
        return out

    def sweep_batch(self, deltas, scales, steps=500, threads=1):
        """Config 4 through the reference. Returns (pops (B,9), ens_sum (9,9), seconds)."""
        deltas = np.ascontiguousarray(deltas, np.float64)
        scales = np.ascontiguousarray(scales, np.float64)
        B = deltas.shape[0]
        pops = np.zeros((B, 9))
        ens = np.zeros((9, 9), np.complex128)
        secs = C.c_double()
        self._rc(self.lib.ref_sweep_batch(_ptr(deltas), _ptr(scales), B, steps, _ptr(pops), _ptr(ens),
                                          threads, C.byref(secs)), "sweep_batch")
        return pops, ens, secs.value

    # ---- kernel benchmark harness (bench.cpp) ----
    def bench_inputs(self, dim, seed=42):
        """(P, v0) exactly as lb::run_bench draws them (bench.cpp:81-86)."""
        L = self.lib
        L.ref_bench_inputs.argtypes = [C.c_size_t, C.c_uint64, _dp, _dp]
        n = dim * dim
        p = np.zeros((n, n), np.complex128)
        v = np.zeros(n, np.complex128)
        self._rc(L.ref_bench_inputs(dim, seed, _ptr(p), _ptr(v)), "bench_inputs")
        return p, v

    def run_bench(self, dim, variant="soa", reps=50000, warmup=10, seed=42, profile=""):
        """lb::run_bench -> dict(ns_per_step, gflops, gbs, checksum)."""
        L = self.lib
        L.ref_run_bench.argtypes = [C.c_size_t, C.c_int, C.c_size_t, C.c_size_t, C.c_uint64, C.c_char_p, _dp]
        out = np.zeros(5)
        v = {"aos": 0, "soa": 1, "simd": 2}[variant]
        self._rc(L.ref_run_bench(dim, v, reps, warmup, seed, profile.encode(), _ptr(out)), "run_bench")
        return dict(ns_per_step=out[0], gflops=out[1], gbs=out[2], checksum=complex(out[3], out[4]))

    def write_bench(self, rows, machine, json=False, profile="b200"):
        """lb::write_csv / lb::write_json (bench.cpp:202-248) of rows: dicts with dim,
        variant, reps, warmup and either failed/error or ns_per_step, gflops, gbs, checksum."""
        L = self.lib
        sz = C.c_size_t
        L.ref_write_bench.argtypes = [C.c_int, sz, C.POINTER(sz), C.POINTER(C.c_int), C.POINTER(sz),
                                      C.POINTER(sz), C.POINTER(C.c_int), _dp, C.c_char_p, C.c_char_p,
                                      C.c_char_p, C.c_char_p, sz, C.POINTER(sz)]
        n = len(rows)
        arr = lambda t, xs: (t * max(n, 1))(*xs)  # noqa: E731
        dims = arr(sz, [r["dim"] for r in rows])
        var = arr(C.c_int, [{"aos": 0, "soa": 1, "simd": 2}[r["variant"]] for r in rows])
        reps = arr(sz, [r["reps"] for r in rows])
        warm = arr(sz, [r["warmup"] for r in rows])
        failed = arr(C.c_int, [int(r.get("failed", False)) for r in rows])
        vals = np.zeros(5 * max(n, 1))
        for i, r in enumerate(rows):
            if not r.get("failed"):
                c = complex(r["checksum"])
                vals[5 * i:5 * i + 5] = [r["ns_per_step"], r["gflops"], r["gbs"], c.real, c.imag]
        errs = "\n".join(r.get("error", "") for r in rows).encode()
        ln = sz()
        self._rc(L.ref_write_bench(int(json), n, dims, var, reps, warm, failed, _ptr(vals), errs,
                                   profile.encode(), machine.encode(), None, 0, C.byref(ln)), "write_bench")
        buf = C.create_string_buffer(ln.value + 1)
        self._rc(L.ref_write_bench(int(json), n, dims, var, reps, warm, failed, _ptr(vals), errs,
                                   profile.encode(), machine.encode(), buf, ln.value + 1, C.byref(ln)),
                 "write_bench")
        return buf.value.decode()

    # ---- roofline (roofline.cpp) ----
    def read_profile(self, text, name="m"):
        L = self.lib
        L.ref_read_profile.argtypes = [C.c_char_p, C.c_char_p, _dp, _dp, C.POINTER(C.c_uint64)]
        peak = C.c_double()
        bw = np.zeros(4)
        cap = (C.c_uint64 * 3)()
        self._rc(L.ref_read_profile(text.encode(), name.encode(), C.byref(peak), _ptr(bw), cap), "read_profile")
        return dict(peak_gflops=peak.value, bandwidth_gbs=list(bw), capacity_bytes=list(cap))

    def write_profile(self, name, peak, bw, cap):
        L = self.lib
        L.ref_write_profile.argtypes = [C.c_char_p, C.c_double, _dp, C.POINTER(C.c_uint64), C.c_char_p,
                                        C.c_size_t, C.POINTER(C.c_size_t)]
        bw = np.ascontiguousarray(bw, np.float64)
        capa = (C.c_uint64 * 3)(*cap)
        ln = C.c_size_t()
        self._rc(L.ref_write_profile(name.encode(), peak, _ptr(bw), capa, None, 0, C.byref(ln)), "write_profile")
        buf = C.create_string_buffer(ln.value + 1)
        self._rc(L.ref_write_profile(name.encode(), peak, _ptr(bw), capa, buf, ln.value + 1, C.byref(ln)),
                 "write_profile")
        return buf.value.decode()

    def roofline(self, d, peak, bw, cap):
        """characterize -> place -> classify: dict(flops, bytes, ai, placement, bound, attainable_gflops)"""
        L = self.lib
        L.ref_roofline.argtypes = [C.c_size_t, C.c_double, _dp, C.POINTER(C.c_uint64), _dp]
        out = np.zeros(6)
        bw = np.ascontiguousarray(bw, np.float64)
        self._rc(L.ref_roofline(d, peak, _ptr(bw), (C.c_uint64 * 3)(*cap), _ptr(out)), "roofline")
        return dict(flops=int(out[0]), bytes=int(out[1]), ai=out[2], placement=int(out[3]), bound=int(out[4]),
                    attainable_gflops=out[5])
