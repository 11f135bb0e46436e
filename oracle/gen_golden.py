"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libref.so,
compiled from /root/reference/proj/src by oracle/Makefile). Test infrastructure.

    make -C oracle && python oracle/gen_golden.py

Fixtures (seeded inputs from oracle/lbo.c's counter stream, seed 42):
  golden_models.npz     H, L_k, L, P of configs 0..3 (P of config 3 omitted: 8.5 MB)
  golden_evolve.npz     rho0 and reference-evolved rho for config subsets:
                          c0: the full run (1 trajectory, 10^4 steps)
                          c1: 64 trajectories x 1000 steps
                          c2: 8 trajectories x 1000 steps
                          c3: 2 trajectories x 200 steps
  golden_sweep.npz      config 4: 32 trajectories (delta, s), populations after
                          500 steps and the ensemble sum, via make_model +
                          build_lindbladian + expm + evolve (grape_chain style)
  golden_kat.npz        reference known-answer cases: amplitude damping
                          (test_propagate.cpp:156-176, acceptance.cpp:211-243),
                          transmon preset generator, expm vs Taylor oracle inputs
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.bindings import Oracle, Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
SEED = 42
SUBSETS = {0: (1, 10000), 1: (64, 1000), 2: (8, 1000), 3: (2, 200)}


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    o, r = Oracle(), Reference()
    models, evo = {}, {}
    for cfg in range(4):
        h, ops = r.config_model(cfg)
        L = r.build_lindbladian(h, ops)
        models[f"c{cfg}_h"], models[f"c{cfg}_ops"] = h, ops
        if cfg < 3:
            models[f"c{cfg}_L"] = L
        P = r.expm(L, 0.1)
        if cfg < 3:
            models[f"c{cfg}_P"] = P
        d = h.shape[0]
        B, S = SUBSETS[cfg]
        if cfg == 0:
            rho0 = np.zeros((1, d, d), np.complex128)
            rho0[0, 0, 0] = 1.0
        else:
            rho0 = np.stack([o.ginibre_rho(SEED, cfg, b, d) for b in range(B)])
        out, _ = r.evolve_batch(P, rho0, S, threads=min(B, 8))
        evo[f"c{cfg}_rho0"], evo[f"c{cfg}_out"] = rho0, out
        evo[f"c{cfg}_steps"] = np.int64(S)
        print(f"config {cfg}: d={d} B={B} S={S} |L dt|_1={o.one_norm(L) * 0.1:.4f}")
    np.savez_compressed(os.path.join(OUT, "golden_models.npz"), **models)
    np.savez_compressed(os.path.join(OUT, "golden_evolve.npz"), **evo)

    B = 32
    deltas = np.array([o.sweep_params(SEED, b)[0] for b in range(B)])
    scales = np.array([o.sweep_params(SEED, b)[1] for b in range(B)])
    pops, ens, _ = r.sweep_batch(deltas, scales, steps=500, threads=8)
    np.savez_compressed(os.path.join(OUT, "golden_sweep.npz"), delta=deltas, scale=scales, pops=pops,
                        ens_sum=ens, steps=np.int64(500))

    # known-answer cases from the reference's own tests
    kat = {}
    gamma, dt = 0.7, 0.004  # test_propagate.cpp:156-176
    h = np.zeros((2, 2), np.complex128)
    lop = np.zeros((1, 2, 2), np.complex128)
    lop[0, 0, 1] = np.sqrt(gamma)
    Lad = r.build_lindbladian(h, lop)
    kat["ad_L"] = Lad
    kat["ad_P"] = r.expm(Lad, dt)
    rho0 = np.zeros((1, 2, 2), np.complex128)
    rho0[0, 1, 1] = 1.0
    kat["ad_out"] = r.evolve_batch(kat["ad_P"], rho0, 500)[0]
    # transmon preset-like model at realistic magnitude (lindblad.cpp:82-100)
    h3, ops3 = r.config_model(0)
    kat["tr_L"] = r.build_lindbladian(h3, ops3)
    # expm vs Taylor: random 9x9 scaled to target norms (acceptance.cpp:198-206)
    rng = np.random.default_rng(7)
    a = rng.uniform(-1, 1, (9, 9)) + 1j * rng.uniform(-1, 1, (9, 9))
    kat["expm_a"] = a / o.one_norm(a) * 1.3
    kat["expm_p"] = r.expm(kat["expm_a"], 1.0)
    big = a / o.one_norm(a) * 40.0  # forces scaling and squaring
    kat["expm_big_a"] = big
    kat["expm_big_p"] = r.expm(big, 1.0)
    np.savez_compressed(os.path.join(OUT, "golden_kat.npz"), **kat)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
