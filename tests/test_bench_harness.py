"""The kernel-benchmark harness (include/lbg.h lbg_run_bench / lbg_write_bench_*)
against the reference's own lb::run_bench inputs and lb::write_csv / write_json
(proj/src/bench.cpp:70-158, 202-248), compiled from its sources (oracle/_ref).

CPU: inputs bit-identical, report text identical apart from the GPU columns.
GPU (-m gpu): the timed chain's checksum against the reference's chain.
"""
import json
import math

import numpy as np
import pytest

GPU_COLS = ("batch", "algo", "traj_steps_per_s")


def _rows(lbg):
    cfgs = [lbg.bench_config(3, "aos", 400, 7, 99), lbg.bench_config(9, "soa", 1000, 10),
            lbg.bench_config(27, "soa", 100, 2, batch=4), lbg.bench_config(3, "simd", 10, 1)]
    vals = [(70.31234, 9.2165, 17.3, 1.234567e-5, -3.5e-300), (2713.5, 19.34, 40.1, 0.0, -0.0),
            (621012.25, 5.8e4, 1.5e-7, 123456789012345.0, 1e16)]
    res = [lbg.BenchResult() for _ in cfgs]
    for r, v in zip(res, vals):
        r.ns_per_step, r.gflops, r.gbs, r.checksum_re, r.checksum_im = v
    res[3].failed = 1
    res[3].error = b'bench: simd variant "unavailable" \\ here'
    rows = []
    for c, r in zip(cfgs, res):
        row = dict(dim=c.dim, variant={0: "aos", 1: "soa", 2: "simd"}[c.variant], reps=c.reps, warmup=c.warmup)
        if r.failed:
            row.update(failed=True, error=r.error.decode())
        else:
            row.update(ns_per_step=r.ns_per_step, gflops=r.gflops, gbs=r.gbs,
                       checksum=complex(r.checksum_re, r.checksum_im))
        rows.append(row)
    return cfgs, res, rows


@pytest.mark.parametrize("dim,seed", [(1, 42), (2, 5), (3, 42), (3, 99), (9, 123), (27, 42)])
def test_bench_inputs_bit_identical(lbg, reference, dim, seed):
    p, v = lbg.bench_inputs(dim, seed)
    rp, rv = reference.bench_inputs(dim, seed)
    assert np.array_equal(p.view(np.float64), rp.view(np.float64))
    assert np.array_equal(v.view(np.float64), rv.view(np.float64))


def _strip_header(text):
    lines = text.splitlines()
    assert lines[0].startswith("# lindbench ") and "machine-profile=B200 x1" in lines[0]
    return lines[1:]


def test_csv_matches_reference_writer(lbg, reference):
    cfgs, res, rows = _rows(lbg)
    ours = _strip_header(lbg.write_bench_csv(cfgs, res, "B200 x1"))
    theirs = _strip_header(reference.write_bench(rows, "B200 x1"))
    assert ours[0] == theirs[0] + "," + ",".join(GPU_COLS)
    body = [ln if ln.startswith("#") else ",".join(ln.split(",")[:-3]) for ln in ours[1:]]
    assert body == theirs[1:]
    assert ours[-1].endswith(",1,none,nan")  # failed row: GPU columns present, value nan


def test_json_matches_reference_writer(lbg, reference):
    cfgs, res, rows = _rows(lbg)
    ours = lbg.write_bench_json(cfgs, res, "B200 x1")
    theirs = reference.write_bench(rows, "B200 x1", json=True)
    strip = [ln for ln in ours.splitlines() if not any(f'"{k}":' in ln for k in GPU_COLS)]
    drop_ts = lambda ls: [ln for ln in ls if '"timestamp"' not in ln]  # noqa: E731
    assert drop_ts(strip) == drop_ts(theirs.splitlines())
    doc = json.loads(ours)
    assert [r["batch"] for r in doc["results"]] == [1, 1, 4, 1]


def test_json_number_formatting_matches_nlohmann(lbg, reference):
    """every magnitude class of the shortest round-trip printer"""
    rng = np.random.default_rng(0)
    xs = [0.0, -0.0, 1.0, -2.5, 0.1, 1e-4, 1e-5, 0.00012345, 1e15, 1e16, 123456789012345.0, 1234567890123456.0,
          5e-324, 1.7976931348623157e308, 2.0 ** -1074, 1 / 3, 2 / 3, 100.0, 1e100, 1.5e-100]
    xs += list(10.0 ** rng.uniform(-320, 300, 400) * rng.choice([-1, 1], 400))
    xs += list(rng.integers(-10**6, 10**6, 50).astype(float))
    for i in range(0, len(xs), 5):
        chunk = xs[i:i + 5] + [1.0] * (5 - len(xs[i:i + 5]))
        c = lbg.bench_config(3, "aos", 1, 0)
        r = lbg.BenchResult()
        r.ns_per_step, r.gflops, r.gbs, r.checksum_re, r.checksum_im = chunk
        ours = json.loads(lbg.write_bench_json([c], [r], "m"))["results"][0]
        row = dict(dim=3, variant="aos", reps=1, warmup=0, ns_per_step=chunk[0], gflops=chunk[1], gbs=chunk[2],
                   checksum=complex(chunk[3], chunk[4]))
        theirs_txt = reference.write_bench([row], "m", json=True)
        ours_txt = lbg.write_bench_json([c], [r], "m")
        for key in ("ns_per_step", "gflops", "gbs", "checksum_re", "checksum_im"):
            a = [ln for ln in ours_txt.splitlines() if f'"{key}"' in ln]
            b = [ln for ln in theirs_txt.splitlines() if f'"{key}"' in ln]
            assert a == b, (key, a, b)
        assert ours["dim"] == 3 and not math.isnan(ours["gflops"])


def test_writers_empty_and_buffer_contract(lbg):
    assert '"results": []' in lbg.write_bench_json([], [], "m")
    assert lbg.write_bench_csv([], [], "m").splitlines()[1].startswith("profile,dim,variant")


# ----------------------------------------------------------------- GPU ---
@pytest.mark.gpu
@pytest.mark.parametrize("dim,variant,reps,warmup,seed", [
    (3, "aos", 400, 7, 99), (3, "soa", 300, 5, 123), (9, "soa", 100, 10, 42), (9, "aos", 120, 3, 7),
    (27, "aos", 60, 2, 42), (27, "soa", 40, 1, 11)])
def test_gpu_bench_checksum_vs_reference_chain(lbg, reference, dim, variant, reps, warmup, seed):
    r = lbg.run_bench(lbg.bench_config(dim, variant, reps, warmup, seed))
    want = reference.run_bench(dim, variant, reps, warmup, seed, "baseline")["checksum"]
    got = complex(r.checksum_re, r.checksum_im)
    assert want != 0 and abs(got - want) <= 1e-12 * abs(want), (got, want)
    d2 = dim * dim
    assert r.gflops == pytest.approx(8 * d2 * d2 / r.ns_per_step)
    assert r.gbs == pytest.approx(16 * (d2 * d2 + 2 * d2) / r.ns_per_step)
    assert not r.failed and r.algo > 0


@pytest.mark.gpu
def test_gpu_bench_reference_properties(lbg):
    """bench.cpp contract (test_bench.cpp): identical configs -> identical
    checksums; long chains decay to the same (zero) checksum; batch copies of
    the chain agree with the single chain; bad configs fail like the reference."""
    a = lbg.run_bench(lbg.bench_config(3, "soa", 700, 5, 123))
    b = lbg.run_bench(lbg.bench_config(3, "soa", 700, 5, 123))
    assert (a.checksum_re, a.checksum_im) == (b.checksum_re, b.checksum_im)
    c1 = lbg.run_bench(lbg.bench_config(3, "aos", 3000, 10))
    c2 = lbg.run_bench(lbg.bench_config(3, "aos", 6000, 10))
    assert (c1.checksum_re, c1.checksum_im) == (c2.checksum_re, c2.checksum_im) == (0.0, 0.0)
    one = lbg.run_bench(lbg.bench_config(9, "aos", 200, 3, 5, batch=1))
    many = lbg.run_bench(lbg.bench_config(9, "aos", 200, 3, 5, batch=64))
    assert abs(complex(one.checksum_re, one.checksum_im) - complex(many.checksum_re, many.checksum_im)) <= \
        1e-12 * abs(complex(one.checksum_re, one.checksum_im))
    assert many.traj_steps_per_s > one.traj_steps_per_s
    with pytest.raises(ValueError):
        lbg.run_bench(lbg.bench_config(0, "aos", 10, 1))
    with pytest.raises(ValueError):
        lbg.run_bench(lbg.bench_config(3, "aos", 0, 1))
    with pytest.raises(RuntimeError):
        lbg.run_bench(lbg.bench_config(3, "simd", 10, 1))
    r = lbg.run_bench(lbg.bench_config(3, "aos", 1, 0), raise_on_error=False)
    # one launch already spans more than 10x the 0.5 us event resolution; if
    # not, the reference's timer-resolution error is reported
    assert (not r.failed) or b"timer resolution" in r.error
    cfgs, res = lbg.run_matrix([3, 9], ["aos", "soa", "simd"], reps=200, warmup=2)
    csv = lbg.write_bench_csv(cfgs, res, "B200")
    assert csv.count("# failed:") == 2 and len(csv.splitlines()) == 2 + 6 + 2


@pytest.mark.gpu
def test_gpu_lindbench_cli(tmp_path):
    from paper_2603_18052_b200 import lindbench
    out = tmp_path / "r.json"
    rc = lindbench.main(["bench", "--dims", "3,9", "--variants", "aos,soa", "--reps", "2000", "--warmup", "5",
                         "--format", "json", "--output", str(out)])
    assert rc == 0
    doc = json.loads(out.read_text())
    assert len(doc["results"]) == 4 and all(r["ns_per_step"] > 0 for r in doc["results"])
    assert lindbench.main(["bench", "--dims", "3", "--variants", "simd", "--reps", "100",
                           "--output", str(tmp_path / "f.csv")]) == 3


def test_lindbench_cli_input_errors(capsys):
    from paper_2603_18052_b200 import lindbench
    assert lindbench.main(["bench", "--variants", "avx9"]) == 2
    assert lindbench.main(["bench", "--reps", "0"]) == 2
