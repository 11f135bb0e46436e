"""bench.py's multi-rank path (torchrun, one rank per GPU, max-over-ranks
timing, the config-4 ensemble allreduce) exercised on the single GPU of the
test box: both ranks share cuda:0 with a gloo process group
(LBG_BENCH_SHARED_GPU=1). No kernel waits on another rank, so sharing one GPU
cannot deadlock; the numbers are not scaling measurements."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, port):
    env = dict(os.environ, LBG_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", *args]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg,port", [(1, 29611), (4, 29612)])
def test_two_ranks_one_line(cfg, port):
    line = _run(["--config", str(cfg), "--steps", "2", "--warmup", "1", "--no-cpu", "--no-extra"], port)
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["value"] > 0
    # strong scaling: the config's global batch, split [floor(rB/W), floor((r+1)B/W))
    assert line["config"]["global_batch"] == {1: 1 << 20, 4: 65536}[cfg]
    assert line["roofline"]["trajectories_this_rank"] == line["config"]["global_batch"] // 2
    assert line["scaling"] == "strong" and line["gpu_launches"] > 0
    assert line["e2e"]["max_abs_diff_vs_device"] <= 1e-12 if cfg == 1 else True
    if cfg == 4:
        assert "lbg_ensemble_mean_dev" in line["config"]["collective"]


def test_reference_arm_rank0_only():
    line = _run(["--impl", "reference", "--config", "2", "--steps", "1", "--warmup", "0"], 29613)
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["global_batch"] == 4096 and line["cpu_baseline"]["cpu_model"]


def test_weak_scaling_option():
    line = _run(["--config", "2", "--steps", "2", "--warmup", "1", "--no-cpu", "--no-extra", "--scaling", "weak"],
                29614)
    assert line["scaling"] == "weak" and line["config"]["global_batch"] == 2 * 4096
