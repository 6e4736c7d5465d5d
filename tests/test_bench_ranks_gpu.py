"""GPU tier: bench.py's N > 1 path end to end on a one-GPU box -- two ranks
under torchrun, both on cuda:0, gloo for the barrier and the reductions
(BENCH_DIST_BACKEND / BENCH_DEVICE: a functional check, not a measurement;
the ranks' kernels never wait on one another).  Covers what a SCALE run
exercises: the cost-balanced partition, a Context per rank, the ranks'
first_col offsets, the max / sum reductions and rank 0's single JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, config, extra=()):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--config", config, "--steps", "3", "--warmup", "3",
           "--no-cpu", "--no-loop", "--e2e-steps", "2", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c2", "c3"])
def test_two_rank_bench_line(config):
    one = _run(1, config)
    two = _run(2, config)
    assert two["n_gpus"] == 2 and two["scaling"] == "strong"
    assert two["config"] == one["config"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0
    # the job is the same grid however it is split: same FLOPs and bytes,
    # same trigger count, and both ranks' outputs pass the full parity check
    assert two["step_roofline"]["flops"] == one["step_roofline"]["flops"]
    assert two["step_roofline"]["bytes"] == one["step_roofline"]["bytes"]
    assert two["workload_notes"]["triggered_deep"] == one["workload_notes"]["triggered_deep"]
    assert two["e2e"]["h2d_bytes_per_step"] == one["e2e"]["h2d_bytes_per_step"]
    assert two["e2e"]["d2h_bytes_per_step"] == one["e2e"]["d2h_bytes_per_step"]
    assert two["gpu_launches"] > 0


@pytest.mark.gpu
def test_reference_arm_prints_once_under_torchrun():
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "2",
           "--warmup", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
