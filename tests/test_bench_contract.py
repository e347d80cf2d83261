"""bench.py keeps the driver's JSON contract (one line, required keys)."""
from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    j = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "1",
                  "--cpu-budget", "0.5")
    assert j["impl"] == "reference" and j["unit"] == "GCUPS" and j["value"] > 0
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "config"):
        assert k in j
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_gpu_arm_line():
    j = run_bench("--config", "1", "--engine", "packed", "--steps", "3", "--warmup", "3",
                  "--cpu-budget", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in j, k
    assert j["value"] > 0 and j["gpu_launches"] > 0
    assert j["roofline"]["bound"] == "int" and 0 < j["roofline"]["frac"] < 1.2
    assert j["e2e"]["h2d_bytes_per_step"] == 1024 * 16 * 8 and j["e2e"]["value"] > 0
    assert j["cpu_baseline"]["value"] > 0
    b = run_bench("--engine", "byte", "--config", "1", "--steps", "3", "--warmup", "3",
                  "--byte-depth", "1", "--no-cpu")
    assert b["roofline"]["bound"] == "hbm" and b["value"] > 0
    b = run_bench("--engine", "byte", "--config", "1", "--steps", "3", "--warmup", "3", "--no-cpu")
    assert b["roofline"]["bound"] == "int" and b["config"]["temporal_depth"] == 4
    assert b["e2e"]["value"] > 0 and 0 < b["roofline"]["frac"] < 1.0
    r = run_bench("--config", "1", "--steps", "3", "--warmup", "3", "--no-cpu")  # auto -> resident
    assert r["config"]["cluster_ctas"] >= 1 and r["value"] > 0 and r["e2e"]["value"] > 0
    assert 0 < r["roofline"]["frac"] < 1.0 and r["gpu_launches"] == 3


@pytest.mark.gpu
@pytest.mark.parametrize("halo", ["peer", "nccl"])
def test_multirank_path_on_one_gpu(halo):
    """bench.py's N>1 path (row bands, peer or NCCL halos, max-over-ranks
    timing, e2e band copies) with 2 ranks sharing cuda:0 over gloo -- host
    barriers only, so no kernel waits on another rank."""
    import os
    import socket
    if halo == "nccl":
        pytest.skip("NCCL refuses two ranks on one GPU; the send/recv driver is covered "
                    "by tests/test_bands_gloo.py and test_gpu_bands.py")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, LIFE_BENCH_DEVICE="0", LIFE_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), "bench.py", "--gpus", "2", "--config", "1", "--steps", "3",
                        "--warmup", "3", "--halo", halo], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["config"]["parallelism"] == "rowbands2"
    assert "peer" in j["config"]["halo"] or "NCCL" in j["config"]["halo"]
    assert j["e2e"]["value"] > 0 and j["cpu_baseline"] is None


def test_reference_arm_under_torchrun_prints_once():
    """`--impl reference` launched like the GPU arm at N > 1: rank 0 alone
    runs the reference CPU engine and prints one JSON line; the others exit 0."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), "bench.py", "--impl", "reference", "--gpus", "2", "--config",
                        "1", "--steps", "1", "--warmup", "0", "--cpu-budget", "0.3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0 and j["e2e"]["d2h_bytes_per_step"] == 0
