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


def test_gpus_n_without_enough_devices_fails_loudly():
    """`python bench.py --gpus 2` must not silently measure one GPU: with fewer
    visible CUDA devices than requested it exits non-zero (here: none)."""
    import os
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this box has two GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "LIFE_BENCH_DEVICE")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "1", "--steps",
                        "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300, env=env)
    assert r.returncode != 0
    assert "refusing" in r.stderr
    assert not [l for l in r.stdout.splitlines() if l.strip().startswith("{")]


@pytest.mark.gpu
@pytest.mark.parametrize("config", [1, 3])
def test_gpus_2_self_launches_ranks_with_parity(config):
    """`python bench.py --gpus 2` (no torchrun) starts 2 ranks itself; the
    LIFE_BENCH_DEVICE emulation puts both on cuda:0 over gloo (host barriers,
    no kernel waits on another rank).  The line reports n_gpus 2, per-rank
    stats, and parity against the reference golden after the timed run."""
    import os
    env = dict(os.environ, LIFE_BENCH_DEVICE="0", LIFE_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", str(config),
                        "--steps", "3", "--warmup", "3", "--no-e2e"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["config"]["parallelism"] == "rowbands2"
    assert j["parity"]["ok"] is True, j["parity"]
    assert [x["rank"] for x in j["ranks"]] == [0, 1]
    assert all(x["interior_ms"] > 0 for x in j["ranks"])
    assert j["config"]["emulated_ranks_on_one_gpu"] is True


@pytest.mark.gpu
def test_single_process_multi_device_context_line():
    """--single-process: one process, 3 bands through life_ctx_create_multi
    (emulated on cuda:0), parity against the reference golden."""
    import os
    env = dict(os.environ, LIFE_BENCH_DEVICE="0")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--single-process", "--gpus", "3",
                        "--config", "4", "--steps", "2", "--warmup", "3"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    j = json.loads([l for l in r.stdout.splitlines() if l.strip().startswith("{")][0])
    assert j["n_gpus"] == 3 and j["parity"]["ok"] is True and len(j["bands"]) == 3
    assert j["e2e"]["value"] > 0 and j["e2e"]["h2d_bytes_per_step"] == 12289 * 641 * 8
    assert j["config"]["bounds"] == [0, 4097, 8193, 12289]


@pytest.mark.gpu
def test_one_gpu_line_carries_parity():
    j = run_bench("--config", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e")
    assert j["parity"]["ok"] is True and j["n_gpus"] == 1
    assert j["roofline"]["kernel"].startswith("packed_")  # config 2: the pair layout (auto rule)
    assert 0.5 < j["roofline"]["step_frac"] <= j["roofline"]["frac"] * 1.05


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
    assert j["parity"]["ok"] is True


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
