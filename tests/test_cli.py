"""life-bench-gpu (paper_1209_4408_b200/host/life_bench_gpu.cpp), the
reference's CLI (tools/life_bench.cpp) on the GPU engine, driven through a
subprocess like proj/tests/test_cli.cpp: exit codes 0/2/3, the checkpoint
summary, stdout/stderr switching when rendering, the pinned CSV."""
from __future__ import annotations

import subprocess

import numpy as np
import pytest


@pytest.fixture(scope="module")
def cli():
    from paper_1209_4408_b200 import build
    build.build_lib()
    return build.build_cli()


def run(cli, *args, timeout=300):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=timeout)


def test_help_exits_zero(cli):
    r = run(cli, "--help")
    assert r.returncode == 0 and "run" in r.stdout and "bench" in r.stdout


@pytest.mark.parametrize("args", [
    ("run", "--height", "5", "--iterations", "1"),                     # missing --width
    ("run", "--width", "5", "--height", "5", "--iterations", "1", "--strategy", "rows"),
    ("run", "--width", "5", "--height", "5", "--iterations", "1", "--render", "svg"),
    ("run", "--width", "5", "--height", "5", "--iterations", "x"),
    ("run", "--width", "5", "--height", "5", "--iterations", "1", "--bogus", "1"),
    ("bench", "--sizes", "12"),
    ("bench", "--strategies", "gpu:99"),
    ("frobnicate",),
])
def test_configuration_errors_exit_2(cli, args):
    r = run(cli, *args)
    assert r.returncode == 2, (r.stdout, r.stderr)
    assert "error" in r.stderr


def test_pattern_parse_errors_exit_3(cli, tmp_path):
    bad = tmp_path / "bad.rle"
    bad.write_text("x = 3, y = 1\noqo!")
    r = run(cli, "run", "--width", "8", "--height", "8", "--iterations", "1", "--pattern", bad)
    assert r.returncode == 3
    assert "line 2, column 2" in r.stderr
    badc = tmp_path / "bad.cells"
    badc.write_text("OXO")
    assert run(cli, "run", "--width", "8", "--height", "8", "--iterations", "1",
               "--pattern", badc).returncode == 3


def test_pattern_excludes_seed(cli, tmp_path):
    p = tmp_path / "g.rle"
    p.write_text("x = 3, y = 3\nbo$2bo$3o!")
    r = run(cli, "run", "--width", "8", "--height", "8", "--iterations", "1", "--pattern", p,
            "--seed", "3")
    assert r.returncode == 2


@pytest.mark.gpu
def test_run_reports_checkpoints_and_final_population(cli, oracle):
    r = run(cli, "run", "--width", "120", "--height", "60", "--iterations", "100",
            "--strategy", "gpu:8", "--seed", "7", "--density", "0.3", "--checkpoints", "0,50,100")
    assert r.returncode == 0, r.stderr
    _, pops = oracle.run(oracle.random_fill(120, 60, 0.3, 7), 100, [0, 50, 100])
    lines = r.stdout.strip().splitlines()
    assert lines == [f"checkpoint 0 population {pops[0]}", f"checkpoint 50 population {pops[1]}",
                     f"checkpoint 100 population {pops[2]}",
                     f"final population {pops[2]} after 100 generations"]


@pytest.mark.gpu
def test_run_renders_glider_lap_to_stdout_with_summary_on_stderr(cli, tmp_path):
    p = tmp_path / "glider.rle"
    p.write_text("x = 3, y = 3\nbo$2bo$3o!")
    # the cluster-resident engine needs W % 32 == 0: a 64x64 lap (256 generations)
    r = run(cli, "run", "--width", "64", "--height", "64", "--iterations", "256",
            "--strategy", "gpu-resident", "--pattern", p)
    assert r.returncode == 0 and "final population 5 after 256 generations" in r.stdout + r.stderr
    for strat in ("gpu", "gpu-byte", "gpu-byte:5"):
        r = run(cli, "run", "--width", "16", "--height", "16", "--iterations", "64",
                "--strategy", strat, "--pattern", p, "--render", "ascii")
        assert r.returncode == 0
        assert "final population 5 after 64 generations" in r.stderr
        rows = r.stdout.rstrip("\n").split("\n")
        # centred at ((16-3)/2, (16-3)/2) = (6, 6) and home again after 64
        want = np.zeros((16, 16), np.uint8)
        for (x, y) in [(1, 0), (2, 1), (0, 2), (1, 2), (2, 2)]:
            want[6 + y, 6 + x] = 1
        got = np.array([[c == "#" for c in row] for row in rows], np.uint8)
        assert np.array_equal(got, want)


@pytest.mark.gpu
def test_run_writes_pbm_to_out(cli, tmp_path):
    out = tmp_path / "g.pbm"
    r = run(cli, "run", "--width", "40", "--height", "5", "--iterations", "3", "--render", "pbm",
            "--out", out)
    assert r.returncode == 0 and "final population" in r.stdout
    text = out.read_text()
    assert text.startswith("P1\n40 5\n") and all(len(l) <= 70 for l in text.splitlines())


@pytest.mark.gpu
def test_bench_emits_pinned_csv(cli, tmp_path, oracle):
    csv = tmp_path / "m.csv"
    r = run(cli, "bench", "--sizes", "64x32,96x40", "--iterations", "4,8", "--strategies",
            "gpu,gpu:4,gpu-byte,gpu-byte:3,gpu-resident", "--repetitions", "2", "--warmup", "0",
            "--csv", csv)
    assert r.returncode == 0, r.stderr
    lines = csv.read_text().strip().splitlines()
    assert lines[0] == ("width,height,iterations,strategy,workers,seed,density,repetitions,"
                        "median_s,speedup,hardware_threads,final_population")
    rows = [l.split(",") for l in lines[1:]]
    assert len(rows) == 2 * 2 * 5
    assert [r[3] for r in rows[:5]] == ["gpu", "gpu:4", "gpu-byte", "gpu-byte:3", "gpu-resident"]
    assert rows[0][9] == "1.00"                        # baseline row
    pops = {(r[0], r[1], r[2]) for r in rows}
    for key in pops:                                   # every engine: the oracle's population
        w, h, it = map(int, key)
        seed, dens = [(int(r[5]), float(r[6])) for r in rows if (r[0], r[1], r[2]) == key][0]
        want, _ = oracle.run(oracle.random_fill(w, h, dens, seed), it)
        assert {r[11] for r in rows if (r[0], r[1], r[2]) == key} == {str(int(want.sum()))}
    r2 = run(cli, "bench", "--sizes", "64x32", "--iterations", "4", "--strategies", "gpu",
             "--repetitions", "1", "--warmup", "0", "--gpu-columns")
    assert r2.returncode == 0
    assert r2.stdout.splitlines()[0].endswith("final_population,gcups,roofline_frac")
