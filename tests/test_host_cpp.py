"""The C++ host mirror (paper_1209_4408_b200/host/life_gpu.hpp): its test
driver on the GPU, and -- in the CPU container, where the reference tree
exists -- a compile check that it accepts the reference's own life::Grid."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

HOST = os.path.join(ROOT, "paper_1209_4408_b200", "host")


@pytest.mark.gpu
def test_host_driver_on_gpu():
    from paper_1209_4408_b200 import build
    exe = build.build_host_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


def test_header_accepts_reference_grid(tmp_path):
    ref = "/root/reference/proj/core/include"
    if not os.path.isdir(ref):
        pytest.skip("reference headers not present (GPU box)")
    src = tmp_path / "dropin.cpp"
    src.write_text('''
#include <cstdint>
#include "life/grid.hpp"
#include "life_gpu.hpp"
// The reference's Grid goes straight into the GPU run():
int use(life::Grid g) {
  lifegpu::RunConfig c;
  c.iterations = 10;
  lifegpu::RunResult<life::Grid> r = lifegpu::run(std::move(g), c, {0, 10});
  life::Grid one = lifegpu::step_parallel(r.grid, c);
  return one.width() + static_cast<int>(r.stats.population_checkpoints.size());
}
''')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-include", "cstdint", "-I", ref,
                        "-I", HOST, "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_host_driver_builds():
    from paper_1209_4408_b200 import build
    exe = build.build_host_test()
    assert os.path.exists(exe)
