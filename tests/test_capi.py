"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/life_gpu.h declares, and its host-only logic (band_bounds, pitches,
error codes without a device) behaves like the reference's."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "life_gpu.h")


def header_functions() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(life_[a-z0-9_]+)\(", text,
                                 re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1209_4408_b200 import build, capi
    build.build_lib()
    return capi.lib()


def test_header_declares_the_boundary():
    fns = header_functions()
    for required in ["life_ctx_create", "life_grid_upload_u8", "life_grid_download_u8",
                     "life_grid_init_random", "life_run", "life_population",
                     "life_grid_window_u8", "life_dev_packed_step", "life_band_bounds"]:
        assert required in fns


def test_library_exports_every_header_symbol(lib):
    from paper_1209_4408_b200 import capi
    names = {n for n, _, _ in capi.SIGNATURES}
    for fn in header_functions():
        assert hasattr(lib, fn), fn
        assert fn in names, f"{fn} missing from capi.SIGNATURES"


def test_band_bounds_matches_reference_partition(lib, golden_small):
    from paper_1209_4408_b200 import life
    for key, cuts in golden_small["partition_rows"].items():
        h, p = map(int, key.split("/"))
        assert life.band_bounds(h, p) == cuts
    with pytest.raises(life.TooManyParts):
        life.band_bounds(5, 6)
    with pytest.raises(life.TooManyParts):
        life.band_bounds(5, 0)


def test_pitches(lib):
    for w in (3, 31, 32, 64, 65, 1000, 40961, 65536, 262144):
        pw = lib.life_packed_pitch_words(w)
        assert pw % 32 == 0 and pw >= 2 * ((w + 63) // 64)
        pb = lib.life_byte_pitch(w)
        assert pb % 16 == 0 and pb >= w


def test_no_device_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1209_4408_b200 import life
    with pytest.raises(life.NoDevice):
        life.Engine(0)


def test_grid_contract_errors():
    from paper_1209_4408_b200 import life
    with pytest.raises(life.DimensionTooSmall):
        life.Grid(2, 5)
    with pytest.raises(life.DimensionTooSmall):
        life.Grid(5, 2)
    g = life.Grid(5, 4)
    assert g.wrap(5, 4) == (0, 0) and g.wrap(-1, -1) == (4, 3) and g.wrap(12, -9) == (2, 3)
    assert life.parse_strategy("gpu:8") == life.Strategy.gpu_packed(8)
    assert life.to_string(life.parse_strategy("gpu-byte")) == "gpu-byte"
    assert life.to_string(life.parse_strategy("gpu-byte:3")) == "gpu-byte:3"
    assert life.to_string(life.parse_strategy("gpu-resident")) == "gpu-resident"
    with pytest.raises(life.ConfigError):
        life.parse_strategy("gpu:17")
    with pytest.raises(life.ConfigError):
        life.parse_strategy("rows")


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1209_4408_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).replace("oracle/", ""), f


def test_interleave_auto_rule(lib):
    """life_interleave_auto (host logic): the layout and depth temporal_depth 0
    picks by width and size, the LIFE_OPT_PAIR_DEPTH / _QUAD_DEPTH overrides,
    and that an explicit temporal_depth keeps the plain kernels."""
    def pick(w, h, pair=-1, quad=-1, td=0):
        d = C.c_int32(-1)
        il = lib.life_interleave_auto(w, h, pair, quad, td, C.byref(d))
        return il, d.value
    # wide tori: quad K = 6; 16384..32768 columns: pair K = 10; narrow or small: plain
    assert pick(262144, 262144) == (4, 7)           # config 5
    assert pick(262144, 32768) == (4, 7)            # ... one of 8 row bands
    assert pick(65536, 65536) == (4, 7)             # config 3
    assert pick(49152, 49152) == (4, 7)
    assert pick(65536, 16384) == (4, 6)             # below 2^31 cells
    assert pick(32768, 32768) == (2, 10)
    assert pick(16384, 65536) == (2, 10)
    assert pick(8192, 131072) == (0, 0)
    assert pick(16384, 16384) == (2, 10)            # config 2: pair from 2^27 cells
    assert pick(12288, 12288) == (2, 10)
    assert pick(16384, 8192) == (2, 10)             # 2^27 cells
    assert pick(65536, 4096) == (2, 10)             # quad only from 2^29 cells
    assert pick(8192, 8192) == (0, 0)               # below 2^27 cells
    assert pick(8192, 32768) == (0, 0)              # 8192 columns: plain fills its strips best
    assert pick(40961, 12289) == (0, 0)             # config 4: W % 64 != 0
    assert pick(262208, 262144) == (2, 10)          # W % 128 != 0, W % 64 == 0
    # options: 0 disables a layout, > 0 forces it where the width allows
    assert pick(262144, 262144, quad=0) == (2, 10)
    assert pick(262144, 262144, pair=0, quad=0) == (0, 0)
    assert pick(1024, 100, quad=3) == (4, 3)
    assert pick(1024, 100, pair=7) == (2, 7)
    assert pick(1024, 100, pair=7, quad=3) == (4, 3)
    assert pick(192, 100, pair=7, quad=3) == (2, 7)  # W % 128 != 0: the quad option is skipped
    assert pick(100, 100, pair=7, quad=3) == (0, 0)
    # explicit depth: plain kernels unless forced
    assert pick(262144, 262144, td=16) == (0, 0)
    assert pick(262144, 262144, quad=5, td=16) == (4, 5)
    assert pick(0, 10) == (0, 0)
