"""Row-band decomposition with the real CUDA kernels on ONE GPU: P emulated
bands (paper_1209_4408_b200.bands.LocalBands) with device-copy halos must give
the same torus as the single-band engine and the oracle -- band seams, ghost
addressing, interior/edge split, band_bounds remainders."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def words_to_cells(words: np.ndarray, width: int) -> np.ndarray:
    u = np.ascontiguousarray(words).view(np.uint32)
    bits = np.unpackbits(u.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :width].astype(np.uint8)


@pytest.mark.parametrize("W,H,P,depth,gens,overlap", [
    (70, 37, 2, 4, 13, True),
    (1000, 97, 3, 16, 50, True),
    (1000, 97, 3, 16, 50, False),
    (4096, 1025, 8, 16, 100, True),
    (40961, 12289 // 16, 8, 7, 30, True),
    (333, 64, 4, 16, 33, True),
])
def test_local_bands_match_oracle(oracle, W, H, P, depth, gens, overlap):
    import torch
    from paper_1209_4408_b200.bands import LocalBands
    lb = LocalBands(W, H, P, depth, torch.device("cuda", 0), overlap=overlap)
    lb.init_random(0.4, 9)
    lb.run(gens)
    torch.cuda.synchronize()
    got = words_to_cells(lb.gather().cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 9), gens)
    assert np.array_equal(got, want)


@pytest.mark.slow
def test_cfg5_bands_equal_single_gpu_windows(oracle):
    """Config 5 split into 8 emulated bands: windows at every band seam equal
    the reference-generated light-cone goldens."""
    import torch
    from conftest import load_golden
    from paper_1209_4408_b200.bands import LocalBands
    gold = load_golden("golden_cfg5_windows.json")
    W = H = 262144
    lb = LocalBands(W, H, 8, 16, torch.device("cuda", 0))
    lb.init_random(0.4, 42)
    lb.run(16)
    full = lb.gather()
    for w in gold["windows_16"]:
        ys = (np.arange(w["S"]) + w["y0"]) % H
        rows = full[torch.as_tensor(ys, device=full.device)].cpu().numpy()
        cells = words_to_cells(rows, W)
        xs = (np.arange(w["S"]) + w["x0"]) % W
        win = np.ascontiguousarray(cells[:, xs])
        assert f"{oracle.fnv1a64(win):016x}" == w["fnv_bytes"], w
