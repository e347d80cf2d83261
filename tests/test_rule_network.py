"""CPU checks of the packed engine's ALGORITHM (not the CUDA code): the
11-op bit-sliced B3/S23 network of csrc/kernels.cuh verified exhaustively
against next_state (grid.cpp:22-28), and a lane-exact numpy model of
packed_tb_kernel (strips of 32 lanes with ghost lanes 0/31, shuffle edge
semantics, wrapped word loads, segmented K-stage row pipeline) checked
against the oracle.  The GPU parity tests then pin the CUDA code itself."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

M32 = np.uint32(0xFFFFFFFF)


def maj(a, b, c):
    return (a & b) | (a & c) | (b & c)


def hsum(xl, x, xr):
    L = ((x << np.uint32(1)) | (xl >> np.uint32(31))) & M32
    R = ((x >> np.uint32(1)) | (xr << np.uint32(31))) & M32
    return L ^ x ^ R, maj(L, x, R)


def lop3(x, y, z, lut):
    """PTX lop3.b32: bit i of the result is bit (x_i << 2 | y_i << 1 | z_i) of lut."""
    out = np.uint32(0)
    for k in range(8):
        if (lut >> k) & 1:
            tx = x if k & 4 else ~x
            ty = y if k & 2 else ~y
            tz = z if k & 1 else ~z
            out |= tx & ty & tz
    return out & M32


def rule(a, b, c, self_):
    t0 = a[0] ^ b[0] ^ c[0]
    k0 = maj(a[0], b[0], c[0])
    p = a[1] ^ b[1] ^ c[1]
    q = maj(a[1], b[1], c[1])
    g1 = lop3(t0, self_, q, 0x53)
    g2 = lop3(p, k0, q, 0x43)
    return lop3(t0, g1, g2, 0x42)


def next_state(alive, n):  # grid.cpp:22-28
    return int(n in (2, 3)) if alive else int(n == 3)


def test_lop3_semantics():
    x, y, z = np.uint32(0xF0F0F0F0), np.uint32(0xCCCCCCCC), np.uint32(0xAAAAAAAA)
    for lut in (0x00, 0x42, 0x43, 0x53, 0x96, 0xE8, 0xFF):
        assert int(lop3(x, y, z, lut)) == lut * 0x01010101


def test_network_exhaustive_512_neighbourhoods():
    # Put each 3x3 neighbourhood at bit 1 of three words (bits 0..2 = columns).
    for bits in range(512):
        cells = [(bits >> i) & 1 for i in range(9)]
        rows = [np.uint32(cells[0] | cells[1] << 1 | cells[2] << 2),
                np.uint32(cells[3] | cells[4] << 1 | cells[5] << 2),
                np.uint32(cells[6] | cells[7] << 1 | cells[8] << 2)]
        z = np.uint32(0)
        hs = [hsum(z, r, z) for r in rows]
        out = rule(hs[0], hs[1], hs[2], rows[1])
        n = sum(cells) - cells[4]
        assert int((out >> np.uint32(1)) & np.uint32(1)) == next_state(cells[4], n), bits


def pack32(g):
    h, w = g.shape
    nw = (w + 31) // 32
    out = np.zeros((h, nw), np.uint32)
    for x in range(w):
        out[:, x // 32] |= (g[:, x].astype(np.uint32) << np.uint32(x % 32))
    return out


def unpack32(p, w):
    cols = [((p[:, x // 32] >> np.uint32(x % 32)) & np.uint32(1)).astype(np.uint8) for x in range(w)]
    return np.stack(cols, axis=1)


def load_word(row, wi, W):
    """load_word_wrapped: 32 cells from column 32*wi of the periodic row."""
    nw = len(row)
    c = (32 * int(wi)) % W
    v, filled = 0, 0
    while filled < 32:
        n = min(W - c, 32 - filled)
        w0 = c >> 5
        lo = int(row[w0])
        hi = int(row[w0 + 1]) if w0 + 1 < nw else 0
        bits = ((hi << 32 | lo) >> (c & 31)) & 0xFFFFFFFF
        if n < 32:
            bits &= (1 << n) - 1
        v |= bits << filled
        filled += n
        c += n
        if c >= W:
            c = 0
    return np.uint32(v & 0xFFFFFFFF)


def seam_word(row, wi, W, junk):
    """make_seam_plan (kernels.cuh): ((A >> sh) & m1) | ((B << s2) & ~m1) from two
    aligned words; words right of nw and left of -1 are don't-care (`junk`)."""
    nw = len(row)
    r = W % 32
    d = 32 - r
    if 0 <= wi < nw - 1:
        return np.uint32(row[wi])
    if wi == nw - 1:
        p0, p1, sh, s2, m1 = nw - 1, 0, 0, r, (1 << r) - 1
    elif wi == nw:
        p0, p1, sh, s2, m1 = 0, 1, d, r, (1 << r) - 1
    elif wi == -1:
        p0, p1, sh, s2, m1 = nw - 2, nw - 1, r, d, (1 << d) - 1
    else:
        return np.uint32(junk)
    lo = int(row[p0]) >> sh
    hi = (int(row[p1]) << s2) & 0xFFFFFFFF
    return np.uint32((lo & m1) | (hi & ~m1 & 0xFFFFFFFF))


def run_segment(p, W, K, strip, y, n, out):
    """One pipeline segment of packed_pass: strip `strip`, output rows y..y+n-1."""
    H, nw = p.shape
    wi = np.arange(32) + strip * 31 - 1
    tail = W % 32
    tail_mask = np.uint32(0xFFFFFFFF if tail == 0 else (1 << tail) - 1)
    lag = 3 * K - 1
    aligned = [(w >= 0 and (w + 1) * 32 <= W) for w in wi]
    seam = W >= 64 and W % 32 != 0 and not all(aligned)   # kPathSeam (else fast / general)
    rng = np.random.default_rng(strip * 7919 + y)
    sa = [(np.zeros(32, np.uint32), np.zeros(32, np.uint32)) for _ in range(K)]
    sb = [(np.zeros(32, np.uint32), np.zeros(32, np.uint32)) for _ in range(K)]
    ss = [np.zeros(32, np.uint32) for _ in range(K)]
    xin = [np.zeros(32, np.uint32) for _ in range(K)]
    for i in range(n + lag):
        r = (y - K + i) % H
        if seam:
            junk = rng.integers(0, 1 << 32, 32)
            xin[0] = np.array([seam_word(p[r], int(w), W, junk[lane]) for lane, w in enumerate(wi)],
                              np.uint32)
        else:
            xin[0] = np.array([p[r, w] if ok else load_word(p[r], w, W)
                               for w, ok in zip(wi, aligned)], np.uint32)
        ys = []
        for g in range(K):  # skewed: stage g eats stage g-1's previous output
            x = xin[g]
            xl = np.concatenate([x[:1], x[:-1]])   # shfl_up: lane 0 keeps own
            xr = np.concatenate([x[1:], x[-1:]])   # shfl_down: lane 31 keeps own
            c = hsum(xl, x, xr)
            ys.append(rule(sa[g], sb[g], c, ss[g]))
            sa[g], sb[g], ss[g] = sb[g], c, x
        for g in range(1, K):
            xin[g] = ys[g - 1]
        j = i - lag
        if 0 <= j < n:
            for lane in range(32):
                w = wi[lane]
                if not (0 <= w < nw):
                    continue
                v = int(ys[K - 1][lane] & (tail_mask if w == nw - 1 else M32))
                cur = int(out[y + j, w])
                if 1 <= lane <= 30:
                    cur = v
                elif lane == 0:   # high half of the word shared with the previous strip
                    cur = (cur & 0xFFFF) | (v & 0xFFFF0000)
                else:             # lane 31: low half
                    cur = (cur & 0xFFFF0000) | (v & 0xFFFF)
                out[y + j, w] = cur


def model_packed_pass(p, W, K, seg_rows):
    """Lane-exact model of packed_tb_kernel<K> over a torus: tiles of one
    strip (32 lanes, strips advancing by 31 words) x seg_rows rows, each a
    fresh pipeline."""
    H, nw = p.shape
    n_strips = -(-(nw + 1) // 31)
    out = np.zeros_like(p)
    for y0 in range(0, H, seg_rows):
        for strip in range(n_strips):
            run_segment(p, W, K, strip, y0, min(seg_rows, H - y0), out)
    return out


@pytest.mark.parametrize("W,H,K,seg", [(3, 3, 1, 1), (5, 7, 3, 4), (31, 9, 4, 5), (33, 17, 16, 6),
                                       (64, 12, 2, 12), (97, 23, 5, 7), (1000, 11, 16, 64),
                                       (1921, 6, 8, 4), (992, 5, 16, 3), (961, 4, 2, 9),
                                       (65, 9, 16, 9), (95, 8, 16, 4), (127, 7, 9, 7),
                                       (2017, 5, 16, 5)])
def test_kernel_model_matches_oracle(oracle, W, H, K, seg):
    g = oracle.random_fill(W, H, 0.45, W * 31 + H)
    p = pack32(g)
    got = unpack32(model_packed_pass(p, W, K, seg), W)
    want, _ = oracle.run(g, K)
    assert np.array_equal(got, want)
