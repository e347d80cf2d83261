"""The NCCL halo exchange (bands.BandDriver) and the neighbour token
(bands.neighbour_token) under the REAL NCCL backend on one GPU: a single rank
that is its own neighbour above and below, so every send matches one of its
own receives.  What a one-GPU box can check of the N > 1 path: the P2POp
batches, their matching order when up == down, and NCCL's stream ordering
around the pass kernels -- bit-exact against the oracle."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_halo_and_token_single_rank():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "nccl_self_worker.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["backend"] == "nccl" and out["world"] == 1
    assert len(out["cases"]) == 5
    for c in out["cases"]:
        assert c["grid"] and c["pops"], c
        assert c["exchange_bytes"] > 0, c   # the halos really went through send / recv
    assert len(out["peer_cases"]) == 10
    for c in out["peer_cases"]:
        assert c["grid"] and c["pops"], c
        assert c["passes"] > 0 or c["case"][5].endswith("_overlap"), c  # (those passes carry no events)
        assert c["sync"] == c["case"][5], c   # NCCL group: the stream-ordered sync, not the host barrier
    assert out["tokens"] == [[1, 1], [2, 2], [3, 3]]
