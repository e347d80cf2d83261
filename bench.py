#!/usr/bin/env python
"""Benchmark of the generation-step hot path (BASELINE.json metric:
cell-updates/s at 1/2/4/8 B200, as a fraction of the int/HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--depth 0=auto]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the reference's own CPU engine
    python bench.py --config 2 --engine byte       # byte engine (HBM-bound)
    python bench.py --config 1 --engine resident   # cluster-resident engine (small tori)

One JSON line on rank 0.  A "step" is one full run of the configuration's
generations (config 5: 500 generations of the 262144^2 torus) over the
row-band decomposition, inputs resident in HBM; `e2e` repeats it through
the public API with the packed grid copied from pinned host memory and back
inside the timed region.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/sec (GCUPS) at 1/2/4/8 B200 and % of HBM/int roofline"
UNIT = "GCUPS"
OPS_PER_WORD = 11            # bit-sliced rule network (2 SHF + 9 LOP3), csrc/kernels.cuh
OPS_PER_UPDATE = OPS_PER_WORD / 32.0
# interleaved layouts (csrc/kernels_pair.cuh): pair = 1 SHF + 9 LOP3 per word,
# quad = 2 SHF + 36 LOP3 per 4 words
IL_OPS_PER_UPDATE = {0: OPS_PER_UPDATE, 2: 10 / 32.0, 4: 9.5 / 32.0}
IL_NAME = {0: "plain", 2: "interleaved-pair", 4: "interleaved-quad"}


def pick_depth(L, args, W: int, rows: int):
    """(depth, il) as life_run picks them for `--depth` / `--pair-depth` /
    `--quad-depth` on a W-wide torus (or band) of `rows` rows
    (life_interleave_auto: the quad or pair layout when forced, or when
    everything is left to the engine and the torus is large; else the
    plain-layout kernels at --depth or life_packed_auto_depth)."""
    import ctypes as C
    d = C.c_int32(0)
    il = int(L.life_interleave_auto(W, rows, args.pair_depth, args.quad_depth, args.depth,
                                    C.byref(d)))
    depth = d.value if il else (args.depth or int(L.life_packed_auto_depth(W, rows)))
    return depth, il


CONFIGS = {
    1: dict(w=1024, h=1024, p=0.5, gens=100,
            desc="cfg1: 1024x1024 torus, p=0.5, seed 42, 100 generations, bit-packed engine"),
    2: dict(w=16384, h=16384, p=0.3, gens=1000,
            desc="cfg2: 16384x16384 torus, p=0.3, seed 42, 1000 generations, bit-packed engine"),
    3: dict(w=65536, h=65536, p=0.5, gens=1000,
            desc="cfg3: 65536x65536 torus (512 MiB packed), p=0.5, seed 42, 1000 generations"),
    4: dict(w=40961, h=12289, p=0.5, gens=5000, soup=True,
            desc="cfg4: 12289 rows x 40961 cols torus, 5x5 Bernoulli(0.5) soups at 2% coverage "
                 "(device-generated, seed 42), 5000 generations, bit-packed engine"),
    5: dict(w=262144, h=262144, p=0.4, gens=500,
            desc="cfg5: 262144x262144 torus (8 GiB packed), p=0.4, seed 42, 500 generations, "
                 "row bands over the GPUs"),
}
L2_BYTES = 126 * 2 ** 20


def set_il_options(eng, args) -> None:
    from paper_1209_4408_b200 import capi
    if args.pair_depth >= 0:
        eng.set_option(capi.OPT_PAIR_DEPTH, args.pair_depth)
    if args.quad_depth >= 0:
        eng.set_option(capi.OPT_QUAD_DEPTH, args.quad_depth)


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def ncu_traffic(config: int, depth, engine: str = ""):
    """dram bytes per launch of the dominant kernel from the committed ncu capture
    (key cfg{config}_k{depth}, byte engine cfg{config}_byte_k{depth})."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"cfg{config}_{engine + '_' if engine else ''}k{depth}")
    except (OSError, ValueError):
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms.  Started
    before the warm-up (nvidia-smi takes ~0.2 s to emit its first sample);
    mark() brackets the timed region and summary() keeps the samples whose
    timestamps fall inside it (the closest ones if the region is shorter
    than the sampling interval)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.window = [None, None]

    def __enter__(self):
        import threading
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                if line.strip():
                    self.lines.append(line)
                    first.set()
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        first.wait(5.0)  # the first sample is out before the measured work starts
        return self

    def mark(self, which: int) -> None:
        self.window[which] = time.time()

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.06)  # one more sample after the region
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)

    def summary(self) -> dict:
        import datetime
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        rows = []
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]), parts[3:7]))
            except ValueError:
                continue
        t0, t1 = self.window
        inside = rows
        if t0 is not None and t1 is not None and rows:
            inside = [r for r in rows if t0 <= r[0] <= t1]
            if not inside:  # region shorter than the interval: the nearest samples
                mid = 0.5 * (t0 + t1)
                inside = sorted(rows, key=lambda r: abs(r[0] - mid))[:2]
        reasons = set()
        for r in inside:
            for n, v in zip(names, r[3]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm = [r[1] for r in inside]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": inside[-1][2] if inside else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "window_s": round(t1 - t0, 3) if t0 and t1 else None}


def blocks_shape(n: int) -> tuple[int, int]:
    m = int(math.sqrt(n))
    while n % m:
        m -= 1
    return n // m, m


# ---------------------------------------------------------------------------
# CPU legs (the reference's own engine, oracle/_ref; else the oracle port)
# ---------------------------------------------------------------------------
def cpu_engine():
    from oracle.oracle import REF_SO, Oracle, Reference
    if os.path.exists(REF_SO):
        return "reference", Reference()
    return "port", Oracle()


def cpu_measure(cfg: dict, budget_s: float,
                variants=("serial", "rows", "cols", "blocks")) -> dict:
    """Times the reference's run() (bench.cpp:77-111 time_run semantics: the
    timer includes run()'s buffer allocation and thread spawn) on a bounded
    sample of the workload: a 8192x8192 torus with the config's density and
    seed, generations sized so all variants together take ~budget_s.  The
    reference's parallel variants are its Strategy::rows / cols / blocks(m,n)
    over std::thread workers = all host threads (it has no OpenMP code,
    SURVEY.md section 0); serial is the single-threaded baseline."""
    kind, eng = cpu_engine()
    threads = os.cpu_count() or 1
    side = min(8192, cfg["w"], cfg["h"])
    if kind != "reference":
        variants = ("serial",)
    share = {v: (0.1 if v == "serial" and len(variants) > 1 else 1.0) for v in variants}
    norm = sum(share.values())
    res = {}
    for var in variants:
        per = budget_s * share[var] / norm
        workers = 1 if var == "serial" else threads
        bx, by = blocks_shape(threads) if var == "blocks" else (1, 1)
        if kind == "reference":
            cal = 4 if var == "serial" else 12
            t1, _, _ = eng.time_run(side, side, cal, var, workers, (bx, by), 42, cfg["p"], 1, 0)
            gens = max(2, int(per / max(t1 / cal, 1e-6)))
            t, _, hw = eng.time_run(side, side, gens, var, workers, (bx, by), 42, cfg["p"], 1, 0)
        else:  # single-threaded C port of compute_region
            g = eng.random_fill(side, side, cfg["p"], 42)
            t0 = time.perf_counter()
            eng.run(g, 1)
            t1 = time.perf_counter() - t0
            gens = max(1, int(per / max(t1, 1e-6)))
            t0 = time.perf_counter()
            eng.run(g, gens)
            t = time.perf_counter() - t0
            workers = 1
        name = f"blocks:{bx}x{by}" if var == "blocks" else var
        res[name] = {"value": side * side * gens / t / 1e9, "seconds": round(t, 3), "gens": gens,
                     "threads": workers}
    best = max(res, key=lambda v: res[v]["value"])
    return {"value": res[best]["value"], "unit": UNIT, "cores": res[best]["threads"], "kind": kind,
            "sample": f"{side}x{side} torus, p={cfg['p']}, seed 42, {res[best]['gens']} generations, "
                      f"best reference variant = {best} x{res[best]['threads']} threads "
                      f"(reference time_run; timer includes allocation + thread spawn)",
            "variants": {k: {"gcups": round(v["value"], 4), "threads": v["threads"],
                             "gens": v["gens"], "seconds": v["seconds"]} for k, v in res.items()},
            "host_threads": threads}


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    kind, eng = cpu_engine()
    threads = os.cpu_count() or 1
    side = min(8192, cfg["w"], cfg["h"])
    bx, by = blocks_shape(threads)
    strategy = "blocks"
    # calibrate so the whole K+W run stays within ~3 minutes, with the fastest
    # of the reference's parallel strategies (rows / cols / blocks) on this box
    if kind == "reference":
        per = {}
        for var in ("rows", "cols", "blocks"):
            t1, _, _ = eng.time_run(side, side, 12, var, threads, (bx, by), 42, cfg["p"], 1, 0)
            per[var] = t1 / 12
        strategy = min(per, key=per.get)
        per_gen = per[strategy]
    else:
        g = eng.random_fill(side, side, cfg["p"], 42)
        t0 = time.perf_counter()
        eng.run(g, 1)
        per_gen = time.perf_counter() - t0
    per_step = min(args.cpu_budget, 170.0 / max(1, args.steps + args.warmup))
    gens = max(1, int(per_step / max(per_gen, 1e-6)))
    times = []
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            t, _, _ = eng.time_run(side, side, gens, strategy, threads, (bx, by), 42, cfg["p"], 1, 0)
        else:
            t0 = time.perf_counter()
            eng.run(g, gens)
            t = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(t)
    total = sum(times)
    value = side * side * gens * len(times) / total / 1e9
    cores = threads if kind == "reference" else 1
    sname = f"blocks:{bx}x{by}" if strategy == "blocks" else strategy
    sample = (f"{side}x{side} torus, p={cfg['p']}, seed 42, {gens} generations per step, "
              f"reference run() strategy {sname} x{cores} threads (fastest of rows / cols / "
              f"blocks on this box)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": cfg["desc"], "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Parity after the timed region: the run is repeated from the initial grid
# and compared with fixtures the REFERENCE generated (tests/golden/, written
# by tests/golden/make_golden.py from oracle/_ref): light-cone windows for
# config 5 (they include the 2/4/8-band seams and the wrap corners), the
# full-grid packed FNV-1a-64 for the others.  Only the committed JSON is read
# here; nothing under oracle/ is imported.
# ---------------------------------------------------------------------------
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def golden_for(config: int, gens: int):
    def load(name):
        try:
            with open(os.path.join(GOLDEN_DIR, name)) as f:
                return json.load(f)
        except OSError:
            return None
    if config == 5:
        g = load("golden_cfg5_windows.json")
        if g:
            for key in ("windows_500", "windows_16"):
                ws = [w for w in g.get(key, []) if w["T"] == gens]
                if ws:
                    return {"kind": "windows", "windows": ws, "source": "golden_cfg5_windows.json"}
        return None
    name = {1: "golden_small.json", 2: "golden_cfg2.json", 3: "golden_cfg3.json",
            4: "golden_cfg4.json"}[config]
    g = load(name)
    if g is None:
        return None
    sched = g["cfg1"] if config == 1 else g["gens"]
    if str(gens) in sched:
        return {"kind": "hash", "fnv_packed": sched[str(gens)]["fnv_packed"],
                "population": sched[str(gens)]["population"], "source": name}
    return None


def band_window_rows(band, y0b: int, H: int, W: int, x0: int, y0: int, S: int) -> dict:
    """Rows of the wrapped S x S window at (x0, y0) (Grid::wrap, grid.hpp:48-54)
    that lie in this band ([y0b, y0b + rows) of the torus), as 0/1 bytes keyed
    by window row; `band` is the band's packed uint32 rows on the device."""
    import numpy as np
    import torch
    rows = (y0 + np.arange(S)) % H
    sel = np.nonzero((rows >= y0b) & (rows < y0b + band.shape[0]))[0]
    if not len(sel):
        return {}
    cols = (x0 + np.arange(S)) % W
    widx = np.unique(cols // 32)
    ri = torch.as_tensor(rows[sel] - y0b, device=band.device)
    wi = torch.as_tensor(widx, device=band.device)
    sub = band.index_select(0, ri).index_select(1, wi).cpu().numpy().view(np.uint32)
    pos = np.searchsorted(widx, cols // 32)
    bits = ((sub[:, pos] >> (cols % 32).astype(np.uint32)) & 1).astype(np.uint8)
    return {int(i): bits[j].tobytes() for j, i in enumerate(sel)}


def fnv(data: bytes, h: int = 0) -> int:
    from paper_1209_4408_b200 import capi
    return int(capi.lib().life_fnv1a64(data, len(data), h))


def check_windows(gold: dict, rows_of) -> dict:
    """rows_of(x0, y0, S) -> {window row: bytes} for the whole window."""
    bad = []
    for w in gold["windows"]:
        rows = rows_of(w["x0"], w["y0"], w["S"])
        data = b"".join(rows[i] for i in range(w["S"]))
        got = f"{fnv(data):016x}"
        pop = sum(data)
        if got != w["fnv_bytes"] or pop != w["population"]:
            bad.append({"x0": w["x0"], "y0": w["y0"], "got": got, "want": w["fnv_bytes"]})
    return {"ok": not bad, "kind": f"{len(gold['windows'])} light-cone windows "
                                    f"{gold['windows'][0]['S']}^2 at T={gold['windows'][0]['T']}",
            "mismatches": bad}


def parity_bands(drv, geo, cfg: dict, config: int, gens: int, world: int, rank: int,
                 soup_host) -> dict:
    """Re-runs the configuration on the band driver(s) from the initial grid
    and compares with the reference-generated golden fixture."""
    import torch
    import torch.distributed as dist
    gold = golden_for(config, gens)
    if gold is None:
        return {"ok": None, "reason": f"no reference golden for config {config} at {gens} generations"}
    if soup_host is not None:
        drv.load_rows(soup_host)
    else:
        drv.init_random(cfg["p"], 42)
    drv.run(gens)
    torch.cuda.synchronize()
    band = drv.band()
    W, H = geo.width, geo.height
    if gold["kind"] == "windows":
        mine = {(w["x0"], w["y0"]): band_window_rows(band, geo.y0, H, W, w["x0"], w["y0"], w["S"])
                for w in gold["windows"]}
        if world > 1:
            allp = [None] * world
            dist.all_gather_object(allp, mine)
            merged = {}
            for part in allp:
                for key, rows in part.items():
                    merged.setdefault(key, {}).update(rows)
        else:
            merged = mine
        res = check_windows(gold, lambda x0, y0, S: merged[(x0, y0)]) if rank == 0 else {}
    else:
        # fnv_packed: FNV-1a-64 over the packed exchange format (rows of
        # ceil(W/64) little-endian uint64), chained band by band in row order.
        wpr = -(-W // 64)
        data = band[:, :2 * wpr].contiguous().cpu().numpy().tobytes()
        cdev = band.device if world > 1 and dist.get_backend() == "nccl" else torch.device("cpu")

        def as_t(v):  # uint64 hash state in an int64 tensor
            return torch.tensor([v - (1 << 64) if v >= 1 << 63 else v], dtype=torch.int64,
                                device=cdev)
        h = as_t(0)
        if rank > 0:
            dist.recv(h, rank - 1)
        hv = fnv(data, int(h.item()) & (2 ** 64 - 1))
        if rank + 1 < world:
            dist.send(as_t(hv), rank + 1)
        if world > 1:  # the last band holds the whole-grid hash
            t = as_t(hv)
            dist.broadcast(t, world - 1)
            hv = int(t.item()) & (2 ** 64 - 1)
        pop = drv.population()
        got = f"{hv:016x}"
        res = {"ok": got == gold["fnv_packed"] and pop == gold["population"],
               "kind": "full-grid packed FNV-1a-64 + population", "got": got,
               "want": gold["fnv_packed"], "population": pop}
    res["source"] = "tests/golden/" + gold["source"] + " (written by the reference, oracle/_ref)"
    res["generations"] = gens
    return res


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_gpu_arm(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_1209_4408_b200 import capi
    from paper_1209_4408_b200.bands import BandDriver, make_geometry
    from paper_1209_4408_b200.life import Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # LIFE_BENCH_DEVICE / LIFE_BENCH_BACKEND exist for the single-GPU test of
    # the multi-rank path (ranks sharing cuda:0 over gloo, host barriers only,
    # so no kernel ever waits on another rank): tests/test_bench_contract.py.
    emulated = bool(os.environ.get("LIFE_BENCH_DEVICE"))
    if emulated:
        local = int(os.environ["LIFE_BENCH_DEVICE"])
    elif torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} CUDA "
                         f"device(s) visible -- refusing to measure fewer GPUs than requested")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("LIFE_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        # Communicator evidence for the log: every rank names its GPU.
        props = torch.cuda.get_device_properties(dev)
        print(f"[bench rank {rank}/{dist.get_world_size()}] backend {dist.get_backend()} "
              f"cuda:{local} {props.name} pci {getattr(props, 'pci_bus_id', '?')} "
              f"uuid {getattr(props, 'uuid', '?')}", file=sys.stderr, flush=True)
    L = capi.lib()
    cfg = CONFIGS[args.config]
    W, H, gens = cfg["w"], cfg["h"], args.gens or cfg["gens"]
    bounds0 = [H * r // world for r in range(world + 1)]
    band_rows_max = max(b - a for a, b in zip(bounds0, bounds0[1:])) + 1
    # depth 0: the engine's own auto rule (life_interleave_auto / life_packed_auto_depth)
    depth, il = pick_depth(L, args, W, H if world == 1 else band_rows_max)
    ops_per_update = IL_OPS_PER_UPDATE[il]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    int_ops = 0.0
    import ctypes as C
    o, s = C.c_double(), C.c_double()
    if L.life_measure_int_peak(local, 4000, C.byref(o), C.byref(s)) == 0:
        int_ops = o.value

    geo = make_geometry(W, H, rank, world, depth, il)
    # Per-launch CUDA events are recorded only in one extra PROFILED step after
    # the timed region (events between launches serialise programmatic
    # dependent launch, so the timed steps carry none).
    launches = []
    from paper_1209_4408_b200.bands import cuda_stepper
    base_step = cuda_stepper(W, il)
    record = {"on": False}

    def timed_step(inp, in_row0, in_rows, out, out_row0, out_rows, k):
        if record["on"]:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            base_step(inp, in_row0, in_rows, out, out_row0, out_rows, k)
            e1.record()
            launches.append((e0, e1, out_rows * W * k, k, out_rows))
        else:
            base_step(inp, in_row0, in_rows, out, out_row0, out_rows, k)

    halo = "none" if world == 1 else args.halo
    drv = None
    peer = False
    if halo == "peer":
        # Fused halo: the pass kernels read the neighbour bands' rows over
        # NVLink (CUDA IPC); a neighbour-only NCCL token orders the passes.
        from paper_1209_4408_b200.bands import PeerBandDriver
        err = None
        try:
            drv = PeerBandDriver(geo, dev, sync=args.pass_sync)
        except Exception as exc:  # no IPC / peer access on this rank
            err, drv = exc, None
        # Collective decision: every rank falls back if any rank could not open
        # its neighbours' buffers (mixed halo schemes would deadlock).
        ok = torch.tensor([0 if drv is None else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            if drv is not None:
                drv.close()
            drv = None
            print(f"peer halo unavailable on some rank ({err!r}); using NCCL send/recv",
                  file=sys.stderr)
            halo = "nccl"
        else:
            peer = True
    torus = None
    if drv is None and world == 1:
        # One GPU: the whole torus, one life_dev_packed_run per step.
        from paper_1209_4408_b200.bands import TorusDriver
        drv = torus = TorusDriver(geo, dev)
    elif drv is None:
        drv = BandDriver(geo, dev, stepper=timed_step)
    soup_host = None
    if cfg.get("soup"):
        with Engine(local) as e:  # device soup, shared by every rank's band
            e.init_soup(W, H, 0.02, 5, cfg["p"], 42, capi.ENGINE_PACKED)
            soup_host = e.download_packed()
        drv.load_rows(soup_host)
    else:
        drv.init_random(cfg["p"], 42)
    grid_bytes = H * math.ceil(W / 64) * 8
    flush = None
    if grid_bytes * 2 < 4 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)

    clocks = ClockSampler(local).__enter__()  # running through warm-up and timed steps
    for _ in range(args.warmup):
        drv.run(gens)
    barrier()
    step_ms = []
    l0 = L.life_kernel_launches()
    clocks.mark(0)
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        drv.run(gens)
        e1.record()
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    clocks.mark(1)
    clocks.__exit__(None, None, None)
    gpu_launches = int(L.life_kernel_launches() - l0)
    barrier()
    total_ms = max_over_ranks(sum(step_ms))
    cells = W * H * gens * args.steps
    value = cells / (total_ms * 1e-3) / 1e9

    # ---- one profiled step: per-launch events on the launching stream ----
    if flush is not None:
        flush.fill_(1)
    barrier()
    record["on"] = True
    if peer:
        drv.profile = True
    if torus is not None:
        def on_launch(kind, g, fn):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            n = g // depth if kind == "full" else 1  # kernel passes inside the call
            launches.append((e0, e1, H * W * g, depth if kind == "full" else g, H, n))
        torus.on_launch = on_launch
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record()
    drv.run(gens)
    p1.record()
    torch.cuda.synchronize()
    record["on"] = False
    prof_ms = p0.elapsed_time(p1)
    rank_stats = {"rank": rank, "device": local, "y0": geo.y0, "rows": geo.band_rows,
                  "timed_ms": sum(step_ms), "profiled_step_ms": prof_ms}
    if peer:
        drv.profile = False
        st = drv.stats()
        # the interior launch of each full-depth pass is the dominant kernel
        rank_stats.update({"interior_ms": st["interior_ms"], "pass_ms": st["pass_ms"],
                           "barrier_ms": st["barrier_ms"], "passes": st["passes"],
                           "pass_sync": drv.sync})
        n_full = sum(1 for k in st["ks"] if k == depth)
        kern_ms = st["interior_full_ms"]
        kern_cells = n_full * (geo.band_rows - 2 * depth if geo.band_rows > 2 * depth
                               else geo.band_rows) * W * depth
        all_kern_ms = st["interior_ms"]
        n_main = max(n_full, 1)
    else:
        if torus is not None:
            torus.on_launch = None
        launches[:] = [x if len(x) == 6 else (*x, 1) for x in launches]
        full = max((r for (_, _, _, k, r, _) in launches if k == depth), default=0)
        main = [(a.elapsed_time(b), n, m) for (a, b, n, k, r, m) in launches
                if k == depth and r == full]
        kern_ms = sum(t for t, _, _ in main)
        kern_cells = sum(n for _, n, _ in main)
        all_kern_ms = sum(a.elapsed_time(b) for (a, b, _, _, _, _) in launches)
        n_main = max(sum(m for _, _, m in main), 1)
        rank_stats.update({"interior_ms": kern_ms, "kernel_ms": all_kern_ms,
                           "launches": len(launches)})
        if world > 1:
            rank_stats["halo_wait_ms"] = prof_ms - all_kern_ms
    launches.clear()
    if world > 1:
        allst = [None] * world
        dist.all_gather_object(allst, rank_stats)
    else:
        allst = [rank_stats]

    achieved_ops = kern_cells * ops_per_update / (kern_ms * 1e-3) if kern_ms else 0.0
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    alg_bytes_per_update = 0.25 / depth
    hbm_achieved = kern_cells * alg_bytes_per_update / (kern_ms * 1e-3) / 1e9 if kern_ms else 0.0
    traffic = ncu_traffic(args.config, depth, {0: "", 2: "pair", 4: "quad"}[il])
    kind = -2 if il else int(L.life_packed_launch_kind(W, geo.band_rows if world > 1 else H,
                                                       depth))
    kname = {-2: f"packed_il_kernel<{depth}, {il}>",
             capi.LAUNCH_STEP1: "packed_step1_kernel",
             capi.LAUNCH_FAST: f"packed_tb_fast_kernel<{depth}>",
             capi.LAUNCH_ALL_PATHS: f"packed_tb_kernel<{depth}>",
             capi.LAUNCH_SPLIT: f"split: packed_tb_fast_kernel<{depth}> (inner strips) + "
                                f"packed_tb_kernel<{depth}> (seam strips, side stream)"}.get(kind, "?")
    step1 = kind == capi.LAUNCH_STEP1
    roofline = {
        "bound": "int",
        "kernel": kname,
        "achieved": achieved_ops / 1e12, "peak": int_ops / 1e12, "unit": "Tops/s",
        "frac": achieved_ops / int_ops if int_ops else None,
        "peak_source": "measured (life_measure_int_peak: LOP3 throughput, all SMs, this run)",
        "ops_per_cell_update": ops_per_update,
        "algorithmic_per_launch": {"cell_updates": kern_cells / n_main,
                                   "int_ops": kern_cells / n_main * ops_per_update,
                                   "hbm_bytes": kern_cells / n_main * alg_bytes_per_update},
        "mean_launch_ms": kern_ms / n_main,
        "timing": "per-launch CUDA events on the launching stream over one profiled step "
                  "right after the timed steps (same work; the timed steps carry no "
                  "per-launch events, which would serialise programmatic dependent launch)",
        "kernel_share_of_step": all_kern_ms / prof_ms if prof_ms else None,
        "step_frac": (value * 1e9 * ops_per_update / world) / int_ops if int_ops else None,
        "traffic": traffic,
        "hbm": {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_achieved / hbm_peak, "bytes_per_cell_update": alg_bytes_per_update,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"},
        "roofline_updates_per_s": min(int_ops / ops_per_update if int_ops else float("inf"),
                                      hbm_peak * 1e9 / alg_bytes_per_update),
    }
    if step1:
        roofline.update({"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak,
                         "unit": "GB/s", "frac": hbm_achieved / hbm_peak,
                         "peak_source": roofline["hbm"]["peak_source"],
                         "int": {"achieved": achieved_ops / 1e12, "peak": int_ops / 1e12,
                                 "unit": "Tops/s",
                                 "frac": achieved_ops / int_ops if int_ops else None}})

    # ---- parity: the same run again, against the reference's golden -------
    parity = {"ok": None, "reason": "--no-parity"}
    if not args.no_parity:
        parity = parity_bands(drv, geo, cfg, args.config, gens, world, rank, soup_host)
    if hasattr(drv, "close"):
        drv.close()
    del drv
    torch.cuda.empty_cache()

    # ---- e2e through the public API, host buffers ------------------------
    e2e = None
    if not args.no_e2e:
        steps_e2e = max(2, args.steps)
        if world == 1:
            # life_run_batch: every step uploads its packed grid from pinned
            # memory, runs the generations and downloads the result; step i's
            # copies overlap step i+-1's compute (copy engines).
            eng = Engine(local)
            set_il_options(eng, args)
            api_depth = args.depth  # 0: the engine's auto rule (the same choice as `depth`)
            wpr = math.ceil(W / 64)
            host_in = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True)
            host_out = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True)
            if soup_host is not None:
                eng.upload_packed(soup_host, W)
            else:
                eng.init_random(W, H, cfg["p"], 42, capi.ENGINE_PACKED)
            hin = host_in.numpy().view("uint64")
            hout = host_out.numpy().view("uint64")
            eng.download_packed(hin)
            eng.run_batch([hin], [hout], W, gens, api_depth)  # warm-up (allocates buffers)
            e2e_ms = eng.run_batch([hin] * steps_e2e, [hout] * steps_e2e, W, gens, api_depth)
            # Drop-in latency: one synchronous run() per call -- upload, run,
            # download, nothing overlapped across calls (what lifegpu::run
            # does for one caller), host-timed.
            eng.upload_packed(hin, W)
            eng.run(gens, capi.ENGINE_PACKED, api_depth)
            eng.download_packed(hout)
            sync_s = []
            for _ in range(steps_e2e):
                t0 = time.perf_counter()
                eng.upload_packed(hin, W)
                eng.run(gens, capi.ENGINE_PACKED, api_depth)
                eng.download_packed(hout)
                sync_s.append(time.perf_counter() - t0)
            # The same single-grid call through life_run_batch(n = 1): its
            # trapezoid schedule overlaps the grid's own upload and download
            # with the first and last passes.
            one_s = []
            for _ in range(steps_e2e):
                t0 = time.perf_counter()
                eng.run_batch([hin], [hout], W, gens, api_depth)
                one_s.append(time.perf_counter() - t0)
            eng.close()
            bi = bo = H * wpr * 8
            sync = {"value": W * H * gens / statistics.median(sync_s) / 1e9, "unit": UNIT,
                    "ms_per_call": 1e3 * statistics.median(sync_s),
                    "api": "C-ABI life_grid_upload_packed + life_run + life_grid_download_packed "
                           "per call from/to pinned host memory, serial (drop-in latency; "
                           "host-timed median)",
                    "one_grid_batch": {
                        "value": W * H * gens / statistics.median(one_s) / 1e9, "unit": UNIT,
                        "ms_per_call": 1e3 * statistics.median(one_s),
                        "api": "C-ABI life_run_batch with n = 1 (the grid's own copies overlap "
                               "its first / last passes; host-timed median)"}}
        else:
            e2e_ms, bi, bo = e2e_bands(args, geo, dev, halo, cfg, gens, soup_host, steps_e2e,
                                       barrier, max_over_ranks)
            sync = None
        e2e = {"value": W * H * gens * steps_e2e / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
               "api": "C-ABI life_run_batch (per step: H2D packed grid, run, D2H; copies "
                      "overlapped with the neighbouring steps' compute)"
                      if world == 1 else
                      "band driver per rank: pinned-host band upload / run / download, "
                      "copies overlapped with the neighbouring steps' compute",
               "steps": steps_e2e}
        if sync:
            e2e["sync_call"] = sync

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_measure(cfg, args.cpu_budget)
        except Exception as exc:  # reported, not fatal
            cpu = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "u32 bit-sliced (32 cells/word, exact integer)", "data": "synthetic",
            "config": {"workload": cfg["desc"], "width": W, "height": H, "generations": gens,
                       "temporal_depth": depth, "layout": IL_NAME[il],
                       "global_cells": W * H,
                       "parallelism": f"rowbands{world}" if world > 1 else "single-gpu",
                       "halo": {"peer": "in-kernel NVLink peer reads (CUDA IPC) + "
                                        f"{args.pass_sync} pass ordering",
                                "nccl": "NCCL send/recv of k ghost rows, interior overlapped",
                                "none": "torus wraps inside the kernel"}[halo],
                       "emulated_ranks_on_one_gpu": emulated,
                       "l2": ("inputs larger than L2" if flush is None else
                              "L2 flushed (256 MiB write) between steps")},
            "roofline": roofline,
            "parity": parity,
            "ranks": allst,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    ok = parity.get("ok") is not False
    if world > 1:
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = bool(t.item())
        dist.destroy_process_group()
    if not ok:
        print("bench.py: PARITY MISMATCH against the reference golden", file=sys.stderr)
        sys.exit(3)


def e2e_bands(args, geo, dev, halo, cfg, gens, soup_host, steps_e2e, barrier, max_over_ranks):
    """N > 1 e2e: each rank uploads its band from pinned host memory, runs,
    downloads; step i's copies overlap step i+-1's compute."""
    import torch
    import torch.distributed as dist

    from paper_1209_4408_b200.bands import BandDriver, PeerBandDriver
    if halo == "peer":
        drv = PeerBandDriver(geo, dev, sync=args.pass_sync)
    else:
        drv = BandDriver(geo, dev)
    host = torch.empty(tuple(drv.band().shape), dtype=torch.int32, pin_memory=True)
    if soup_host is not None:
        drv.load_rows(soup_host)
    else:
        drv.init_random(cfg["p"], 42)
    host.copy_(drv.band())
    # Step i's band upload (pinned host -> staging buffer) and step i-1's
    # download (staging -> pinned host) run on a copy stream while the band
    # computes; the band itself is only touched by two on-device copies per
    # step.  Timed from the first upload to the last download, max over ranks.
    stage_in = torch.empty_like(drv.band())
    stage_out = torch.empty_like(drv.band())
    copy = torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)
    up_done = [torch.cuda.Event() for _ in range(steps_e2e)]
    e2e_ms = 0.0
    for warm in (True, False):
        n_steps = 1 if warm else steps_e2e
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        copy.wait_stream(main)
        with torch.cuda.stream(copy):
            stage_in.copy_(host, non_blocking=True)
            up_done[0].record(copy)
        for i in range(n_steps):
            main.wait_event(up_done[i])
            drv.set_band(stage_in)              # on-device, after upload i
            if i + 1 < n_steps:                 # upload i+1 overlaps compute i
                copy.wait_stream(main)
                with torch.cuda.stream(copy):
                    stage_in.copy_(host, non_blocking=True)
                    up_done[i + 1].record(copy)
            drv.run(gens)
            stage_out.copy_(drv.band())         # on-device
            copy.wait_stream(main)
            with torch.cuda.stream(copy):       # download i overlaps compute i+1
                host.copy_(stage_out, non_blocking=True)
        main.wait_stream(copy)
        e1.record()
        torch.cuda.synchronize()
        if not warm:
            e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    del stage_in, stage_out
    t = torch.tensor([host.numel() * 4], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    if hasattr(drv, "close"):
        drv.close()
    return e2e_ms, int(t.item()), int(t.item())


def run_ctx_arm(args) -> None:
    """--single-process: ONE process drives all N GPUs through the multi-device
    C-ABI context (life_ctx_create_multi: row bands by band_bounds, in-kernel
    NVLink halos, neighbour-only event ordering) -- the drop-in run() of the
    reference over N workers (engine.cpp:162-214).  Time = max over the bands
    of the CUDA-event time on each band's device (life_band_stats.run_ms)."""
    import torch

    from paper_1209_4408_b200 import capi
    from paper_1209_4408_b200.life import Engine
    n = args.gpus
    emulated = bool(os.environ.get("LIFE_BENCH_DEVICE"))
    if emulated:
        devices = [int(os.environ["LIFE_BENCH_DEVICE"])] * n
    else:
        if torch.cuda.device_count() < n:
            raise SystemExit(f"bench.py: --gpus {n} but only {torch.cuda.device_count()} CUDA "
                             f"device(s) visible")
        devices = list(range(n))
    L = capi.lib()
    cfg = CONFIGS[args.config]
    W, H, gens = cfg["w"], cfg["h"], args.gens or cfg["gens"]
    import ctypes as C
    o, s = C.c_double(), C.c_double()
    int_ops = o.value if L.life_measure_int_peak(devices[0], 4000, C.byref(o), C.byref(s)) == 0 \
        else 0.0
    e = Engine(devices=devices)
    set_il_options(e, args)

    def init():
        if cfg.get("soup"):
            e.init_soup(W, H, 0.02, 5, cfg["p"], 42, capi.ENGINE_PACKED)
        else:
            e.init_random(W, H, cfg["p"], 42, capi.ENGINE_PACKED)
    init()
    b = e.bands()
    depth = args.depth or 0
    clocks = ClockSampler(devices[0]).__enter__()  # running through warm-up and timed steps
    for _ in range(args.warmup):
        e.run(gens, capi.ENGINE_PACKED, depth)
    l0 = L.life_kernel_launches()
    ms = []
    clocks.mark(0)
    for _ in range(args.steps):
        e.run(gens, capi.ENGINE_PACKED, depth)
        ms.append(max(st["run_ms"] for st in e.band_stats()))
    clocks.mark(1)
    clocks.__exit__(None, None, None)
    gpu_launches = int(L.life_kernel_launches() - l0)
    e.set_option(capi.OPT_PROFILE, 1)
    e.run(gens, capi.ENGINE_PACKED, depth)
    stats = e.band_stats()
    e.set_option(capi.OPT_PROFILE, 0)
    value = W * H * gens * args.steps / (sum(ms) * 1e-3) / 1e9
    parity = {"ok": None, "reason": "--no-parity"}
    gold = None if args.no_parity else golden_for(args.config, gens)
    if not args.no_parity and gold is None:
        parity = {"ok": None, "reason": f"no reference golden for config {args.config} at {gens}"}
    elif gold is not None:
        init()
        e.run(gens, capi.ENGINE_PACKED, depth)
        if gold["kind"] == "windows":
            parity = check_windows(gold, lambda x0, y0, S: {
                i: r.tobytes() for i, r in enumerate(e.window(x0, y0, S, S))})
        else:
            got = f"{fnv(e.download_packed().tobytes()):016x}"
            pop = e.population()
            parity = {"ok": got == gold["fnv_packed"] and pop == gold["population"],
                      "kind": "full-grid packed FNV-1a-64 + population", "got": got,
                      "want": gold["fnv_packed"], "population": pop}
        parity["source"] = "tests/golden/" + gold["source"]
    e2e = None
    if not args.no_e2e:
        # life_run_batch on the multi-device context: every step's packed grid
        # from pinned host memory to the bands and back, copies overlapped with
        # the neighbouring steps' compute; CUDA-event time (life_run_batch's
        # elapsed_ms, max over the bands' devices).
        wpr = (W + 63) // 64
        hin = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True).numpy().view("uint64")
        hout = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True).numpy().view("uint64")
        init()
        e.download_packed(hin)
        steps_e2e = max(2, args.steps)
        e.run_batch([hin], [hout], W, gens, depth)  # warm-up (allocates buffers)
        e2e_ms = e.run_batch([hin] * steps_e2e, [hout] * steps_e2e, W, gens, depth)
        e2e = {"value": W * H * gens * steps_e2e / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": H * wpr * 8, "d2h_bytes_per_step": H * wpr * 8,
               "api": "C-ABI life_run_batch on the multi-device context (per step: H2D of "
                      "every band, run, D2H; copies overlapped with the neighbouring steps)",
               "steps": steps_e2e}
    e.close()
    eff_depth, il = pick_depth(L, args, W, max(y - x for x, y in zip(b["bounds"], b["bounds"][1:])))
    ops_per_update = IL_OPS_PER_UPDATE[il]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sum(ms) / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "u32 bit-sliced (32 cells/word, exact integer)", "data": "synthetic",
        "config": {"workload": cfg["desc"], "width": W, "height": H, "generations": gens,
                   "temporal_depth": eff_depth,
                   "layout": IL_NAME[il],
                   "parallelism": f"rowbands{n} (one process, "
                   "multi-device C-ABI context)", "devices": devices,
                   "bounds": b["bounds"], "halo": {0: "peer", 1: "copy"}.get(b["halo"], "none"),
                   "emulated_ranks_on_one_gpu": emulated},
        "roofline": {"bound": "int", "achieved": value * 1e9 * ops_per_update / n / 1e12,
                     "peak": int_ops / 1e12, "unit": "Tops/s",
                     "ops_per_cell_update": ops_per_update,
                     "frac": value * 1e9 * ops_per_update / n / int_ops if int_ops else None,
                     "basis": "whole step per GPU (band_stats run_ms, max over bands)",
                     "traffic": None},
        "parity": parity, "bands": stats, "cpu_baseline": None, "e2e": e2e,
        "gpu_launches": gpu_launches, "clocks": clocks.summary()}
    print(json.dumps(line), flush=True)
    if parity.get("ok") is False:
        print("bench.py: PARITY MISMATCH against the reference golden", file=sys.stderr)
        sys.exit(3)


def self_launch(args) -> int:
    """`python bench.py --gpus N` without torchrun: refuse if fewer than N
    GPUs are visible, else re-run this command as N ranks under
    torch.distributed.run (one process per GPU)."""
    if not os.environ.get("LIFE_BENCH_DEVICE"):
        try:
            import torch
            n = torch.cuda.device_count()
        except Exception:  # noqa: BLE001
            n = 0
        if n < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {n} CUDA device(s) visible -- "
                  f"refusing to measure fewer GPUs than requested", file=sys.stderr)
            return 2
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


# byte_tb2_kernel per 32-bit word = 4 columns x 2 row streams = 8 cell-updates
# (csrc/kernels.cuh byte_row_fma / nib_rule): ALU pipe -- 2 funnel shifts, n & 7,
# (n|x)^3, ~y & m, >>3; FMA pipe (IMAD a*one+b) -- the adds hn, h, the two
# vertical adds and +0x77777777.  (Round 1's one-stream byte_tb_kernel: 5 + 5
# per 4 cells.)
BYTE_ALU_OPS_PER_UPDATE = 6 / 8.0
BYTE_FMA_OPS_PER_UPDATE = 5 / 8.0


def byte_roofline(cell_updates: float, k: int, kern_ms: float, hbm_peak: float, int_ops: float,
                  traffic) -> dict:
    """Roofline of one byte-engine pass of depth k: HBM-bound at k = 1 (2 B per
    cell-update); for k >= 2 instruction-bound: 0.75 ALU-pipe + 0.625 FMA-pipe
    ops per cell-update (two row streams per word), each pipe at the measured
    LOP3 lane rate P and one instruction issued per cycle per sub-partition:
    the ALU pipe binds: achieved = ALU-pipe ops/s of the kernel, peak = P,
    bound P / 0.75 cell-updates/s."""
    t = kern_ms * 1e-3
    hbm = {"achieved": 2.0 / k * cell_updates / t / 1e9, "peak": hbm_peak, "unit": "GB/s",
           "bytes_per_cell_update": 2.0 / k}
    hbm["frac"] = hbm["achieved"] / hbm_peak
    if k == 1 or not int_ops:
        return {"bound": "hbm", "kernel": "byte_step_kernel" if k == 1 else f"byte_tb2_kernel<{k}>",
                **hbm, "mean_launch_ms": kern_ms, "traffic": traffic}
    ops = BYTE_ALU_OPS_PER_UPDATE + BYTE_FMA_OPS_PER_UPDATE
    ach = cell_updates * BYTE_ALU_OPS_PER_UPDATE / t / 1e12
    peak = int_ops / 1e12
    return {"bound": "int", "kernel": f"byte_tb2_kernel<{k}>", "achieved": ach, "peak": peak,
            "unit": "Tops/s", "frac": ach / peak, "ops_per_cell_update": ops,
            "alu_ops_per_cell_update": BYTE_ALU_OPS_PER_UPDATE,
            "fma_ops_per_cell_update": BYTE_FMA_OPS_PER_UPDATE,
            "peak_source": "measured LOP3 lane rate (the ALU pipe, which binds)",
            "roofline_updates_per_s": int_ops / BYTE_ALU_OPS_PER_UPDATE,
            "issue_frac": cell_updates * ops / t / (2 * int_ops),
            "vs_one_stream_bound": cell_updates / t / (int_ops / 1.25),
            "hbm": hbm, "mean_launch_ms": kern_ms, "traffic": traffic}


def run_byte_arm(args) -> None:
    """The byte engine (one generation per pass, 2 B of HBM per cell-update)
    on one GPU: config's grid, per-launch CUDA events, HBM roofline."""
    import torch

    from paper_1209_4408_b200 import capi
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "unavailable": "byte engine is single-GPU"}))
        return
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L = capi.lib()
    cfg = CONFIGS[args.config]
    W, H, gens = cfg["w"], cfg["h"], args.gens or cfg["gens"]
    pitch = int(L.life_byte_pitch(W))
    if 2 * pitch * H > 120e9:
        print(json.dumps({"metric": METRIC, "unavailable": "grid too large for the byte layout"}))
        return
    bufs = [torch.zeros((H, pitch), dtype=torch.uint8, device=dev) for _ in range(2)]
    stream = torch.cuda.current_stream(dev).cuda_stream
    from paper_1209_4408_b200.life import check
    def init_grid(buf):
        if cfg.get("soup"):  # config 4: the device soup, byte layout
            from paper_1209_4408_b200.life import Engine
            with Engine(0) as e:
                e.init_soup(W, H, 0.02, 5, cfg["p"], 42, capi.ENGINE_BYTE)
                cells = e.download()
            buf[:, :W].copy_(torch.from_numpy(cells))
        else:
            check(L.life_dev_byte_random(buf.data_ptr(), pitch, W, 0, H, cfg["p"], 42, stream))
    init_grid(bufs[0])
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if 2 * pitch * H < 4 * L2_BYTES else None
    launches = []
    cur = [0]

    depth = args.byte_depth or (8 if W * H >= 2 ** 26 else 4)  # life_run's byte auto rule
    if W % 16 and W < 33:
        depth = 1

    def step(record: bool):
        done = 0
        while done < gens:
            k = min(depth, gens - done)
            a, b = bufs[cur[0]], bufs[cur[0] ^ 1]
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            check(L.life_dev_byte_pass(a.data_ptr(), pitch, 0, H, b.data_ptr(), pitch, 0, W, H, k,
                                       stream))
            if record:
                e1.record()
                launches.append((e0, e1, k))
            cur[0] ^= 1
            done += k

    clocks = ClockSampler(0).__enter__()  # running through warm-up and timed steps
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    l0 = L.life_kernel_launches()
    ms = []
    clocks.mark(0)
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step(False)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    clocks.mark(1)
    clocks.__exit__(None, None, None)
    n_launch = int(L.life_kernel_launches() - l0)
    # One profiled step after the timed ones: per-launch events (they would
    # serialise programmatic dependent launch inside the timed steps).
    if flush is not None:
        flush.fill_(1)
    torch.cuda.synchronize()
    step(True)
    torch.cuda.synchronize()
    # Parity: the configuration again from the initial grid, against the
    # reference's golden (FNV-1a-64 over the W*H 0/1 bytes).
    parity = {"ok": None, "reason": "--no-parity"}
    gold = None if args.no_parity else golden_for(args.config, gens)
    if gold is not None and gold["kind"] == "hash":
        with open(os.path.join(GOLDEN_DIR, gold["source"])) as f:
            gj = json.load(f)
        want = (gj["cfg1"] if args.config == 1 else gj["gens"])[str(gens)]
        init_grid(bufs[cur[0]])
        step(False)
        torch.cuda.synchronize()
        got = f"{fnv(bufs[cur[0]][:, :W].contiguous().cpu().numpy().tobytes()):016x}"
        parity = {"ok": got == want["fnv_bytes"], "kind": "full-grid byte FNV-1a-64",
                  "got": got, "want": want["fnv_bytes"], "generations": gens,
                  "source": "tests/golden/" + gold["source"]}
    full = [(a.elapsed_time(b), k) for a, b, k in launches if k == depth] or \
        [(a.elapsed_time(b), k) for a, b, k in launches]
    kern_ms = sum(t for t, _ in full) / len(full)
    k_main = full[0][1]
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    value = W * H * gens * args.steps / (sum(ms) * 1e-3) / 1e9
    int_ops = 0.0
    if k_main > 1:
        import ctypes as C
        o, sec = C.c_double(), C.c_double()
        if L.life_measure_int_peak(0, 4000, C.byref(o), C.byref(sec)) == 0:
            int_ops = o.value
    e2e = None
    if not args.no_e2e:
        # The public API a user calls: Engine.upload (uint8 grid from pinned host
        # memory) -> life_run(engine=BYTE) -> Engine.download, all synchronous C-ABI
        # calls, host-timed per step (the context's own stream; no torch events).
        from paper_1209_4408_b200 import life
        host = torch.empty((H, W), dtype=torch.uint8, pin_memory=True).numpy()
        host[:] = bufs[cur[0]][:, :W].cpu().numpy()
        hout = torch.empty((H, W), dtype=torch.uint8, pin_memory=True).numpy()
        steps_e2e = max(2, args.steps)
        with life.Engine(0) as eng:
            eng.upload(host)
            eng.run(1, capi.ENGINE_BYTE, depth)
            eng.download(hout)
            t0 = time.perf_counter()
            for _ in range(steps_e2e):
                eng.upload(host)
                eng.run(gens, capi.ENGINE_BYTE, depth)
                eng.download(hout)
            e2e_s = time.perf_counter() - t0
            byte_final = hout.copy()
        e2e = {"value": W * H * gens * steps_e2e / e2e_s / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": W * H, "d2h_bytes_per_step": W * H,
               "api": "C-ABI life_grid_upload_u8 + life_run(LIFE_ENGINE_BYTE) + "
                      "life_grid_download_u8 from/to pinned host memory (host-timed)",
               "steps": steps_e2e}
        # The same byte-per-cell API with the packed engine behind it: the
        # uint8 grid is packed on the device at upload (warp ballots), runs
        # the temporal-blocked packed passes and is unpacked at download --
        # north_star's "converted at the API boundary".
        with life.Engine(0) as eng:
            eng.upload(host)
            eng.run(1, capi.ENGINE_PACKED, 0)
            eng.download(hout)
            eng.upload(host)
            eng.run(gens, capi.ENGINE_PACKED, 0)
            eng.download(hout)
            ok = fnv(hout.tobytes()) == fnv(byte_final.tobytes()) if byte_final is not None \
                else None
            t0 = time.perf_counter()
            for _ in range(steps_e2e):
                eng.upload(host)
                eng.run(gens, capi.ENGINE_PACKED, 0)
                eng.download(hout)
            pk_s = time.perf_counter() - t0
        e2e["packed_behind_byte_api"] = {
            "value": W * H * gens * steps_e2e / pk_s / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": W * H, "d2h_bytes_per_step": W * H,
            "api": "C-ABI life_grid_upload_u8 (device pack) + life_run(LIFE_ENGINE_PACKED, "
                   "depth auto) + life_grid_download_u8 (device unpack), pinned host memory, "
                   "host-timed",
            "same_result_as_byte_engine": ok, "steps": steps_e2e}
    cpu = None
    if not args.no_cpu:
        try:
            cpu = cpu_measure(cfg, args.cpu_budget)
        except Exception as exc:  # reported, not fatal
            cpu = {"error": repr(exc)}
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sum(ms) / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8 (byte per cell)", "data": "synthetic",
        "config": {"workload": cfg["desc"].replace("bit-packed engine", "byte engine"),
                   "engine": "byte", "generations": gens, "temporal_depth": depth,
                   "l2": "inputs larger than L2" if flush is None else "L2 flushed between steps"},
        "roofline": byte_roofline(W * H * k_main, k_main, kern_ms, hbm_peak, int_ops,
                                  ncu_traffic(args.config, k_main, "byte")),
        "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": n_launch, "clocks": clocks.summary()}), flush=True)
    if parity.get("ok") is False:
        print("bench.py: PARITY MISMATCH against the reference golden", file=sys.stderr)
        sys.exit(3)


def run_resident_arm(args) -> None:
    """The cluster-resident engine (whole torus in one thread-block cluster's
    shared memory, every generation of a step in one launch) on one GPU;
    small tori with W % 32 == 0 (config 1)."""
    import ctypes as C

    import torch

    from paper_1209_4408_b200 import capi
    from paper_1209_4408_b200.life import check
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "unavailable": "resident engine is single-GPU"}))
        return
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L = capi.lib()
    cfg = CONFIGS[args.config]
    W, H, gens = cfg["w"], cfg["h"], args.gens or cfg["gens"]
    n_cta = int(L.life_resident_cluster_size(W, H))
    if n_cta == 0:
        print(json.dumps({"metric": METRIC, "unavailable": f"{W}x{H} does not fit the resident engine"}))
        return
    pitch = int(L.life_packed_pitch_words(W))
    bufs = [torch.zeros((H, pitch), dtype=torch.int32, device=dev) for _ in range(2)]
    stream = torch.cuda.current_stream(dev).cuda_stream
    check(L.life_dev_packed_random(bufs[0].data_ptr(), pitch, W, 0, H, cfg["p"], 42, stream))
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    int_ops = 0.0
    o, sec = C.c_double(), C.c_double()
    if L.life_measure_int_peak(0, 4000, C.byref(o), C.byref(sec)) == 0:
        int_ops = o.value
    cur = [0]

    def step():
        a, b = bufs[cur[0]], bufs[cur[0] ^ 1]
        check(L.life_dev_packed_run_resident(a.data_ptr(), b.data_ptr(), pitch, W, H, gens, stream))
        cur[0] ^= 1

    clocks = ClockSampler(0).__enter__()  # running through warm-up and timed steps
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = L.life_kernel_launches()
    ms = []
    clocks.mark(0)
    for _ in range(args.steps):
        flush.fill_(1)  # the grid fits in L2: flush between steps
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    clocks.mark(1)
    clocks.__exit__(None, None, None)
    n_launch = int(L.life_kernel_launches() - l0)
    parity = {"ok": None, "reason": "--no-parity"}
    gold = None if args.no_parity else golden_for(args.config, gens)
    if gold is not None and gold["kind"] == "hash" and not cfg.get("soup"):
        check(L.life_dev_packed_random(bufs[cur[0]].data_ptr(), pitch, W, 0, H, cfg["p"], 42,
                                       stream))
        step()
        torch.cuda.synchronize()
        wpr = (W + 63) // 64
        got = f"{fnv(bufs[cur[0]][:, :2 * wpr].contiguous().cpu().numpy().tobytes()):016x}"
        parity = {"ok": got == gold["fnv_packed"], "kind": "full-grid packed FNV-1a-64",
                  "got": got, "want": gold["fnv_packed"], "generations": gens,
                  "source": "tests/golden/" + gold["source"]}
    step_ms = sum(ms) / len(ms)
    value = W * H * gens * args.steps / (sum(ms) * 1e-3) / 1e9
    achieved = W * H * gens * OPS_PER_UPDATE / (step_ms * 1e-3) / 1e12
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_cluster = int_ops / 1e12 * n_cta / sms
    e2e = None
    if not args.no_e2e:
        # Public API: packed grid from pinned host memory -> life_run(RESIDENT)
        # -> packed grid back, synchronous C-ABI calls, host-timed per step.
        from paper_1209_4408_b200 import life
        wpr = (W + 63) // 64
        host = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True).numpy()
        host[:] = bufs[cur[0]].cpu().numpy().view("int64")[:, :wpr]
        hout = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True).numpy()
        steps_e2e = max(5, args.steps)
        with life.Engine(0) as eng:
            # life_run_batch with temporal_depth 0 runs each grid on the resident
            # engine; grid i's copies overlap grid i+-1's compute.
            hu = host.view("uint64")
            eng.run_batch([hu], [hout.view("uint64")], W, gens, 0)  # warm-up (buffers)
            e2e_ms = eng.run_batch([hu] * steps_e2e, [hout.view("uint64")] * steps_e2e, W, gens, 0)
        e2e = {"value": W * H * gens * steps_e2e / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": H * wpr * 8, "d2h_bytes_per_step": H * wpr * 8,
               "api": "C-ABI life_run_batch(temporal_depth 0 -> cluster-resident engine) from/to "
                      "pinned host memory (per step: H2D packed grid, run, D2H; CUDA events "
                      "from the first upload to the last download)",
               "note": "grids run back to back with their copies overlapped, so e2e can "
                       "exceed the device value, which times each step alone (L2 flushed, "
                       "launch latency of the 70-us step included)",
               "steps": steps_e2e}
    cpu = None
    if not args.no_cpu:
        try:
            cpu = cpu_measure(cfg, args.cpu_budget)
        except Exception as exc:  # reported, not fatal
            cpu = {"error": repr(exc)}
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "u32 bit-sliced (32 cells/word, exact integer)", "data": "synthetic",
        "config": {"workload": cfg["desc"].replace("bit-packed engine", "cluster-resident engine"),
                   "engine": "resident", "generations": gens, "cluster_ctas": n_cta,
                   "l2": "L2 flushed between steps"},
        "roofline": {"bound": "int", "kernel": "packed_resident_kernel",
                     "achieved": achieved, "peak": peak_cluster, "unit": "Tops/s",
                     "frac": achieved / peak_cluster if peak_cluster else None,
                     "peak_source": f"measured LOP3 peak x {n_cta}/{sms} SMs (one cluster)",
                     "frac_of_gpu": achieved / (int_ops / 1e12) if int_ops else None,
                     "ops_per_cell_update": OPS_PER_UPDATE, "mean_launch_ms": step_ms,
                     "traffic": None},
        "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": n_launch, "clocks": clocks.summary()}), flush=True)
    if parity.get("ok") is False:
        print("bench.py: PARITY MISMATCH against the reference golden", file=sys.stderr)
        sys.exit(3)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--depth", type=int, default=0,
                    help="generations per packed pass; 0 = the engine's auto rule (16; 12 for "
                         "one-launch W %% 32 != 0 tori such as config 4)")
    ap.add_argument("--pair-depth", type=int, default=-1,
                    help="pair-layout kernel (W %% 64 == 0 tori): -1 = the engine's auto "
                         "rule when --depth is 0 too, 0 = off, 1..12 = forced depth")
    ap.add_argument("--quad-depth", type=int, default=-1,
                    help="quad-layout kernel (W %% 128 == 0 tori): -1 = auto, 0 = off, "
                         "1..7 = forced depth")
    ap.add_argument("--gens", type=int, default=0, help="override the config's generations")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--engine", choices=["auto", "packed", "byte", "resident"], default="auto",
                    help="auto: the cluster-resident engine for small W %% 32 == 0 tori on one "
                         "GPU (config 1, as life_run's depth-0 auto mode), else packed")
    ap.add_argument("--byte-depth", type=int, default=0,
                    help="byte engine generations per pass (0 = auto, 1 = HBM-bound single step)")
    ap.add_argument("--halo", choices=["peer", "nccl"], default="peer",
                    help="multi-GPU halo: in-kernel NVLink peer reads or NCCL send/recv")
    ap.add_argument("--pass-sync", choices=["neighbour", "neighbour_overlap", "flag", "flag_overlap", "allreduce"], default="neighbour",
                    help="peer halo: order passes by a token with the two neighbour ranks "
                         "(default) or by an all-rank NCCL all-reduce")
    ap.add_argument("--single-process", action="store_true",
                    help="N GPUs from ONE process through the multi-device C-ABI context "
                         "(life_ctx_create_multi) instead of one rank per GPU")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-run comparison with the reference's golden fixture")
    args = ap.parse_args()
    ranked = "WORLD_SIZE" in os.environ
    if args.impl == "ours" and args.gpus > 1 and not ranked and not args.single_process:
        sys.exit(self_launch(args))
    if args.engine == "auto":
        c = CONFIGS[args.config]
        small = c["w"] % 32 == 0 and c["w"] * c["h"] <= 2 ** 22
        args.engine = "resident" if small and int(os.environ.get("WORLD_SIZE", "1")) == 1 \
            else "packed"
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.single_process:
        run_ctx_arm(args)
    elif args.engine == "byte":
        run_byte_arm(args)
    elif args.engine == "resident":
        run_resident_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
