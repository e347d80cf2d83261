"""Summarise an ncu capture (--set full) and a launch list into profiles/.

usage: python tools/summarize_profile.py REP.ncu-rep LAUNCHES.csv OUT_PREFIX KEY
  writes OUT_PREFIX.md (key metrics + stall breakdown), updates
  profiles/ncu_traffic.json[KEY] = dram read+write bytes per launch.
"""
import collections, csv, io, json, os, subprocess, sys

rep, launches, prefix, key = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))

def g(k, scale=1.0):
    try:
        return float(m[k].replace(",", "")) * scale
    except (KeyError, ValueError):
        return None

def to_bytes(k):
    unit = u.get(k, "byte")
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return g(k, f)

rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
dur_ms = g("gpu__time_duration.sum", {"usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6}.get(u.get("gpu__time_duration.sum", "msecond"), 1.0))
lines = [f"# ncu summary: {os.path.basename(rep)} ({m.get('Kernel Name', '')})", ""]
lines.append("| metric | value |")
lines.append("|---|---|")
for k in ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__cycles_active.avg", "sm__cycles_active.min", "sm__cycles_active.max",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]:
    if k in m:
        lines.append(f"| {k} | {m[k]} {u.get(k, '')} |")
stalls = sorted(((float(v or 0), k) for k, v in m.items()
                 if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")), reverse=True)
tot = sum(x for x, _ in stalls) or 1
lines += ["", "Warp-state samples (share of all samples):", ""]
for x, k in stalls[:10]:
    lines.append(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {x / tot:.1%}")
if launches and os.path.exists(launches):
    lrows = [r for r in csv.reader(open(launches)) if len(r) > 10]
    h = lrows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot_t, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in lrows[1:]:
        name = r[ki].split("(")[0]
        tot_t[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        cnt[name] += 1
    s = sum(tot_t.values())
    lines += ["", f"Launch list ({os.path.basename(launches)}; cold-cache, serialised; whole process incl. untimed init):", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k in sorted(tot_t, key=lambda k: -tot_t[k]):
        lines.append(f"| {k} | {cnt[k]} | {tot_t[k]:.3f} | {tot_t[k] / s:.3f} |")
open(prefix + ".md", "w").write("\n".join(lines) + "\n")
tpath = os.path.join(os.path.dirname(prefix), "ncu_traffic.json")
t = json.load(open(tpath)) if os.path.exists(tpath) else {}
if rd is not None and wr is not None:
    t[key] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "duration_ms": dur_ms,
              "source": os.path.basename(rep)}
json.dump(t, open(tpath, "w"), indent=1, sort_keys=True)
print("\n".join(lines))
