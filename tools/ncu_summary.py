"""Summarise a round's ncu artefacts into profiles/ (dev tool, runs here).

usage: python tools/ncu_summary.py <prof dir> <round tag> [--config=N] [--no-traffic]
  * launch list (gpu__time_duration per launch) -> per-kernel totals/shares
  * each .ncu-rep -> key metrics (duration, DRAM bytes, pipe utilisation,
    occupancy, stall reasons) and profiles/ncu_traffic.json (DRAM bytes per
    launch for the roofline `traffic` key of bench.py)
"""
import csv
import glob
import json
import os
import subprocess
import sys
from collections import defaultdict

src, tag = sys.argv[1], sys.argv[2]
CFG = next((a.split("=", 1)[1] for a in sys.argv[3:] if a.startswith("--config=")), "4")
dst = os.path.join("profiles", tag)
os.makedirs(dst, exist_ok=True)

# ---- launch list
lpath = os.path.join(src, "launches.csv")
rows = list(csv.reader(open(lpath))) if os.path.exists(lpath) else []
hdr = None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].split("<")[0].replace("void ", "")
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
if tot:
    all_ms = sum(tot.values())
    lines = ["kernel,launches,total_ms,avg_ms,share"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"{k},{cnt[k]},{v:.3f},{v / cnt[k]:.4f},{v / all_ms:.4f}")
    open(os.path.join(dst, "launch_shares.csv"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:8]))

# ---- full captures
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
traffic_path = os.path.join("profiles", "ncu_traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    if len(rr) < 3:
        continue
    h, u, v = rr[0], rr[1], rr[2]
    d = {k: (x, un) for k, un, x in zip(h, u, v)}
    kname = d.get("Kernel Name", ("?", ""))[0].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].replace("void ", "")
    summ = {"kernel": kname, "source": os.path.basename(rep)}
    for k in want:
        if k in d:
            summ[k] = f"{d[k][0]} {d[k][1]}".strip()
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(x[0])
              for k, x in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
              and x[0] not in ("", "n/a")}
    summ["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    base = os.path.splitext(os.path.basename(rep))[0]
    json.dump(summ, open(os.path.join(dst, f"ncu_{base}.json"), "w"), indent=1)
    def tobytes(x):
        val, unit = x
        val = float(val.replace(",", ""))
        return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
        # keyed "cfg<id>/<bench kernel class>" (csrc/launch.h KernelClass names)
        short = kname.split("::")[-1].split("<")[0]
        short = {"conv_site_dmma_kernel": "conv_site_kernel", "tt_inner_chunk_kernel": "tt_inner_kernel",
                 "tt_inner_split_kernel": "tt_inner_kernel"}.get(short, short)
        traffic[f"cfg{CFG}/{short}"] = {
            "bytes_per_launch": tobytes(d["dram__bytes_read.sum"]) + tobytes(d["dram__bytes_write.sum"]),
            "source": f"ncu --set full, {os.path.basename(rep)} ({tag}): dram__bytes_read.sum + dram__bytes_write.sum"}
    print(json.dumps(summ, indent=1))
if "--no-traffic" not in sys.argv[3:]:  # secondary captures at other configs leave the bench's traffic alone
    json.dump(traffic, open(traffic_path, "w"), indent=1)
