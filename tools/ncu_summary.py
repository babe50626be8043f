"""Summarise ncu captures into profiles/<round>/ (tracked) from gpurun_out/ (scratch).

    python tools/ncu_summary.py --round r1 --read gpurun_out/prof_read_r1.ncu-rep \
        --write gpurun_out/prof_write_v2.ncu-rep --launches gpurun_out/launches_r1.csv

Writes:
  profiles/<round>/<kernel>_ncu.txt   key metrics of one `ncu --set full` launch
  profiles/<round>/launches.csv       the launch list (gpu__time_duration per launch)
  profiles/<round>/launch_shares.txt  per-kernel share of one bench step (scaled from the list)
  profiles/traffic.json               dram bytes per launch (read by bench.py's roofline.traffic)
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "lts__t_bytes.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, units))) for r in rows[2:]]


def summarise(rep, label, outdir):
    res = {}
    all_lines = []
    for d, u in raw(rep):
        lines = [f"# {label}: {d.get('Kernel Name', '?')}", f"# source: {os.path.basename(rep)} (ncu --set full, 1 launch)"]
        for k in KEYS:
            if k in d:
                lines.append(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
        rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rdb = rd * scale.get(u["dram__bytes_read.sum"], 1)
        wrb = wr * scale.get(u["dram__bytes_write.sum"], 1)
        tscale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
        t_ns = float(d["gpu__time_duration.sum"]) * tscale.get(u["gpu__time_duration.sum"], 1)
        lines.append(f"# dram traffic per launch = {rdb + wrb:.4e} B; achieved {(rdb + wrb) / t_ns:.1f} GB/s "
                     f"(cold-cache, serialised replay)")
        all_lines += lines + [""]
        res = {"dram_bytes_per_launch": rdb + wrb, "dram_read": rdb, "dram_write": wrb, "time_ns": t_ns,
               "source": os.path.relpath(os.path.join(outdir, f"{label}_ncu.txt"), ROOT)}
    open(os.path.join(outdir, f"{label}_ncu.txt"), "w").write("\n".join(all_lines))
    return res


def shares(launches, outdir, read_per_window=127 * 36 + 36, write_per_window=1):   # r2: one WRITE launch (all layers)
    lines_in = [l for l in open(launches) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines_in))))
    per = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            unit = r.get("Metric Unit", "nsecond")
            per[name].append(float(r["Metric Value"]) * {"usecond": 1e3, "msecond": 1e6}.get(unit, 1))
    lines = ["# per-kernel launch times from the ncu launch list (cold-cache, serialised: compare SHARES)",
             "kernel, launches, mean_us"]
    means = {}
    for k, v in sorted(per.items()):
        means[k] = sum(v) / len(v) / 1e3
        lines.append(f"{k}, {len(v)}, {means[k]:.2f}")
    rk = [k for k in means if "read_decode" in k]
    wk = [k for k in means if "write_tc" in k or "write_simt" in k]
    if rk and wk:
        tr = means[rk[0]] * read_per_window
        tw = means[wk[0]] * write_per_window
        lines.append(f"# one bench step (128-token window x 36 layers): {read_per_window} READ launches + "
                     f"{write_per_window} WRITE launches")
        lines.append(f"READ share = {tr / (tr + tw):.3f}, WRITE share = {tw / (tr + tw):.3f} "
                     f"(window kernel time {1e-3 * (tr + tw):.1f} ms)")
    open(os.path.join(outdir, "launch_shares.txt"), "w").write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--read")
    ap.add_argument("--write")
    ap.add_argument("--launches")
    ap.add_argument("--chunk")
    ap.add_argument("--extra", action="append", default=[], help="label=path.ncu-rep")
    a = ap.parse_args()
    outdir = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(outdir, exist_ok=True)
    traffic = {}
    if a.read:
        traffic["read_decode_kernel"] = summarise(a.read, "read_decode", outdir)
    if a.write:
        traffic["write_tc_kernel"] = summarise(a.write, "write_tc", outdir)
    if a.chunk:
        traffic["read_chunk_tc_kernel"] = summarise(a.chunk, "read_chunk_tc", outdir)
    for e in a.extra:
        label, path = e.split("=", 1)
        summarise(path, label, outdir)
    if a.launches:
        shutil.copy(a.launches, os.path.join(outdir, "launches.csv"))
        shares(a.launches, outdir)
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    old = json.load(open(tf)) if os.path.exists(tf) else {}
    old.update(traffic)
    old["_round"] = a.round
    json.dump(old, open(tf, "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
