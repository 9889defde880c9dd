"""Turns a round's raw ncu outputs (gpurun_out/<tag>_*) into the committed
evidence under profiles/:
  profiles/<tag>_launches.csv     per-launch device times of the bench command
  profiles/<tag>_kernels.md       launch-list shares + ncu --set full metrics and
                                  top stall locations of each kernel
  profiles/trace_traffic.json     DRAM bytes per K3 launch (read by bench.py)
Usage: python tools/summarize_profiles.py r01
"""
from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
RAW = ROOT / "gpurun_out"
OUT = ROOT / "profiles"

KEEP = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Issued Warp Per Scheduler", "Grid Size", "Block Size",
        "Avg. Active Threads Per Warp"]
RAW_METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
               "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
               "smsp__issue_active.avg.pct_of_peak_sustained_active",
               "lts__t_bytes.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
               "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum"]


def ncu_csv(args):
    r = subprocess.run(["ncu", *args], capture_output=True, text=True)
    return list(csv.reader(r.stdout.splitlines()))


def launch_table(tag):
    rows = list(csv.reader(open(RAW / f"{tag}_launches.csv")))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    keep = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("vxm::", "")
            try:
                per[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
            except ValueError:
                pass
            keep.append([d["ID"], name, d["Grid Size"], d["Block Size"], d["Metric Name"], d["Metric Value"]])
    with open(OUT / f"{tag}_launches.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "metric", "value"])
        w.writerows(keep)
    total = sum(sum(v.get("gpu__time_duration.sum", [])) for v in per.values())
    lines = ["| kernel | launches | mean ns | share of device time | DRAM read B/launch | DRAM write B/launch |",
             "|---|---|---|---|---|---|"]
    for name, m in sorted(per.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", []))):
        t = m.get("gpu__time_duration.sum", [])
        rd, wr = m.get("dram__bytes_read.sum", [0]), m.get("dram__bytes_write.sum", [0])
        lines.append(f"| {name} | {len(t)} | {sum(t) / max(1, len(t)):.0f} | {sum(t) / total:.1%} | "
                     f"{sum(rd) / max(1, len(rd)):.0f} | {sum(wr) / max(1, len(wr)):.0f} |")
    return "\n".join(lines)


def kernel_section(tag, k):
    rep = RAW / f"{tag}_{k}.ncu-rep"
    if not rep.exists():
        note = " (not launched: K2a is fused into the dilation tiles when dims_x % 4 == 0)" if k == "dilate_rows" else ""
        return f"### {k}\n\n(no capture{note})", None
    det = ncu_csv(["-i", str(rep), "--page", "details", "--csv"])
    out = [f"### {k}", "", "| metric | value | unit |", "|---|---|---|"]
    vals = {}
    for r in det:
        if len(r) > 4 and r[-4] in KEEP:
            out.append(f"| {r[-4]} | {r[-2]} | {r[-3]} |")
            if r[-4] == "Executed Instructions":
                try:
                    vals["executed_instructions"] = float(r[-2].replace(",", ""))
                except ValueError:
                    pass
    raw = ncu_csv(["-i", str(rep), "--page", "raw", "--csv"])
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    if len(raw) >= 3:
        for key, unit, v in zip(raw[0], raw[1], raw[2]):
            if key in RAW_METRICS:
                try:
                    val = float(v.replace(",", "")) * scale.get(unit, 1.0)
                except ValueError:
                    continue
                vals[key] = val
                shown = f"{val:.0f} | byte" if unit in scale else f"{v} | {unit}"
                out.append(f"| {key} | {shown} |")
    src = ncu_csv(["-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"])
    if len(src) > 2 and "Warp Stall Sampling (All Samples)" in src[1]:
        hdr, data = src[1], src[2:]
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        tot = sum(int(r[i_s] or 0) for r in data) or 1
        out += ["", "Top stall locations (share of warp-stall samples):", "", "```"]
        for r in sorted(data, key=lambda r: -int(r[i_s] or 0))[:10]:
            out.append(f"{int(r[i_s] or 0) / tot:6.1%}  {r[1].strip()[:90]}")
        out.append("```")
        st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        sums = {hdr[i][6:]: sum(int(r[i] or 0) for r in data) for i in st}
        s_all = sum(sums.values()) or 1
        out += ["", "Warp stall reasons (share of samples): " + ", ".join(
            f"{k} {v / s_all:.1%}" for k, v in sorted(sums.items(), key=lambda kv: -kv[1]) if v > 0.01 * s_all)]
    return "\n".join(out), vals


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    OUT.mkdir(exist_ok=True)
    md = [f"# Kernel evidence, round tag `{tag}`", "",
          "Raw captures: `tools/profile_round.sh` under gpurun (1 B200; clocks from "
          f"`{tag}_gpu.txt`). Launch list = `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
          "dram__bytes_write.sum --clock-control none` of `bench.py --steps 2 --warmup 3` (cold-cache and "
          "serialised: compare shares, not absolutes). Per-kernel sections = `ncu --set full` of one launch in a "
          "batched cfg2 step (64 streams); merge_sequence from one 64-frame call of a single moving stream; "
          "merge_tma (the TMA-staged K4 of rows that are not word-aligned or longer than 1024 cells) from 8 cfg2 frames on a 101x100x50 grid.", ""]
    gpu = RAW / f"{tag}_gpu.txt"
    if gpu.exists():
        md += ["```", gpu.read_text().strip(), "```", ""]
    md += ["## Launch list of the bench command", "", launch_table(tag), ""]
    traffic = alu = issue = None
    step_instr = {}
    for k in ("trace_bundle", "populate_depth", "dilate_rows", "dilate_tiles", "merge_shift", "merge_sequence",
              "merge_tma"):
        sec, vals = kernel_section(tag, k)
        md += [sec, ""]
        if vals and k in ("trace_bundle", "populate_depth", "dilate_rows", "dilate_tiles", "merge_shift"):
            step_instr[k] = vals.get("executed_instructions")
        if k == "trace_bundle" and vals:
            try:
                traffic = float(vals.get("dram__bytes_read.sum", 0)) + float(vals.get("dram__bytes_write.sum", 0))
                alu = vals.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")
                issue = vals.get("smsp__issue_active.avg.pct_of_peak_sustained_active")
            except ValueError:
                traffic = None
    (OUT / f"{tag}_kernels.md").write_text("\n".join(md))
    if traffic is not None:
        (OUT / "trace_traffic.json").write_text(json.dumps(
            {"tag": tag, "kernel": "trace_bundle_kernel", "dram_bytes_per_launch": traffic,
             "alu_pipe_pct_of_peak": alu, "issue_active_pct": issue,
             "launch": "cfg2, 64 streams (one batched step)", "source": f"gpurun_out/{tag}_trace_bundle.ncu-rep"},
            indent=1))
    if step_instr:
        # warp instructions the batched cfg2 step executes (one single-branch
        # launch of each stage over 64 frames; K5 publish is negligible):
        # bench.py turns them into the step's issue floor
        (OUT / "step_instructions.json").write_text(json.dumps(
            {"tag": tag, "workload": "cfg2, 64 streams (one batched step)", "warp_instructions": step_instr,
             "total": sum(v for v in step_instr.values() if v), "source": f"profiles/{tag}_kernels.md"}, indent=1))
    print((OUT / f"{tag}_kernels.md").read_text()[:3000])


if __name__ == "__main__":
    main()
