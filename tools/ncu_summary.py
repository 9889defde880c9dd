"""Summarise an ncu report: key metrics and the hottest SASS lines."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
det = subprocess.run(["ncu", "-i", rep, *kf, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ("Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Issued Warp Per Scheduler", "Memory Throughput", "Theoretical Occupancy",
        "Avg. Active Threads Per Warp", "Block Limit Registers", "Grid Size", "Block Size")
for r in csv.reader(det.splitlines()):
    if len(r) > 4 and r[-4] in keep:
        print(f"  {r[-4]:40s} {r[-2]:>14s} {r[-3]}")
src = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_e = hdr.index("Instructions Executed")
tot = sum(int(r[i_s] or 0) for r in data)
print("  samples", tot, "instructions", sum(int(r[i_e] or 0) for r in data))
for k, r in sorted(enumerate(data), key=lambda kr: -int(kr[1][i_s] or 0))[:top]:
    print(f"  {k:5d} {r[1][:64]:64s} {r[i_s]:>6s} {r[i_e]:>8s}")
# stall reasons summed over the kernel (share of all samples)
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot_st = {hdr[i]: sum(int(r[i] or 0) for r in data) for i in st}
s_all = sum(tot_st.values()) or 1
print("  stalls:", ", ".join(f"{k[6:]} {100*v/s_all:.1f}%" for k, v in sorted(tot_st.items(), key=lambda kv: -kv[1]) if v > 0.01 * s_all))
