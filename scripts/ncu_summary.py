"""Development aid: headline metrics + stall reasons of one kernel in an ncu --set full report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
keys = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Issue Slots Busy",
        "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Avg. Active Threads Per Warp", "Grid Size",
        "Compute (SM) Throughput", "L2 Cache Throughput", "Dynamic Shared Memory Per Block")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for r in csv.reader(out.splitlines()):
    if len(r) > 14 and r[12] in keys:
        print(f"| {r[11]} | {r[12]} | {r[14]} {r[13]} |")
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, v = raw[0], raw[2] if len(raw) > 2 else raw[1]
st = {}
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
        except ValueError:
            pass
tot = sum(st.values()) or 1
for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]:
    print(f"| stall | {k} | {100 * x / tot:.1f}% |")
