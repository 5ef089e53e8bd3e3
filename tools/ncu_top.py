"""Summarise an ncu report: SOL numbers + top stalled SASS lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Active Warps Per SM", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Grid Size"]
for row in csv.reader(det.splitlines()):
    while row and row[-1] == "":
        row = row[:-1]
    if len(row) > 3 and row[-3] in want:
        print(f"{row[-3]:40s} {row[-1]:>14s} {row[-2]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data)
print("total stall samples", tot, "instructions", len(data))
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(float(r[hdr.index(c)] or 0) for r in data) for c in stall_cols}
print("by reason:", sorted(((k, int(v)) for k, v in agg.items() if v), key=lambda kv: -kv[1])[:8])
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:ntop]:
    st = {c: float(r[hdr.index(c)] or 0) for c in stall_cols}
    best = [(k[6:], int(v)) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:2] if v]
    print(f"{r[0][-5:]} {r[i_s]:>5} {r[i_ex]:>7} {r[i_src][:60]:60s} {best}")
