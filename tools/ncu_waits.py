"""Summarise an ncu report's warp-stall samples: share per SASS opcode and per
mbarrier wait site (the TRYWAIT that precedes each hot retry branch)."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else "biqgemm_stream"
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kfilter}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
i_src, i_ex, i_st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
seen = set()
for r in rows[2:]:
    try:
        ex, st = float(r[i_ex] or 0), float(r[i_st] or 0)
    except (ValueError, IndexError):
        continue
    if r[0] in seen:
        break  # second copy of the same kernel
    seen.add(r[0])
    data.append((r[0], r[i_src], ex, st))
tot = sum(d[3] for d in data) or 1
ops = Counter()
for _, s, _, st in data:
    t = s.split()
    if t:
        ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += st
print("stall share by opcode:", [(k, round(v / tot * 100, 1)) for k, v in ops.most_common(10)])
last_wait = None
waits = Counter()
for _, s, _, st in data:
    if "TRYWAIT" in s:
        last_wait = s.split("[")[1].split("]")[0] if "[" in s else s
    if "BRA" in s and st / tot > 0.003 and last_wait:
        waits[last_wait] += st
print("retry-branch stalls by wait site:", [(k, round(v / tot * 100, 1)) for k, v in waits.most_common(10)])
