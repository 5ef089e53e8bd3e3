"""Split an ncu report's warp-stall samples by kernel phase (SASS address
ranges delimited by marker instructions)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
phase = "prologue"
acc = {}
order = []
for r in data:
    ins = r[i_src]
    if "ACQBULK" in ins:
        phase = "after_pdl_wait(build)"
    elif "PHASECHK" in ins and phase.startswith("after_pdl"):
        phase = "query"
    elif "UCGABAR_ARV" in ins or "MEMBAR.ALL.GPU" in ins:
        phase = "cluster_barrier"
    elif "UCGABAR_WAIT" in ins:
        phase = "reduce"
    if phase not in acc:
        acc[phase] = {"samples": 0, "inst": 0, "stalls": {}}
        order.append(phase)
    a = acc[phase]
    a["samples"] += float(r[i_s] or 0)
    a["inst"] += float(r[i_ex] or 0)
    for c in stall_cols:
        a["stalls"][c] = a["stalls"].get(c, 0) + float(r[hdr.index(c)] or 0)
tot = sum(a["samples"] for a in acc.values())
for ph in order:
    a = acc[ph]
    top = sorted(a["stalls"].items(), key=lambda kv: -kv[1])[:4]
    print(f"{ph:24s} samples {a['samples']:6.0f} ({100*a['samples']/tot:5.1f}%)  warp-inst {a['inst']:9.0f}  top: " +
          ", ".join(f"{k[6:]}={v:.0f}" for k, v in top))
