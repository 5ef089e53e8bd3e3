"""Summarise ncu captures into profiles/ (tracked): per-kernel duration,
DRAM bytes, throughput and stall breakdown, plus profiles/ncu_summary.json
(read by bench.py for roofline.traffic).

    python tools/summarize_ncu.py <round-tag> <config>=<report.ncu-rep> ... [--launches <csv>]
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
         "msecond": 1e6, "ms": 1e6,
         "second": 1e9}


def raw_metrics(rep):
    """Rows of the raw page with values converted to base units (bytes, ns)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            f = fnum(v)
            d[h] = f * SCALE[u] if (f is not None and u in SCALE) else v
        kernels.append(d)
    return kernels


def fnum(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    PROF.mkdir(exist_ok=True)
    summary_path = PROF / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    lines = [f"# ncu summary, round {tag}", ""]
    for a in args:
        cfg, rep = a.split("=", 1)
        for k in raw_metrics(rep):
            name = k.get("Kernel Name", "?")
            dur_ns = fnum(k.get("gpu__time_duration.sum"))
            rd = fnum(k.get("dram__bytes_read.sum"))
            wr = fnum(k.get("dram__bytes_write.sum"))
            # ncu reports bytes in scaled units in raw csv units row; normalise by the unit row if present
            d = {
                "kernel": name[:120],
                "duration_us": dur_ns / 1000 if dur_ns else None,
                "dram_read_bytes": rd,
                "dram_write_bytes": wr,
                "sm_throughput_pct": fnum(k.get("sm__throughput.avg.pct_of_peak_sustained_elapsed")),
                "dram_throughput_pct": fnum(k.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
                "lsu_shared_wavefronts": fnum(k.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")),
                "registers": fnum(k.get("launch__registers_per_thread")),
                "grid": k.get("launch__grid_size"),
            }
            lines.append(f"## {cfg}: {name[:100]}")
            for kk, vv in d.items():
                lines.append(f"- {kk}: {vv}")
            lines.append("")
            if "biqgemm" in name:
                summary[cfg] = {"dram_bytes_per_launch": (rd or 0) + (wr or 0), "duration_us_ncu": d["duration_us"],
                                "kernel": d["kernel"], "round": tag}
    if launches:
        lines.append("## launch list (ncu --metrics gpu__time_duration.sum, cold cache, serialised)")
        with open(launches) as f:
            rows = [r for r in csv.reader(f) if len(r) > 10]
        hdr = rows[0]
        for r in rows[1:]:
            rec = dict(zip(hdr, r))
            if rec.get("Metric Name") == "gpu__time_duration.sum":
                lines.append(f"- {rec.get('Kernel Name', '?')[:90]}: {rec.get('Metric Value')} ns")
    (PROF / f"ncu_{tag}.md").write_text("\n".join(lines) + "\n")
    summary_path.write_text(json.dumps(summary, indent=1) + "\n")
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
