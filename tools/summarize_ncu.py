"""Summarise a round's ncu evidence into profiles/ (tracked):

  profiles/ncu_<tag>.md          per-config full-capture metrics of the hot
                                 kernel, stall breakdown, launch-list shares
  profiles/ncu_launches_<tag>_<cfg>.csv   the launch lists themselves
  profiles/ncu_summary.json      per-config DRAM bytes per launch (bench.py
                                 reads it for roofline.traffic)

    python tools/summarize_ncu.py <tag> <dir with full_<cfg>.ncu-rep and launches_<cfg>.csv> <cfg> [<cfg> ...]
"""
import csv
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"
sys.path.insert(0, str(ROOT))

SCALE = {"us": 1e3, "ns": 1, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "second": 1e9, "Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6, "Ghz": 1e9, "Mhz": 1e6}


def fnum(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            f = fnum(v)
            d[h] = f * SCALE.get(u, 1) if f is not None else v
        res.append(d)
    return res


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, im, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
    per = defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) > max(ik, iv, im, iid):
            per[(r[iid], r[ik])][r[im]] = fnum(r[iv])
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), v in per.items():
        a = agg[name.split("(")[0][:70]]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum") or 0
        a[2] += (v.get("dram__bytes_read.sum") or 0)
    return agg


def main():
    tag, d = sys.argv[1], Path(sys.argv[2])
    cfgs = sys.argv[3:]
    from bench import CONFIGS, key_bytes

    PROF.mkdir(exist_ok=True)
    sp = PROF / "ncu_summary.json"
    summary = json.loads(sp.read_text()) if sp.exists() else {}
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    L = [f"# ncu evidence, round {tag}", "",
         "Captured under gpurun on one B200 (tools/profile_r2.sh): `ncu --set full --clock-control none "
         "--import-source on -k regex:<kernel> -s <skip> -c 1` of `python bench.py --config <C> --profile --steps 4 "
         "--warmup 3` (a grouped launch = one bench step = 128 independent calls), and the launch lists "
         "(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`; "
         "cold-cache and serialised: compare shares, not absolutes).", ""]
    for cfg in cfgs:
        if cfg in CONFIGS:
            m, n, beta, b, mu = CONFIGS[cfg]
        else:  # e.g. C4b2: a config with its batch overridden
            base, bb = cfg.split("b", 1)
            m, n, beta, b, mu = CONFIGS[base]
            b = int(bb)
        kb = key_bytes(m, n, beta, mu)
        for rep, kname, calls in ((d / f"full_{cfg}.ncu-rep", "biqgemm_stream_kernel", 128),
                                  (d / f"full_tex_{cfg}.ncu-rep", "biqgemm_tex_kernel", 128),
                                  (d / f"lat_{cfg}.ncu-rep", "biqgemm_latency_kernel", 1),
                                  (d / f"full_lat_{cfg}.ncu-rep", "biqgemm_latency_kernel", 1)):
            if not rep.exists():
                continue
            for k in raw(rep):
                name = k.get("Kernel Name", "?")
                if kname not in name:
                    continue
                dur = k.get("gpu__time_duration.sum")
                rd, wr = k.get("dram__bytes_read.sum") or 0, k.get("dram__bytes_write.sum") or 0
                alg = kb * calls
                lsu = k.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") or 0
                sms = k.get("launch__grid_size")
                clk = k.get("sm__cycles_elapsed.avg.per_second")
                what = (f"one grouped launch, {calls} calls" if calls > 1 else
                        "one single call, standalone under ncu (no PDL overlap, cold caches)")
                L += [f"## {cfg} (m={m} n={n} q={beta} mu={mu} b={b}): `{kname}<{beta}>`", "",
                      "| metric | value |", "|---|---|",
                      f"| duration ({what}) | {dur / 1e3:.2f} us = {dur / 1e3 / calls:.3f} us/call |",
                      f"| algorithmic key bytes / launch | {alg / 1e6:.2f} MB ({kb} B/call) |",
                      f"| achieved (algorithmic) | {alg / dur:.0f} GB/s = {alg / dur / peaks.get('hbm_gbs', 6536.4) * 100:.1f}% of {peaks.get('hbm_gbs', 6536.4)} GB/s measured peak |",
                      f"| DRAM read / write | {rd / 1e6:.2f} MB / {wr / 1e6:.2f} MB (read/algorithmic = {rd / alg:.3f}) |",
                      f"| DRAM throughput | {k.get('dram__bytes_read.sum.per_second', 0) / 1e12:.2f} TB/s read |",
                      f"| shared-memory wavefronts | {lsu / 1e6:.3f} M = {lsu / calls / max(sms or 1, 1):.0f} per CTA per call |",
                      f"| LSU pipe busy | {k.get('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active')} % |",
                      f"| issue active | {k.get('smsp__issue_active.avg.pct_of_peak_sustained_active')} % |",
                      f"| SM clock under ncu | {clk / 1e9 if clk else None} GHz |",
                      f"| registers / threads / grid | {k.get('launch__registers_per_thread')} / {k.get('launch__block_size')} / {sms} |",
                      ""]
                stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v)
                                 for h, v in k.items() if h.startswith("smsp__average_warps_issue_stalled")
                                 and "not_issued" not in h and isinstance(v, float) and v > 0.05), key=lambda t: -t[1])
                L += ["Stalls per issued instruction: " + ", ".join(f"{a} {v:.2f}" for a, v in stalls[:8]), ""]
                if calls > 1:
                    summary[cfg] = {"dram_bytes_per_launch": rd + wr, "calls_per_launch": calls,
                                    "algorithmic_bytes_per_launch": alg, "duration_us_ncu": dur / 1e3,
                                    "kernel": name[:100], "round": tag,
                                    "dram_bytes_per_call": (rd + wr) / calls,
                                    "source": f"profiles/ncu_{tag}.md ({rep.name}: ncu --set full, one launch)"}
        # b >= 2 forms: the two-kernel fast form (tools/fast_sweep.py under ncu)
        fp = d / f"fast_{cfg}.ncu-rep"
        if not fp.exists():
            fp = d / f"full_fast_{cfg}.ncu-rep"
        if fp.exists():
            G = (n + mu - 1) // mu
            lds_alg = 4 * beta * m * G * b  # LUT bytes gathered
            rows = [k for k in raw(fp) if "biqgemm_fast_kernel" in str(k.get("Kernel Name"))
                    or "finalize_kernel" in str(k.get("Kernel Name"))]
            if rows:
                L += [f"## {cfg} (m={m} n={n} q={beta} mu={mu} b={b}): two-kernel fast form, one single call", "",
                      "| kernel | us | LDS GB/s (algorithmic) | shared wavefronts | LSU data pipe % | issue % | DRAM rd / wr MB | regs / threads / grid |",
                      "|---|---|---|---|---|---|---|---|"]
                for k in rows:
                    dur = k.get("gpu__time_duration.sum") or 1
                    nm = str(k.get("Kernel Name")).split("(")[0][:60]
                    lsu = k.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") or 0
                    gbs = lds_alg / dur if "fast_kernel" in nm else 0
                    L.append(f"| `{nm}` | {dur / 1e3:.2f} | {gbs:.0f} | {lsu / 1e6:.2f} M | "
                             f"{k.get('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed')} | "
                             f"{k.get('smsp__issue_active.avg.pct_of_peak_sustained_active')} | "
                             f"{(k.get('dram__bytes_read.sum') or 0) / 1e6:.1f} / {(k.get('dram__bytes_write.sum') or 0) / 1e6:.1f} | "
                             f"{k.get('launch__registers_per_thread')} / {k.get('launch__block_size')} / {k.get('launch__grid_size')} |")
                L += ["", f"LDS roofline (128 B/clk/SM x 148 SMs x 1.9 GHz = 36 TB/s): {lds_alg / 36e12 * 1e6:.1f} us "
                      f"for {lds_alg / 1e6:.0f} MB of gathered LUT bytes.", ""]
        lp = d / f"launches_{cfg}.csv"
        if lp.exists():
            shutil.copy(lp, PROF / f"ncu_launches_{tag}_{cfg}.csv")
            agg = launch_shares(lp)
            tot = sum(a[1] for a in agg.values()) or 1
            L += [f"### {cfg} launch list (whole bench run under ncu, incl. setup kernels)", "",
                  "| kernel | launches | time us | share | DRAM read MB |", "|---|---|---|---|---|"]
            for nm, (c, t, rb) in sorted(agg.items(), key=lambda x: -x[1][1]):
                L.append(f"| `{nm}` | {c} | {t / 1e3:.1f} | {t / tot * 100:.1f}% | {rb / 1e6:.1f} |")
            L.append("")
    (PROF / f"ncu_{tag}.md").write_text("\n".join(L) + "\n")
    sp.write_text(json.dumps(summary, indent=1) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
