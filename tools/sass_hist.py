"""SASS opcode histogram of the hot kernels in the built library (static
instruction counts, cuobjdump -sass), written as markdown.

    python tools/sass_hist.py > profiles/sass_hist_r2.md

Proves which hardware paths each kernel uses (TLD = texture fetches,
UBLKCP/UTMALDG = TMA, LDS/STS = shared memory, FADD2 = paired fp32 adds,
SYNCS = mbarriers, no UTCMMA: tensor cores unused, as the north star asks)."""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2005_09904_b200" / "lib" / "libbiqgemm_b200.so"
HOT = [
    ("biqgemm_tex_kernelILi3ELi1ELi28E", "grouped texture form, beta=3 (C2/C4 step)"),
    ("biqgemm_latency_kernelILi3E", "single-call latency form, beta=3 (C2 dependent chain)"),
    ("biqgemm_stream_kernelILi3E", "grouped TMA-ring form, beta=3 (groups of < 4 calls)"),
    ("biqgemm_fast_kernelILi8ELi4E", "two-kernel form gather, mu=8 BT=4 (C3/C5)"),
    ("biqgemm_cluster_kernelILi8ELi4E", "cluster form, mu=8 BT=4"),
    ("finalize_kernelILi4ELi4E", "two-kernel form finaliser"),
]
KEY = ["LDS", "STS", "PRMT", "FADD2", "FADD", "TLD", "LDG", "STG", "UBLKCP", "UTMALDG", "SYNCS", "DFMA", "F2F",
       "SHFL", "ATOMS", "RED", "UTCMMA", "BAR", "NANOSLEEP"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    print("# SASS opcode histograms (static counts) -- `python tools/sass_hist.py`\n")
    print(f"Library: `{LIB.relative_to(LIB.parent.parent.parent)}` (sm_100a).\n")
    for pat, what in HOT:
        body = next((f for f in funcs if pat in f.split("\n", 1)[0]), None)
        if body is None:
            print(f"## {pat}: not found\n")
            continue
        name = body.split("\n", 1)[0].strip()
        ops = collections.Counter()
        for line in body.splitlines():
            mm = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if mm:
                ops[mm.group(1).split(".")[0]] += 1
        total = sum(ops.values())
        print(f"## {what}\n\n`{name[:140]}`\n\n{total} instructions.\n")
        print("| opcode | count |\n|---|---|")
        for k in KEY:
            if ops.get(k):
                print(f"| {k} | {ops[k]} |")
        rest = sorted(((v, k) for k, v in ops.items() if k not in KEY), reverse=True)[:8]
        print("| (top others) | " + ", ".join(f"{k} {v}" for v, k in rest) + " |\n")


if __name__ == "__main__":
    sys.exit(main())
