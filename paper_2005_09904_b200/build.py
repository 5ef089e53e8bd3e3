"""In-tree build of the CUDA library and the test oracles.

    python -m paper_2005_09904_b200.build          # incremental
    python -m paper_2005_09904_b200.build --force  # full rebuild

Produces ``paper_2005_09904_b200/lib/libbiqgemm_b200.so`` (sm_100a only) with
nvcc, and runs ``make -C oracle`` for the test-infrastructure oracles.  The
built ``.so`` files are git-ignored but travel to the GPU box with gpurun.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
OBJDIR = ROOT / "build" / "obj"
LIB = LIBDIR / "libbiqgemm_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC,-O3,-Wall",
    "-I",
    str(ROOT / "include"),
]


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers():
    return sorted(list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h")))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("command failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def build_library(force: bool = False, verbose: bool = False) -> Path:
    OBJDIR.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    jobs = []
    objs = []
    for src in _sources():
        obj = OBJDIR / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            extra = ["-Xptxas", "-v"] if verbose else []
            jobs.append([NVCC] + NVFLAGS + extra + ["-c", str(src), "-o", str(obj)])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            outs = list(ex.map(_run, jobs))
        if verbose:
            for o in outs:
                sys.stdout.write(o)
    if force or jobs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    return LIB


def build_oracle() -> None:
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


CPP_TEST = ROOT / "build" / "dropin_test"


def build_cpp_tests(force: bool = False) -> Path:
    """The reference's unit/acceptance tests re-expressed against the drop-in
    C++ API (include/biqgemm_b200/), linked to the built library."""
    src = ROOT / "tests" / "cpp" / "dropin_test.cpp"
    deps = [src, LIB] + sorted((ROOT / "include" / "biqgemm_b200").glob("*.hpp")) + [ROOT / "include" / "bqg_capi.h"]
    if force or _stale(CPP_TEST, deps):
        CPP_TEST.parent.mkdir(parents=True, exist_ok=True)
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
              str(src), "-o", str(CPP_TEST), "-L", str(LIBDIR), "-lbiqgemm_b200", "-Wl,-rpath," + str(LIBDIR),
              "-Wl,-rpath,$ORIGIN/../paper_2005_09904_b200/lib", "-L/usr/local/cuda/lib64", "-lcudart",
              "-Wl,-rpath,/usr/local/cuda/lib64"])
    return CPP_TEST


def build(force: bool = False, verbose: bool = False) -> Path:
    lib = build_library(force=force, verbose=verbose)
    build_oracle()
    build_cpp_tests(force=force)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
