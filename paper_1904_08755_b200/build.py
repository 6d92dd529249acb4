"""Builds libmk.so (the C-ABI library) in-tree with nvcc for sm_100a.

No fast-math anywhere: quantization must be IEEE fp32 division + floor (reading R6).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SO = PKG / "libmk.so"
SOURCES = ["context.cu", "region.cu", "coords.cu", "kmap.cu", "conv.cu", "conv_simt.cu", "conv_umma.cu", "conv_split.cu", "pool.cu", "crf.cu", "sort.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include"), "-I", str(CSRC)]


def _stale(obj: Path, src: Path, cmd) -> bool:
    """An object is rebuilt when a source or header is newer, or when its compile command
    (flags, defines) differs from the one recorded next to it."""
    stamp = obj.with_suffix(".cmd")
    if not obj.exists() or not stamp.exists() or stamp.read_text() != " ".join(cmd):
        return True
    deps = [src, *CSRC.glob("*.cuh"), ROOT / "include" / "mk.h"]
    return obj.stat().st_mtime < max(d.stat().st_mtime for d in deps)


def build(verbose: bool = False, jobs: int = 8, trace: bool = False, variant: str = "", defines=()) -> Path:
    """trace=True builds the MK_TRACE instrumented variant as tools/libmk_trace.so
    (development timelines; load it with MK_LIBRARY).  variant="name" with defines=[...]
    builds an experimental variant as build_variants/libmk_<name>.so (A/B measurements)."""
    objdir = PKG / ("build_trace" if trace else f"build_{variant}" if variant else "build")
    so = ROOT / "tools" / "libmk_trace.so" if trace else ROOT / "build_variants" / f"libmk_{variant}.so" if variant else SO
    so.parent.mkdir(exist_ok=True)
    defs = (["-DMK_TRACE"] if trace else []) + [f"-D{d}" for d in defines]
    objdir.mkdir(exist_ok=True)
    procs, objs = [], []
    for s in SOURCES:
        src, obj = CSRC / s, objdir / (Path(s).stem + ".o")
        objs.append(obj)
        cmd = ["nvcc", *ARCH, *FLAGS, *defs, "-c", str(src), "-o", str(obj)]
        if _stale(obj, src, cmd) or verbose:
            run = cmd[:-4] + ["-Xptxas", "-v"] + cmd[-4:] if verbose else cmd
            procs.append((cmd, obj, subprocess.Popen(run, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
            if len(procs) >= jobs:
                _drain(procs, verbose)
    _drain(procs, verbose)
    if not so.exists() or so.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = so.with_suffix(f".so.{os.getpid()}")
        subprocess.check_call(["nvcc", *ARCH, "-shared", "-o", str(tmp), *map(str, objs)])
        os.replace(tmp, so)
    return so


def _drain(procs, verbose):
    while procs:
        cmd, obj, p = procs.pop(0)
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        obj.with_suffix(".cmd").write_text(" ".join(cmd))
        if verbose and out.strip():
            print(out)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, trace="--trace" in sys.argv))
