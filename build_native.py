"""Native build of every shared library in the repo (in-tree, so the .so files travel to the GPU box).

    python build_native.py            # build everything that is stale
    python build_native.py --force    # rebuild everything

Products:
  paper_2301_09310_b200/libsaloba.so  — the C-ABI CUDA library (nvcc, sm_100a only)
  oracle/liboracle.so                 — CPU oracle (gcc; test infrastructure)
  synth/libsynth.so                   — seeded input generator (gcc; shared input module)
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

PKG = os.path.join(ROOT, "paper_2301_09310_b200")
CSRC = os.path.join(PKG, "csrc")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def build_synth(force: bool = False) -> str:
    out = os.path.join(ROOT, "synth", "libsynth.so")
    src = os.path.join(ROOT, "synth", "synth.c")
    if force or _stale(out, [src]):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", out, src, "-lm"])
    return out


def build_oracle(force: bool = False) -> str:
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("oracle.c", "ksw.c", "traceback.c")]
    # -O2 without vectorisation flags: the oracle is timed "as it stands", never tuned.
    if force or _stale(out, srcs):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", out, *srcs])
    return out


def build_saloba(force: bool = False, out: str | None = None, defines: list[str] | None = None,
                 objdir: str | None = None) -> str:
    """libsaloba.so; `out`/`defines`/`objdir` build an experiment variant elsewhere (tools/variants.py)."""
    out = out or os.path.join(PKG, "libsaloba.so")
    objdir = objdir or os.path.join(ROOT, "build")
    defines = defines or []
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "saloba.h")]
    if not srcs:
        return out
    if force or _stale(out, deps):
        objs, jobs = [], []
        os.makedirs(objdir, exist_ok=True)
        for s in srcs:
            o = os.path.join(objdir, os.path.basename(s) + ".o")
            if force or _stale(o, [s] + deps):
                jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                             "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-warn-spills",
                             *defines, "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o])
            objs.append(o)
        # translation units compile in parallel (dp_i16.cu dominates: ~100 kernel instances)
        with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
            list(ex.map(_run, jobs))
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs])
    return out


def build_all(force: bool = False) -> None:
    build_synth(force)
    build_oracle(force)
    build_saloba(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
