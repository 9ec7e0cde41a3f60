#!/usr/bin/env python3
"""Build every native artefact in-tree (sm_100a only).

  oracle/liboracle.so                 plain C oracle (gcc, -ffp-contract=off)
  inputs/libchasegen.so               synthetic-input generator (host + device)
  paper_2303_02508_b200/libchase.so   the product: C ABI + sm_100a kernels

Usage: python build.py [--force] [--only oracle|inputs|chase]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=ROOT)


def build_oracle(force=False):
    src = [os.path.join(ROOT, "oracle", f) for f in ("oracle.c", "oracle.h")]
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, src):
        _run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-std=gnu11",
              "-Wall", "-Wextra", "-shared", "-fPIC", "-o", out, src[0], "-lm"])
    return out


def build_inputs(force=False):
    src = [os.path.join(ROOT, "inputs", f) for f in ("gen.cu", "chase_gen.h")]
    out = os.path.join(ROOT, "inputs", "libchasegen.so")
    if force or _stale(out, src):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC,-fopenmp",
              "-cudart", "static", "-o", out, src[0], "-lgomp"])
    return out


CHASE_SOURCES = ["chase_api.cpp", "envelope.cpp", "kernels.cu"]
CHASE_HEADERS = sorted(f for f in os.listdir(os.path.join(ROOT, "paper_2303_02508_b200", "csrc"))
                       if f.endswith((".h", ".cuh")))  # every header: a change to any rebuilds


def build_chase(force=False):
    csrc = os.path.join(ROOT, "paper_2303_02508_b200", "csrc")
    srcs = [os.path.join(csrc, f) for f in CHASE_SOURCES]
    deps = srcs + [os.path.join(csrc, f) for f in CHASE_HEADERS] + [os.path.join(ROOT, "include", "chase.h")]
    out = os.path.join(ROOT, "paper_2303_02508_b200", "libchase.so")
    if not (force or _stale(out, deps)):
        return out
    objdir = os.path.join(ROOT, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    common = ["-I", os.path.join(ROOT, "include"), "-I", csrc]
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        if s.endswith(".cu"):
            # -fmad=false: the canonical fp64 paths must not contract a*b+c
            # (DESIGN §3 Q9); -Xptxas -v reports registers/spills.
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xptxas", "-v",
                  "-Xcompiler", "-fPIC", *common, "-c", s, "-o", o])
        else:
            _run([NVCC, *ARCH, "-O2", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off", *common,
                  "-c", s, "-o", o])
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-ldl"])
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--only", choices=["oracle", "inputs", "chase"])
    a = ap.parse_args(argv)
    if a.only in (None, "oracle"):
        build_oracle(a.force)
    if a.only in (None, "inputs"):
        build_inputs(a.force)
    if a.only in (None, "chase"):
        build_chase(a.force)


if __name__ == "__main__":
    sys.exit(main())
