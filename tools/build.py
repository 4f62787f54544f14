"""Build every native artefact in-tree.

  harness/libhgen.so                 seeded input generator (test/bench infra)
  oracle/liboracle.so                fp64 oracle (test infra; built, never linked to the product)
  paper_2403_01164_b200/libhg.so     the product: C-ABI library (CUDA sm_100a + host C++)

The product and the oracle are separate compilations with no shared sources.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=ROOT):
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]) + " ...")
    return r.stdout + r.stderr


def _newer(out, srcs):
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(s) <= t for s in srcs)


def build_harness(force=False):
    src = os.path.join(ROOT, "harness", "gen.c")
    out = os.path.join(ROOT, "harness", "libhgen.so")
    if force or not _newer(out, [src]):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", out, src, "-lpthread", "-lm"])
    return out


def build_oracle(force=False):
    src = os.path.join(ROOT, "oracle", "oracle.c")
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or not _newer(out, [src]):
        # no -ffast-math: the fp64 sum stays in source order (no reassociation, no FMA)
        _run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", out, src, "-lpthread"])
    return out


PKG = os.path.join(ROOT, "paper_2403_01164_b200")
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")

# (source, kind) -- kind selects the compiler and flags
PRODUCT_SOURCES = [
    ("plan.cpp", "cxx"),
    ("host_gemv.cpp", "cxx_avx512"),
    ("host_gemv_avx2.cpp", "cxx_avx2"),
    ("host_gemv_amx.cpp", "cxx_amx"),
    ("threadpool.cpp", "cxx"),
    ("host_glue.cpp", "cxx_avx2"),
    ("pinlane.cpp", "cxx"),
    ("gemv_sm100.cu", "cu"),
    ("gemv_tc_sm100.cu", "cu"),
    ("glue_sm100.cu", "cu"),
    ("peer.cu", "cu"),
    ("runtime.cu", "cu"),
    ("dist.cpp", "cxx"),
    ("numa.cpp", "cxx"),
]


def _product_objs(force=False, verbose=False):
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    hdrs = [os.path.join(INC, f) for f in os.listdir(INC)] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    common = ["-O3", "-fPIC", "-I" + INC, "-I" + CSRC, "-ffp-contract=off", "-fvisibility=hidden"]
    jobs = []
    for src, kind in PRODUCT_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        if kind == "cu":
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
                   "-fPIC,-fvisibility=hidden,-ffp-contract=off", "-I" + INC, "-I" + CSRC,
                   "--fmad=true", "-Xptxas", "-v", "-c", s, "-o", o]
        else:
            isa = {"cxx": [], "cxx_avx512": ["-mavx512f", "-mavx512bw", "-mavx512vl", "-mavx512bf16",
                                               "-mfma"],
                   "cxx_avx2": ["-mavx2", "-mfma", "-mf16c"],
                   "cxx_amx": ["-mavx512f", "-mavx512bw", "-mavx512vl", "-mavx512bf16", "-mfma", "-mamx-tile",
                               "-mamx-bf16"]}[kind]
            cmd = ["g++", "-std=c++17", *common, *isa, "-I" + os.path.join(CUDA, "include"),
                   "-c", s, "-o", o]
        jobs.append((cmd, o, [s] + hdrs))
    todo = [j for j in jobs if force or not _newer(j[1], j[2])]
    with ThreadPoolExecutor(max_workers=8) as ex:
        logs = list(ex.map(lambda j: _run(j[0]), todo))
    if verbose:
        for l in logs:
            sys.stdout.write(l)
    return [j[1] for j in jobs], bool(todo)


def build_product(force=False, verbose=False):
    objs, changed = _product_objs(force, verbose)
    out = os.path.join(PKG, "libhg.so")
    if force or changed or not os.path.exists(out):
        # static cudart (nvcc default) so the library does not depend on torch's runtime copy;
        # NCCL is dlopen'ed on demand by dist.cpp (no link-time dependency).
        _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lpthread", "-ldl"])
    return out


def build_all(force=False, verbose=False):
    build_harness(force)
    build_oracle(force)
    return build_product(force, verbose)


if __name__ == "__main__":
    force = "--force" in sys.argv
    if "--oracle-only" in sys.argv:
        print(build_harness(force), build_oracle(force))
    else:
        print(build_all(force, verbose="-v" in sys.argv))
