"""Build script: the CPU oracle (test infrastructure) and the sm_100a CUDA library (product)."""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
PKG = os.path.join(ROOT, "paper_2312_07874_b200")
LIB_SO = os.path.join(PKG, "libes_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    """torch's bundled NCCL (2.28): linking the same libnccl.so.2 torch loads keeps one NCCL per
    process whichever of torch / libes_b200.so is loaded first."""
    try:
        import nvidia.nccl
        d = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    except Exception:
        pass
    return None


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=ROOT)


def _newer(target, sources):
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(s) <= t for s in sources)


def build_oracle(force=False):
    src = [os.path.join(ROOT, "oracle", f) for f in ("oracle.cpp", "oracle.h")]
    if not force and _newer(ORACLE_SO, src):
        return ORACLE_SO
    _run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
          "-o", ORACLE_SO, src[0]])
    return ORACLE_SO


def lib_sources():
    c = os.path.join(PKG, "csrc")
    return sorted(os.path.join(c, f) for f in os.listdir(c) if f.endswith((".cu", ".cpp", ".h", ".cuh", ".inc"))) + \
        [os.path.join(ROOT, "include", "es.h")]


def build_lib(force=False, jobs=8):
    srcs = lib_sources()
    if not force and _newer(LIB_SO, srcs):
        return LIB_SO
    c = os.path.join(PKG, "csrc")
    bdir = os.path.join(ROOT, "build")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    procs = []
    inc = ["-I", os.path.join(ROOT, "include"), "-I", c]
    if os.environ.get("ES_STAMPS"):  # per-element clock stamps (ES_PHASE_TIMING diagnostics)
        inc = ["-DES_STAMPS"] + inc
    if os.environ.get("ES_NVCC_DEFS"):  # tuning experiments, e.g. "-DES_K3_THREADS=192 -DES_K3_MINB=2"
        inc = os.environ["ES_NVCC_DEFS"].split() + inc
    nd = nccl_dir()
    if nd:
        inc = ["-I", os.path.join(nd, "include")] + inc
    for f in sorted(os.listdir(c)):
        p = os.path.join(c, f)
        if f.endswith(".cu"):
            o = os.path.join(bdir, f + ".o")
            cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   *inc, "-c", p, "-o", o]
            if f == "api.cu":
                cmd = [NVCC, *ARCH, "-std=c++17", "-O2", "-Xcompiler", "-fPIC", *inc, "-c", p, "-o", o]
        elif f.endswith(".cpp"):
            o = os.path.join(bdir, f + ".o")
            cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-fopenmp", *inc, "-I", "/usr/local/cuda/include",
                   "-c", p, "-o", o]
        else:
            continue
        objs.append(o)
        print("+", " ".join(cmd), flush=True)
        log = open(o + ".log", "w")
        procs.append((subprocess.Popen(cmd, cwd=ROOT, stdout=log, stderr=subprocess.STDOUT), o, log))
        if len(procs) >= jobs:
            _wait(procs)
            procs = []
    _wait(procs)
    nccl_link = ["-lnccl"]
    if nd:
        nccl_link = ["-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
    _run([NVCC, *ARCH, "-shared", "-o", LIB_SO, *objs, "-Xcompiler", "-fopenmp",
          "-L/usr/local/cuda/lib64", "-lcudart", *nccl_link, "-lquadmath"])
    return LIB_SO


def _wait(procs):
    bad = []
    for pr, o, log in procs:
        rc = pr.wait()
        log.close()
        if rc:
            bad.append(o)
    for o in bad:
        sys.stderr.write(open(o + ".log").read())
    if bad:
        raise RuntimeError("compilation failed: " + ", ".join(bad))


if __name__ == "__main__":
    build_oracle(force="--force" in sys.argv)
    if os.path.isdir(os.path.join(PKG, "csrc")) and any(f.endswith(".cu") for f in os.listdir(os.path.join(PKG, "csrc"))):
        build_lib(force="--force" in sys.argv)
