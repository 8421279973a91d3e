"""Build the in-tree CUDA library ``paper_2008_00672_b200/lib/libfcwave_b200.so``.

nvcc cross-compiles for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``)
with ``-lineinfo`` so ncu source pages map to the kernels.  No torch types, no
JIT cache: the .so lives in the repo tree and travels to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
OBJ_DIR = os.path.join(HERE, "lib", "obj")
LIB = os.path.join(OUT_DIR, "libfcwave_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), "-I", CSRC]

SOURCES_CU = ["fcw_launch.cu", "fcw_link.cu", "fcw_cont.cu", "fcw_k_small.cu", "fcw_k_n4096z.cu", "fcw_k_n1024n.cu", "fcw_k_team.cu", "fcw_symbol.cu"] + [f"fcw_k_n{n}{g}.cu" for n in (4096, 2048, 1024) for g in "bcag"]
SOURCES_CPP = ["fcw_capi.cpp", "fcw_host.cpp"]


def _nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return p


def _cuda_include() -> str:
    return os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(_nvcc()))), "include")


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "fcwave_b200.h"))
    return hs


def _run(cmd: list[str], log: str) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ... (see {log})")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for s in SOURCES_CU:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ_DIR, s + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append(([_nvcc(), *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj], obj + ".log"))
    for s in SOURCES_CPP:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ_DIR, s + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append((["g++", *CXX_FLAGS, "-I", _cuda_include(), "-c", src, "-o", obj], obj + ".log"))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    if force or jobs or _stale(LIB, objs):
        _run([_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB, *objs, "-lcudart_static", "-lrt",
              "-lpthread", "-ldl"], os.path.join(OBJ_DIR, "link.log"))
    if verbose:
        for s in SOURCES_CU:
            with open(os.path.join(OBJ_DIR, s + ".o.log")) as f:
                print(f.read())
    return LIB


def build_variant(name: str, defines: list[str], sources: list[str]) -> str:
    """Dev-only A/B build: the default objects with `sources` recompiled under
    extra -D `defines`, linked as lib/libfcwave_b200_<name>.so (loaded when
    FCW_LIB_VARIANT=<name>)."""
    build()
    vdir = os.path.join(OUT_DIR, "obj_" + name)
    os.makedirs(vdir, exist_ok=True)
    objs = []
    jobs = []
    for s in SOURCES_CU + SOURCES_CPP:
        base = os.path.join(OBJ_DIR, s + ".o")
        if s in sources:
            obj = os.path.join(vdir, s + ".o")
            jobs.append(([_nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s),
                          "-o", obj], obj + ".log"))
            objs.append(obj)
        else:
            objs.append(base)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    lib = os.path.join(OUT_DIR, f"libfcwave_b200_{name}.so")
    _run([_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, *objs, "-lcudart_static", "-lrt",
          "-lpthread", "-ldl"], os.path.join(vdir, "link.log"))
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], sys.argv[i + 2].split(",") if len(sys.argv) > i + 2 else []
        srcs = sys.argv[i + 3].split(",") if len(sys.argv) > i + 3 else ["fcw_k_n4096b.cu"]
        if srcs == ["ALL"]:
            srcs = list(SOURCES_CU)
        print(build_variant(name, [d for d in defs if d], srcs))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
