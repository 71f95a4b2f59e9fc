"""Builds libvqkv_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2603_16435_b200.build        # or __graft_entry__.build()

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
(the 'a' target is required for tcgen05/TMA PTX) and linked into one shared
library with a static CUDA runtime, so the .so is self-contained and travels
to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(OUT_DIR, "libvqkv_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC,-ffp-contract=off",
    "--expt-relaxed-constexpr",
    "-I" + os.path.join(ROOT, "include"),
    "-I" + CSRC,
]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    inc = os.path.join(ROOT, "include")
    for dp, _, fs in os.walk(inc):
        hs += [os.path.join(dp, f) for f in fs if f.endswith((".h", ".hpp"))]
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose=False, obj_dir=OBJ_DIR, extra=()):
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    if not _stale(obj, [src] + _headers()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    os.makedirs(OBJ_DIR, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


DIAG_DIR = os.path.join(ROOT, "build", "diag")
DIAG_LIB = os.path.join(DIAG_DIR, "libvqkv_b200.so")


def build_diag() -> str:
    """Diagnostics build with the encoder's per-phase clock counters compiled in
    (-DVQKV_PHASE_CLOCKS; read by vqkv_encode_phase_clocks, scripts/phase_clocks.py).
    Not the product library: load it with VQKV_LIB=build/diag/libvqkv_b200.so."""
    obj_dir = os.path.join(DIAG_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, False, obj_dir, ("-DVQKV_PHASE_CLOCKS",)), srcs))
    if _stale(DIAG_LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", DIAG_LIB, *objs, "-cudart", "static", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return DIAG_LIB


def build_variant(name: str, defines=()) -> str:
    """Development A/B build with extra -D flags into build/var/<name>.so (load it with VQKV_LIB).
    Not the product library."""
    obj_dir = os.path.join(ROOT, "build", "var", name)
    os.makedirs(obj_dir, exist_ok=True)
    lib = os.path.join(ROOT, "build", "var", name + ".so")
    srcs = _sources()
    extra = tuple("-D" + d for d in defines)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, False, obj_dir, extra), srcs))
    if _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-cudart", "static", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "build", "test_cpp_api")


def build_cpp_tests() -> str:
    """C++ drop-in test program against include/vqkv/*.hpp, linked to the library."""
    lib = build()
    deps = [CPP_TEST_SRC, lib] + _headers()
    if _stale(CPP_TEST_BIN, deps):
        os.makedirs(os.path.dirname(CPP_TEST_BIN), exist_ok=True)
        cmd = ["g++", "-O2", "-std=c++17", "-I" + os.path.join(ROOT, "include"), CPP_TEST_SRC, "-o", CPP_TEST_BIN,
               "-L" + OUT_DIR, "-lvqkv_b200", "-Wl,-rpath," + OUT_DIR, "-Wl,-rpath,$ORIGIN/../paper_2603_16435_b200/lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C++ test build failed:\n{r.stdout}\n{r.stderr}")
    return CPP_TEST_BIN


CLI_SRC = os.path.join(ROOT, "tools", "vqkv_cli.cpp")
CLI_BIN = os.path.join(ROOT, "build", "vqkv")


def build_cli() -> str:
    """The `vqkv` command-line front end (tools/vqkv_cli.cpp) over the drop-in C++ API."""
    lib = build()
    deps = [CLI_SRC, lib] + _headers()
    if _stale(CLI_BIN, deps):
        os.makedirs(os.path.dirname(CLI_BIN), exist_ok=True)
        cmd = ["g++", "-O2", "-std=c++17", "-I" + os.path.join(ROOT, "include"), CLI_SRC, "-o", CLI_BIN,
               "-L" + OUT_DIR, "-lvqkv_b200", "-Wl,-rpath," + OUT_DIR, "-Wl,-rpath,$ORIGIN/../paper_2603_16435_b200/lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    return CLI_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    print(build_cpp_tests())
