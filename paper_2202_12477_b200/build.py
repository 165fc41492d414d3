"""Build libhipbone_b200.so in-tree with nvcc for sm_100a (no torch extension machinery:
the library exports a plain C ABI, include/hipbone_b200.h)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# HB_LIBDIR: tuning harnesses build several flavours side by side (the package loads lib/)
LIBDIR = os.environ.get("HB_LIBDIR") or os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libhipbone_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        cand = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("NCCL headers not found under the nvidia python packages")


SOURCES = ["mesh.cpp", "op.cu"]


def _stamp_name() -> str:
    """Build flavour of the library on disk (plain, or a tuning build for one / all degrees)."""
    if not os.environ.get("HB_TUNE"):
        return ".plain"
    return ".tune" + (f"_n{int(os.environ['HB_TUNE_N'])}" if os.environ.get("HB_TUNE_N") else "")


def _compile(src: str, nccl: str, extra: list[str]) -> str:
    obj = os.path.join(LIBDIR, os.path.splitext(src)[0] + ".o")
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
           "-Xptxas", "-v" if os.environ.get("HB_PTXAS_V") else "-O3",
           *(["-DHB_TUNE"] if os.environ.get("HB_TUNE") else []),
           *([f"-DHB_TUNE_N={int(os.environ['HB_TUNE_N'])}"] if os.environ.get("HB_TUNE") and os.environ.get("HB_TUNE_N") else []),
           *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if os.environ.get("HB_PTXAS_V"):
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, extra: list[str] | None = None) -> str:
    if os.environ.get("HB_PREBUILT") and os.path.exists(LIB):  # tuning harness: library swapped in
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(ROOT, "include", "hipbone_b200.h"))
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        stamp = os.path.join(LIBDIR, _stamp_name())
        if all(os.path.getmtime(f) < t for f in srcs + hdrs + [__file__]) and os.path.exists(stamp):
            return LIB
    nccl = nccl_root()
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, nccl, extra or []), SOURCES))
    cmd = [NVCC, "-shared", *ARCH, "-o", LIB, *objs, "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    for o in objs:
        os.remove(o)
    for st in os.listdir(LIBDIR):
        if st.startswith((".tune", ".plain")):
            os.remove(os.path.join(LIBDIR, st))
    open(os.path.join(LIBDIR, _stamp_name()), "w").close()
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
