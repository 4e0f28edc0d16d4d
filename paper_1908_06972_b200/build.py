"""Build libckks.so in-tree: nvcc for sm_100a (no torch in the ABI, no JIT cache)."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libckks.so")
SOURCES = ["kernels.cu", "codec.cu", "p2p.cu", "chunkdot_tc.cu", "ks_cluster.cu", "ckks.cu", "hostmath.cpp"]
HEADERS = ["modarith.cuh", "ntt.cuh", "internal.h", "hostmath.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I", os.path.join(ROOT, "include")]
CUFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-diag-suppress", "177", *INC]


def _digest(extra: list | None = None) -> str:
    """Content hash of every source, header and flag that goes into the library."""
    h = hashlib.sha256()
    for f in [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ckks.h")]:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    h.update(" ".join(ARCH + CUFLAGS + (extra or [])).encode())
    return h.hexdigest()


def _stale() -> bool:
    """Rebuild unless libckks.so carries the digest of exactly these sources (mtimes are not
    trusted: a snapshot copied to another machine keeps a .so beside possibly newer sources)."""
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".sha256"):
        return True
    with open(LIB + ".sha256") as fh:
        return fh.read().strip() != _digest()


def build(force: bool = False, verbose: bool = False, variant: str = "", defines: tuple = ()) -> str:
    """Compile every CUDA/C++ source for sm_100a and link libckks.so (static cudart).
    variant/defines: an A/B build libckks_<variant>.so with extra -D flags (dev experiments;
    loaded when CKKS_LIB_VARIANT=<variant>)."""
    if variant:
        out = os.path.join(PKG, f"libckks_{variant}.so")
        return _compile(out, [f"-D{d}" for d in defines], verbose)
    if not force and (not _stale() or os.environ.get("CKKS_NO_BUILD")):  # CKKS_NO_BUILD: A/B runs
        return LIB
    return _compile(LIB, [], verbose)


def _compile(LIB: str, extra: list, verbose: bool) -> str:
    digest = _digest(extra)
    cmds, objs = [], []
    for src in SOURCES:
        obj = os.path.join("/tmp", f"libckks_{os.getpid()}_{src}.o")
        if src.endswith(".cpp"):
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", *INC, "-c", os.path.join(CSRC, src), "-o", obj]
        else:
            cmd = [NVCC, *ARCH, *CUFLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs])
    os.replace(tmp, LIB)
    if not extra:
        with open(LIB + ".sha256", "w") as fh:
            fh.write(digest + "\n")
    for o in objs:
        os.remove(o)
    return LIB


def build_int_peak(force: bool = False) -> str:
    """bench/libintpeak.so: the integer-pipe peak microbenchmark used by bench.py's roofline."""
    src = os.path.join(ROOT, "bench", "int_peak.cu")
    so = os.path.join(ROOT, "bench", "libintpeak.so")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        tmp = so + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", tmp, src])
        os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
