"""Build the C-ABI shared library libp2p_b200.so in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libp2p_b200.so")
PEAKS_LIB = os.path.join(LIBDIR, "libp2p_peaks.so")
INCLUDE = os.path.join(ROOT, "include")

SOURCES = ["p2p_capi.cu", "plan_builder.cpp"]
DEPS = SOURCES + ["p2p_kernels.cuh", "plan.h", "plan_device.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-pthread",
    "-Xptxas", "-v",
    "-cudart", "static",
    "-shared",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale(lib: str, deps: list[str]) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in deps)


def _nvcc(sources: list[str], out: str, log: str, verbose: bool, extra: tuple[str, ...] = ()):
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, *sources, "-o", tmp, "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stdout + res.stderr)
    with open(os.path.join(LIBDIR, log), "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> str:
    """Build libp2p_b200.so (the operator) and libp2p_peaks.so (roofline microbenchmarks)."""
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(INCLUDE, "p2p.h")]
    if force or stale(LIB, deps):
        _nvcc([os.path.join(CSRC, s) for s in SOURCES], LIB, "ptxas.log", verbose)
    pdeps = [os.path.join(CSRC, "peaks.cu"), os.path.join(INCLUDE, "p2p_peaks.h"),
             os.path.join(CSRC, "p2p_kernels.cuh")]
    if force or stale(PEAKS_LIB, pdeps):
        _nvcc([os.path.join(CSRC, "peaks.cu")], PEAKS_LIB, "ptxas_peaks.log", verbose)
    return LIB


def build_variant(name: str, defines: list[str]) -> str:
    """A/B experiments: the operator library built with extra -D defines as lib/libp2p_b200_<name>.so
    (load it with P2P_LIB=<path>)."""
    out = os.path.join(LIBDIR, f"libp2p_b200_{name}.so")
    _nvcc([os.path.join(CSRC, s) for s in SOURCES], out, f"ptxas_v_{name}.log", False,
          tuple("-D" + d for d in defines))
    return out


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2 and sys.argv[1] == "variant":  # python _build.py variant NAME DEF=1 ...
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        print(build(force=True, verbose=True))
