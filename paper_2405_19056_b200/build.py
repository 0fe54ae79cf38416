"""Build the in-tree shared libraries for sm_100a (nvcc cross-compiles without a GPU).

  libglassnet.so         product: kernels + C ABI (include/glassnet.h)
  synth/libglassnet_synth.so   harness: device twin of the seeded input generator
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libglassnet.so")
SYNTH_SRC = os.path.join(ROOT, "synth", "synth_dev.cu")
SYNTH_LIB = os.path.join(ROOT, "synth", "libglassnet_synth.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("torch's NCCL (nvidia/nccl) not found")


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _sources(d, exts):
    return sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith(exts))


def build_lib(force=False, verbose=True):
    srcs = _sources(CSRC, (".cu",))
    deps = srcs + _sources(CSRC, (".cuh", ".h")) + [os.path.join(ROOT, "include", "glassnet.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    nccl = _nccl_dir()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if os.environ.get("GN_PTXAS_V") else "-O3",
           *os.environ.get("GN_EXTRA_NVCC", "").split(),
           "-I", os.path.join(nccl, "include"), "-o", LIB, *srcs,
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return LIB


def build_profile_lib(verbose=True, name="libglassnet_prof.so", defines=("GN_TB_PROF",)):
    """Diagnostic variant (bench configuration's T kernel only): by default with the T
    kernel's per-role clock64 counters (-DGN_TB_PROF); `defines` selects ablation switches."""
    global LIB
    keep = LIB
    LIB = os.path.join(PKG, name)
    try:
        os.environ["GN_EXTRA_NVCC"] = " ".join("-D" + d for d in ("GN_DIAG_K8_ONLY",) + tuple(defines))
        return build_lib(force=True, verbose=verbose)
    finally:
        os.environ.pop("GN_EXTRA_NVCC", None)
        LIB = keep


def build_synth(force=False, verbose=True):
    if not force and not _stale(SYNTH_LIB, [SYNTH_SRC]):
        return SYNTH_LIB
    cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-fmad=false", "-shared", "-Xcompiler", "-fPIC",
           "-o", SYNTH_LIB, SYNTH_SRC]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return SYNTH_LIB


def build_all(force=False):
    build_lib(force)
    build_synth(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
