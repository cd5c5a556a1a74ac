"""Build the in-tree CUDA library ``paper_1506_00014_b200/liblpradon_gpu.so``.

Explicit nvcc for sm_100a (B200); nothing is JIT-compiled or installed into
site-packages, so the built .so travels with the repository snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# Experiment variants: LPR_VARIANT=name builds liblpradon_gpu_<name>.so with
# the extra nvcc defines in LPR_DEFS (e.g. "-DLPR_RHO_RADIX9"); the default build
# is the product library.
_VARIANT = os.environ.get("LPR_VARIANT", "")
BUILD = os.path.join(PKG, "_build" + (f"_{_VARIANT}" if _VARIANT else ""))
LIB = os.path.join(PKG, "liblpradon_gpu" + (f"_{_VARIANT}" if _VARIANT else "") + ".so")
EXTRA_DEFS = os.environ.get("LPR_DEFS", "").split() if _VARIANT else []

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_LIB = "/usr/local/cuda/lib64"  # cuFFT (plan-time fp64 spectra only, lpr_spectrum.cu)
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]

CU_SOURCES = ["lpr_kernels.cu", "lpr_transpose.cu", "lpr_capi.cu", "lpr_spectrum.cu", "lpr_em.cu"]
CXX_SOURCES = ["lpr_host.cpp", "lpr_cache.cpp"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _host_cxx() -> str:
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    headers.append(os.path.join(ROOT, "include", "lpradon_gpu.h"))
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        if not os.path.exists(s):
            continue
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if _stale(o, [s] + headers):
            jobs.append(([nvcc, "-ccbin", _host_cxx(), *ARCH, *NVCC_FLAGS, *EXTRA_DEFS, "-c", s, "-o", o], o + ".log"))
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if _stale(o, [s] + headers):
            jobs.append(([_host_cxx(), "-O2", "-std=c++17", "-fPIC", "-I" + os.path.join(ROOT, "include"),
                          "-I" + CSRC, "-c", s, "-o", o], o + ".log"))
    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    if jobs or _stale(LIB, objs):
        _run([nvcc, "-ccbin", _host_cxx(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread",
              "-L" + CUDA_LIB, "-lcufft", "-Xlinker", "-rpath=" + CUDA_LIB],
             os.path.join(BUILD, "link.log"))
    build_cli()
    if verbose:
        for src in CU_SOURCES:
            log = os.path.join(BUILD, src + ".o.log")
            if os.path.exists(log):
                print(open(log).read())
    return LIB


CLI = os.path.join(PKG, "bin", "lpradon")


def build_cli() -> str:
    """The C++ command-line tool (csrc/cli: LPT1 containers + the reference's
    CLI subcommands over the C ABI), linked against the in-tree library."""
    if _VARIANT:
        return CLI
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    srcs = [os.path.join(CSRC, "cli", f) for f in ("lpt1.cpp", "lpradon_cli.cpp")]
    deps = srcs + [LIB, os.path.join(ROOT, "include", "lpradon", "lpt1.hpp"), os.path.join(ROOT, "include", "lpradon_gpu.h")]
    if _stale(CLI, deps):
        _run([_host_cxx(), "-O2", "-std=c++17", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"), *srcs,
              "-o", CLI, "-L" + PKG, "-llpradon_gpu", "-Wl,-rpath,$ORIGIN/.."], os.path.join(BUILD, "cli.log"))
    return CLI


REF_INCLUDE = "/root/reference/proj/include"
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "liblpr_ref.so")
DROPIN = os.path.join(PKG, "_dropin", "dropin_smoke")


def build_dropin() -> str | None:
    """The C++ drop-in layer (include/lpradon/lp_ops.hpp, csrc/dropin/lp_ops.cpp)
    compiled against the reference's own headers, with a smoke driver linked to
    the reference's compiled blocks (oracle/_ref). Only where /root/reference
    exists; the binary then travels to the GPU box with the tree."""
    if not (os.path.isdir(REF_INCLUDE) and os.path.exists(REF_LIB) and os.path.exists(LIB)):
        return None
    os.makedirs(os.path.dirname(DROPIN), exist_ok=True)
    srcs = [os.path.join(CSRC, "dropin", "lp_ops.cpp"), os.path.join(ROOT, "tests", "dropin", "dropin_smoke.cpp")]
    if not _stale(DROPIN, srcs + [LIB, REF_LIB, os.path.join(ROOT, "include", "lpradon", "lp_ops.hpp")]):
        return DROPIN
    _run([_host_cxx(), "-O2", "-std=c++20", "-I" + os.path.join(ROOT, "include"), "-I" + REF_INCLUDE, *srcs,
          "-o", DROPIN, LIB, REF_LIB, "-Wl,-rpath,$ORIGIN/..:$ORIGIN/../../oracle/_ref",
          "/usr/lib/x86_64-linux-gnu/libmpfr.so.6", "/usr/lib/x86_64-linux-gnu/libgmp.so.10", "-fopenmp"],
         os.path.join(BUILD, "dropin.log"))
    return DROPIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
