"""Build the in-tree CUDA libraries for sm_100a with nvcc (no GPU needed).

    python -m paper_2408_16978_b200.build

* ``paper_2408_16978_b200/libfpdt.so`` — the product: C-ABI in include/fpdt.h.
* ``paper_2408_16978_b200/libfpdt_diag.so`` — diagnostics (include/fpdt_diag.h: micro-benchmarks, direct pair /
  layout kernel launches), linked against libfpdt.so; not on the FPDT path.
* ``fpdt_inputs/libfpdt_gen.so``       — the seeded input generator's device twin (test/bench infra).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                 "--expt-relaxed-constexpr", "-cudart", "static"]
# experiment knobs (e.g. FPDT_NVCC_DEFINES="-DFPDT_BWD_EXP=1"); empty for every product build
COMMON += os.environ.get("FPDT_NVCC_DEFINES", "").split()


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("NCCL headers not found (expected the torch-bundled nvidia-nccl wheel)")


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _compile(sources, deps, objdir, force, extra_inc=()):
    nccl_inc, _ = _nccl_dirs()
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in sources:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + deps):
            cmd = [NVCC] + COMMON + ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc"),
                                     "-I", nccl_inc] + [a for d in extra_inc for a in ("-I", d)] + ["-c", src, "-o", obj]
            print(" ".join(cmd), flush=True)
            procs.append(subprocess.Popen(cmd))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    return objs


def _headers():
    csrc = os.path.join(PKG, "csrc")
    return glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def build_product(force: bool = False) -> str:
    csrc = os.path.join(PKG, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu"))) + sorted(glob.glob(os.path.join(csrc, "*.cpp")))
    deps = srcs + _headers()
    out = os.path.join(PKG, "libfpdt.so")
    if not force and not _stale(out, deps):
        return out
    _, nccl_lib = _nccl_dirs()
    objs = _compile(srcs, deps, os.path.join(PKG, "build"), force)
    _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out] + objs +
         ["-L", nccl_lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={nccl_lib}", "-lpthread"])
    return out


def build_diag(force: bool = False) -> str:
    """The diagnostics library: csrc/diag/*, linked against libfpdt.so (rpath $ORIGIN)."""
    ddir = os.path.join(PKG, "csrc", "diag")
    srcs = sorted(glob.glob(os.path.join(ddir, "*.cu"))) + sorted(glob.glob(os.path.join(ddir, "*.cpp")))
    prod = build_product(force)
    deps = srcs + _headers() + [prod]
    out = os.path.join(PKG, "libfpdt_diag.so")
    if not force and not _stale(out, deps):
        return out
    objs = _compile(srcs, srcs + _headers(), os.path.join(PKG, "build", "diag"), force)
    _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out] + objs +
         ["-L", PKG, "-l:libfpdt.so", "-Xlinker=-rpath=$ORIGIN", "-lpthread"])
    return out


def build_generator(force: bool = False) -> str:
    src = os.path.join(ROOT, "fpdt_inputs", "gen_dev.cu")
    out = os.path.join(ROOT, "fpdt_inputs", "libfpdt_gen.so")
    if force or _stale(out, [src]):
        _run([NVCC] + COMMON + ["-shared", "-o", out, src])
    return out


def build_all(force: bool = False):
    return build_product(force), build_diag(force), build_generator(force)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv))
