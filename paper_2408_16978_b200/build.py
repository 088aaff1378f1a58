"""Build the in-tree CUDA libraries for sm_100a with nvcc (no GPU needed).

    python -m paper_2408_16978_b200.build

* ``paper_2408_16978_b200/libfpdt.so`` — the product: C-ABI in include/fpdt.h.
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


def _cublas_lib():
    """The torch-bundled libcublas.so.12 (the copy torch itself loads, so the process holds one cuBLAS); the
    fused QKV projection GEMMs of fpdt_block_fwd/bwd call it.  Headers come from the CUDA toolkit."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    for r in roots:
        lib = os.path.join(r, "cublas", "lib")
        if os.path.exists(os.path.join(lib, "libcublas.so.12")):
            return lib
    return "/usr/local/cuda/lib64"


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_product(force: bool = False) -> str:
    csrc = os.path.join(PKG, "csrc")
    cu = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(csrc, "*.cpp")))
    deps = cu + cpp + glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    out = os.path.join(PKG, "libfpdt.so")
    if not force and not _stale(out, deps):
        return out
    nccl_inc, nccl_lib = _nccl_dirs()
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in cu + cpp:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + deps):
            cmd = [NVCC] + COMMON + ["-I", os.path.join(ROOT, "include"), "-I", csrc, "-I", nccl_inc,
                                     "-c", src, "-o", obj]
            print(" ".join(cmd), flush=True)
            procs.append(subprocess.Popen(cmd))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out] + objs +
         ["-L", nccl_lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={nccl_lib}", "-L", _cublas_lib(), "-l:libcublas.so.12",
          f"-Xlinker=-rpath={_cublas_lib()}", "-lpthread"])
    return out


def build_generator(force: bool = False) -> str:
    src = os.path.join(ROOT, "fpdt_inputs", "gen_dev.cu")
    out = os.path.join(ROOT, "fpdt_inputs", "libfpdt_gen.so")
    if force or _stale(out, [src]):
        _run([NVCC] + COMMON + ["-shared", "-o", out, src])
    return out


def build_all(force: bool = False):
    return build_product(force), build_generator(force)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv))
