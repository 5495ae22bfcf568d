"""In-tree build of the native libraries (no JIT cache: the .so files travel
to the GPU box with the repo snapshot).

Outputs (under paper_2505_23520_b200/lib/ and the package dir):
  libanchorattn_b200.so   C ABI + all CUDA kernels (sm_100a, -lineinfo)
  libanchorattn_cpp.so    C++ shim re-implementing the reference's
                          ``anchorattn::`` operator API over the C ABI
  anchorattn*.so          pybind11 module ``anchorattn`` (reference names)
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "build_obj")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]
NVCC_FLAGS += os.environ.get("AA_NVCC_EXTRA", "").split()  # developer experiments only

CAPI_LIB = os.path.join(LIB, "libanchorattn_b200.so")
CPP_LIB = os.path.join(LIB, "libanchorattn_cpp.so")
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
PYMOD = os.path.join(PKG, "anchorattn" + EXT)


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]) + " ...")
    return r.stdout


def build(verbose: bool = False, force: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objs = []
    jobs = []
    for cu in cus:
        o = os.path.join(OBJ, os.path.basename(cu) + ".o")
        objs.append(o)
        if force or _newer(o, [cu] + headers):
            jobs.append((cu, o))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        futs = [ex.submit(_run, [NVCC] + NVCC_FLAGS + ["-Xptxas", "-v", "-c", cu, "-o", o])
                for cu, o in jobs]
        for f in futs:
            out = f.result()
            if verbose:
                print(out)
    if force or jobs or _newer(CAPI_LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", CAPI_LIB] + objs + ["-lcuda"])

    shim_dir = os.path.join(CSRC, "shim")
    shim_src = os.path.join(shim_dir, "anchorattn.cpp")
    shim_hdr = os.path.join(shim_dir, "anchorattn.hpp")
    cxxflags = ["-O2", "-std=c++20", "-fPIC", "-Wall", "-I", INCLUDE, "-I", shim_dir]
    if force or _newer(CPP_LIB, [shim_src, shim_hdr, CAPI_LIB] + headers):
        _run([CXX] + cxxflags + ["-shared", "-o", CPP_LIB, shim_src, "-L", LIB,
                                  "-lanchorattn_b200", "-Wl,-rpath,$ORIGIN"])

    bind_src = os.path.join(shim_dir, "bindings.cpp")
    if force or _newer(PYMOD, [bind_src, shim_hdr, CPP_LIB]):
        import pybind11

        _run([CXX] + cxxflags + ["-shared", "-o", PYMOD, bind_src,
                                  "-I", pybind11.get_include(),
                                  "-I", sysconfig.get_paths()["include"],
                                  "-L", LIB, "-lanchorattn_cpp", "-lanchorattn_b200",
                                  "-Wl,-rpath,$ORIGIN/lib"])


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print("built", CAPI_LIB, CPP_LIB, PYMOD)
