"""In-tree build of the native libraries (no JIT cache, so the .so files
travel to the GPU box with the repo snapshot):

  _lib/librbe_cuda.so   sm_100a kernels + the C ABI of include/rbe_cuda.h
                        (nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo)
  _lib/librbe.so        host C++ rbe:: API (include/rbe/*.hpp) over the C ABI
  _lib/_core*.so        pybind11 module (drop-in for the reference's rbe._core)
  _lib/rbe-cuda         command-line caller (build / query subcommands of the reference CLI)

Usage: python -m paper_1802_06466_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "_lib")
OBJ = os.path.join(LIB, "obj")
INCLUDE = os.path.join(ROOT, "include")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                     "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]
NVCC_FLAGS += os.environ.get("RBE_NVCC_EXTRA", "").split()  # e.g. -DRBE_PHASE_PROF (profiling builds)
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function", f"-I{INCLUDE}"]

CU_SOURCES = ["index_kernels.cu", "scan_exact.cu", "scan_tensor.cu", "select.cu", "capi.cu"]
CU_HEADERS = ["rbe_common.cuh", "internal.h", "scan_tensor.h"]


def _newer(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if log is not None:
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
    return r


def build(force: bool = False, verbose: bool = False) -> dict:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in CU_HEADERS] + [os.path.join(INCLUDE, "rbe_cuda.h")]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append(([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o], o + ".ptxas.log"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for fut in [ex.submit(_run, c, log) for c, log in jobs]:
            fut.result()
    cuda_so = os.path.join(LIB, "librbe_cuda.so")
    if force or jobs or _newer(cuda_so, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", cuda_so] + objs)

    host_src = os.path.join(CSRC, "host", "rbe_host.cpp")
    host_hdrs = [os.path.join(INCLUDE, "rbe", h) for h in os.listdir(os.path.join(INCLUDE, "rbe"))]
    rbe_so = os.path.join(LIB, "librbe.so")
    if force or _newer(rbe_so, [host_src, cuda_so] + host_hdrs + hdrs):
        _run(["g++"] + CXX_FLAGS + ["-shared", "-o", rbe_so, host_src, f"-L{LIB}", "-lrbe_cuda",
                                    "-Wl,-rpath,$ORIGIN"])

    import pybind11

    ext = sysconfig.get_config_var("EXT_SUFFIX")
    core_so = os.path.join(LIB, "_core" + ext)
    bind_src = os.path.join(CSRC, "host", "bindings.cpp")
    if force or _newer(core_so, [bind_src, rbe_so] + host_hdrs + hdrs):
        _run(["g++"] + CXX_FLAGS + ["-shared", "-o", core_so, bind_src, f"-I{pybind11.get_include()}",
                                    f"-I{sysconfig.get_paths()['include']}", f"-L{LIB}", "-lrbe", "-lrbe_cuda",
                                    "-Wl,-rpath,$ORIGIN"])
    cli_src = os.path.join(CSRC, "host", "cli.cpp")
    cli_bin = os.path.join(LIB, "rbe-cuda")
    if force or _newer(cli_bin, [cli_src, rbe_so] + host_hdrs + hdrs):
        _run(["g++"] + [f for f in CXX_FLAGS if f != "-fPIC"] + ["-o", cli_bin, cli_src, f"-L{LIB}", "-lrbe",
                                                                   "-lrbe_cuda", "-Wl,-rpath,$ORIGIN"])
    init = os.path.join(LIB, "__init__.py")
    if not os.path.exists(init):
        open(init, "w").close()
    if verbose:
        for o in objs:
            log = o + ".ptxas.log"
            if os.path.exists(log):
                print(open(log).read())
    return {"librbe_cuda": cuda_so, "librbe": rbe_so, "core": core_so, "cli": cli_bin}


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
