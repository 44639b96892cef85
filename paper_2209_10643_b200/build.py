"""Build libupir.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2209_10643_b200.build [--force]

Each .cu is compiled to an object in build/ (in parallel), then linked into
paper_2209_10643_b200/libupir.so against the CUDA runtime (static) and the
NCCL shipped with the torch wheel (nvidia/nccl), with an rpath to it.
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "upir")
LIB = os.path.join(PKG, "libupir.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    site = sysconfig.get_paths()["purelib"]
    d = os.path.join(site, "nvidia", "nccl")
    if os.path.exists(os.path.join(d, "include", "nccl.h")):
        return d
    raise RuntimeError("NCCL headers not found under " + d)


def _flags():
    nd = nccl_dir()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default",
                   "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nd, "include"),
                   "--expt-relaxed-constexpr"]


def _deps_mtime():
    files = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "upir.h"), __file__]
    return max(os.path.getmtime(f) for f in files)


def build(force=False, verbose=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    flags = _flags()
    hdr_mtime = max(os.path.getmtime(f) for f in glob.glob(os.path.join(CSRC, "*.h")) +
                    glob.glob(os.path.join(CSRC, "*.cuh")) +
                    [os.path.join(ROOT, "include", "upir.h")])

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(src)
                and os.path.getmtime(obj) >= hdr_mtime):
            return obj
        cmd = [NVCC] + flags + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(compile_one, srcs))
    nd = nccl_dir()
    tmp = LIB + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + [
        "-cudart", "static", "-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2",
        "-Xlinker", "-rpath=" + os.path.join(nd, "lib"), "-lcuda" if False else "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
