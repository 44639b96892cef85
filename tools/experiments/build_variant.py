"""Experiment builds: libupir.so with one source compiled under extra -D flags.

    python tools/experiments/build_variant.py <name> <source.cu> -DFOO=1 ...
writes build/var/libupir_<name>.so (swap it in on the GPU box to compare)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2209_10643_b200 import build as B  # noqa: E402


def main():
    name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    out = os.path.join(ROOT, "build", "var")
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, f"{os.path.basename(src)}.{name}.o")
    path = os.environ.get("SRC_OVERRIDE", os.path.join(B.CSRC, src))   # e.g. an older revision of the file
    subprocess.run([B.NVCC] + B._flags() + ["-I" + B.CSRC] + defs + ["-c", path, "-o", obj], check=True)
    objs = [os.path.join(B.BUILD, f) for f in sorted(os.listdir(B.BUILD))
            if f.endswith(".o") and f != os.path.basename(src) + ".o"] + [obj]
    nd = B.nccl_dir()
    lib = os.path.join(out, f"libupir_{name}.so")
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs + [
        "-cudart", "static", "-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2",
        "-Xlinker", "-rpath=" + os.path.join(nd, "lib"), "-ldl"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
