"""Build libcpd.so in-tree for sm_100a (nvcc; no torch extension machinery).

Each csrc/*.cu compiles to its own object in parallel (build/obj/), then one nvcc link
produces the shared library."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcpd.so")
OBJ = os.path.join(ROOT, "build", "obj")


def nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("NCCL headers not found (nvidia.nccl package)")
    return list(spec.submodule_search_locations)[0]


def build(verbose=False, force=False):
    srcs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.h"))) + [os.path.join(ROOT, "include", "cpd.h")]
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(f) <= t for f in srcs + hdrs + [__file__]):
            return LIB
    nd = nccl_dir()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include")]
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(os.path.getmtime(f) for f in hdrs + [__file__])

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
            return obj, None
        r = subprocess.run([nvcc, *flags, "-c", src, "-o", obj + ".tmp"], capture_output=True, text=True)
        if r.returncode != 0:
            return obj, r.stdout + r.stderr
        os.replace(obj + ".tmp", obj)
        if verbose:
            sys.stderr.write(r.stderr)
        return obj, None

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        res = list(ex.map(compile_one, srcs))
    errs = [e for _, e in res if e]
    if errs:
        sys.stderr.write("\n".join(errs))
        raise RuntimeError("nvcc failed building libcpd.so")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *[o for o, _ in res],
           "-o", LIB + ".tmp", "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libcpd.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv or "--force" in sys.argv)
    print(LIB)
