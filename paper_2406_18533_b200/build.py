"""Build libgs.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2406_18533_b200.build [--force] [--ptxas-v]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgs.so")
BUILD = os.path.join(ROOT, "build", "gs")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # the NCCL torch loads (torch-bundled wheel)
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except Exception:
        pass
    return None, None


def _cudart_dir():
    try:
        import nvidia.cuda_runtime as cr
        d = os.path.join(list(cr.__path__)[0], "lib")
        return d if os.path.exists(os.path.join(d, "libcudart.so.12")) else None
    except Exception:
        return None


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    raise RuntimeError("nvcc not found")


def build(force: bool = False, ptxas_v: bool = False, verbose: bool = False, csrc: str = CSRC,
          out: str = OUT, extra=()) -> str:
    """Compile csrc/*.cu into out.  (csrc/out other than the defaults: A/B builds of another
    revision, loaded by _lib when GS_LIB_VARIANT names them.)"""
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    deps = srcs + glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h")) + \
        [os.path.join(ROOT, "include", "gs.h"), __file__]
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    build_dir = BUILD if out == OUT else BUILD + "_" + os.path.basename(out).replace(".", "_")
    os.makedirs(build_dir, exist_ok=True)
    inc, lib = _nccl_dirs()
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                    "-I" + os.path.join(ROOT, "include")] + list(extra)  # extra: A/B defines
    if inc:
        flags += ["-DGS_WITH_NCCL", "-I" + inc]
    if ptxas_v:
        flags += ["-Xptxas", "-v"]
    nvcc = _nvcc()

    def comp(src):
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        cmd = [nvcc, "-c", src, "-o", obj] + flags
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        if verbose or ptxas_v:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(comp, srcs))
    # dynamic cudart: resolve to the same libcudart.so.12 torch loads (one runtime instance,
    # so torch streams are valid handles here)
    link = [nvcc, "-shared", "--cudart", "shared", "-o", out + ".tmp"] + ARCH + objs
    crt = _cudart_dir()
    if crt:
        link += ["-Xlinker", "-rpath=" + crt]
    if lib:
        link += ["-L" + lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, ptxas_v="--ptxas-v" in sys.argv))
