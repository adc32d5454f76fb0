"""Build libhelix_b200.so in-tree for sm_100a (nvcc; no JIT, no torch extension).

    python -m paper_2507_07120_b200.build [--verbose]

The .so travels to the GPU box with the repo snapshot (it is git-ignored but
not gpurun-ignored). Incremental: objects are rebuilt only when a source or
header is newer.
"""
import argparse
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libhelix_b200.so")
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXSTD = "-std=c++17"


def nccl_dirs():
    """NCCL 2.28 from the torch-bundled nvidia-nccl wheel (same library torch loads)."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except ImportError:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "helix_b200.h")]
    objs = []
    nccl_inc, nccl_lib = nccl_dirs()
    cu_flags = [NVCC, CXXSTD, "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                "-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", nccl_inc]
    if verbose:
        cu_flags += ["-Xptxas", "-v"]
    cu_flags += os.environ.get("HX_NVCC_FLAGS", "").split()  # e.g. -DHX_DEBUG_PUSH (debug builds)
    jobs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer([src] + headers, obj):
            jobs.append(subprocess.Popen(cu_flags + ["-c", src, "-o", obj], stdout=subprocess.PIPE,
                                         stderr=subprocess.STDOUT, text=True))
    failed = False
    for j in jobs:
        out, _ = j.communicate()
        if out.strip() and (verbose or j.returncode != 0):
            print(out)
        if j.returncode != 0:
            failed = True
    if failed:
        raise RuntimeError("nvcc compilation failed")
    if force or jobs or _newer(objs, LIB):
        link = [NVCC, "-shared", *ARCH, "-Xcompiler", "-fPIC", "-cudart", "static", "-o", LIB, *objs,
                "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl_lib}",
                "-Xlinker", "--no-undefined", "-lrt", "-lpthread", "-ldl"]
        subprocess.check_call(link)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(verbose=a.verbose, force=a.force))
