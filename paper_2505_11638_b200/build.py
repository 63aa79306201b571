"""Build libngd_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2505_11638_b200.build

The library is a plain C-ABI shared object (include/ngd.h): CUDA kernels for
sm_100a (every dense product on the in-house DMMA GEMM) + cuSOLVER's polar SVD
for ell > 512 only + NCCL for the multi-GPU all-reduce.  NCCL is linked against the torch-bundled libnccl.so.2
(same SONAME as the system copy) so one process never loads two NCCLs.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libngd_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _nccl_libdir():
    try:
        import nvidia.nccl  # type: ignore

        d = os.path.join(list(nvidia.nccl.__path__)[0], "lib")
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return d
    except Exception:
        pass
    return "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps.append(os.path.join(ROOT, "include", "ngd.h"))
    return any(os.path.getmtime(f) > t for f in deps)


def build(force=False, verbose=False, out=None, defines=()):
    """Compile every csrc/*.cu for sm_100a and link LIB (or `out`, with extra -D defines: tuning
    variants for experiments, loaded through NGD_LIB_PATH)."""
    lib_path = out or LIB
    if not force and out is None and not defines and not _stale():
        return LIB
    build_dir = BUILD if out is None else out + ".objs"
    os.makedirs(build_dir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c", src,
               "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), src))
        objs.append(obj)
    for p, src in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose and out.strip():
            print(out)
    nccl = _nccl_libdir()
    tmp = lib_path + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L/usr/local/cuda/lib64", "-lcusolver",
           f"-L{nccl}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl}:/usr/local/cuda/lib64"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout.decode())
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python -m paper_2505_11638_b200.build --variant OUT.so DEF=1 ...
        k = sys.argv.index("--variant")
        print(build(force=True, out=os.path.abspath(sys.argv[k + 1]), defines=sys.argv[k + 2:]))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
