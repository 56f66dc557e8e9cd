"""Build libmf_b200.so in-tree with nvcc for sm_100a (and the oracle's C
library, which only the tests use).  `python -m paper_1910_13247_b200.build`."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmf_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"torch-bundled NCCL headers not found under {base}")
    return inc, lib


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) + glob.glob(os.path.join(HERE, "csrc", "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = (sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh"))
            + [os.path.join(ROOT, "include", "mf.h")])
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every csrc/ source with nvcc for sm_100a and link LIB (or `out`)."""
    lib_path = out or LIB
    if not force and not defines and not needs_build():
        return LIB
    inc, lib = nccl_dirs()
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.lower() for d in defines))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", inc,
               "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr", *[f"-D{d}" for d in defines],
               "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = []
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for p, cmd in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [NVCC, *ARCH, "-shared", "-o", lib_path, *objs, "-L", lib, "-l:libnccl.so.2",
            f"-Xlinker=-rpath={lib}", "-lcudart"]
    subprocess.check_call(link)
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
