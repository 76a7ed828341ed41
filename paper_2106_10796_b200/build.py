"""Build libcdsgd_b200.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels to the GPU box with the repo snapshot).

Links the same NCCL torch loads (pip ``nvidia/nccl`` 2.28.x, ``libnccl.so.2``)
so one process never carries two NCCL copies (SURVEY §7 toolchain note).
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libcdsgd_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    try:
        import nvidia.nccl as m  # namespace package shipped with torch's wheels

        for p in m.__path__:
            if os.path.exists(os.path.join(p, "include", "nccl.h")):
                return p
    except ImportError:
        pass
    for p in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl")):
        if os.path.exists(os.path.join(p, "include", "nccl.h")):
            return p
    raise RuntimeError("pip NCCL (nvidia/nccl) not found; torch's NCCL is required")


def sources():
    return [os.path.join(CSRC, "cdsgd_b200.cu")]


def deps():
    # every header of csrc/ (a missing one here means a stale .so after editing it)
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "cdsgd_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False, out: str = LIB) -> str:
    if out == LIB and not force and up_to_date():
        return LIB
    nd = nccl_dir()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [
        nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
        "-Xptxas", "-v" if verbose else "-O3",
        "-I", INCLUDE, "-I", CSRC, "-I", os.path.join(nd, "include"),
        *os.environ.get("CDSGD_NVCC_FLAGS", "").split(),  # development A/B builds (-D...)
        *sources(), "-o", out + ".tmp",
        "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib"),
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stdout + res.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=outs[0] if outs else LIB))
