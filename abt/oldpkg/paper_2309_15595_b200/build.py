"""Build libchase.so in-tree with nvcc for sm_100a (B200).  Run: python -m paper_2309_15595_b200.build"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libchase.so")
SOURCES = ["chase.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".inc")))   # every included file


def nccl_dirs():
    """NCCL that torch loads (nvidia-nccl wheel) so both share one libnccl.so.2 in-process."""
    try:
        import nvidia.nccl as nn  # noqa: F401
        base = os.path.dirname(list(nn.__path__)[0] + "/")
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "chase.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True, out: str | None = None, defines=()) -> str:
    lib_out = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    inc, lib = nccl_dirs()
    cmd = [
        "nvcc", "-O3", "-std=c++17", "-lineinfo",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
        *[os.path.join(CSRC, s) for s in SOURCES],
        *[f"-D{d}" for d in defines],
        "-o", lib_out + ".tmp",
        "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}",
    ]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build.log")
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libchase.so (see paper_2309_15595_b200/build.log)")
    os.replace(lib_out + ".tmp", lib_out)
    return lib_out


if __name__ == "__main__":
    # python -m paper_2309_15595_b200.build [--force] [--out PATH -DNAME=V ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print("built", build(force="--force" in args, out=out, defines=defs))
