"""Build libsqr.so (sm_100a) in-tree with nvcc.

    python -m paper_2008_04447_b200.build        # or __graft_entry__.build()

The library is a plain C-ABI shared object (include/sqr.h); it links the
CUDA runtime statically and has no torch dependency.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsqr.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "sqr.h")]
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines=(), name: str = "libsqr.so") -> str:
    """defines/name: variant builds (e.g. ("SQR_NN_BN=128",), "libsqr_v1.so") for experiments."""
    lib_path = os.path.join(HERE, name)
    if not force and not defines and name == "libsqr.so" and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build" if name == "libsqr.so" else "build_" + name.replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, *FLAGS, *("-D" + d for d in defines), "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out = p.communicate()[0]
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"--- nvcc failed on {src}\n{out}\n")
        elif verbose:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("libsqr build failed")
    tmp = lib_path + ".tmp"
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    names = [a[7:] for a in sys.argv[1:] if a.startswith("--name=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                name=names[0] if names else "libsqr.so"))
