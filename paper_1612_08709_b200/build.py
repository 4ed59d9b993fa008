"""Build the sm_100a shared library in-tree: paper_1612_08709_b200/lib/libtssvd_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo, linked against the
NCCL that ships with torch (site-packages/nvidia/nccl), rpath'd so the .so
loads on the GPU box from the same image.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libtssvd_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("NCCL headers not found (expected site-packages/nvidia/nccl)")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps.append(os.path.join(ROOT, "include", "tssvd.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """Compile every csrc/*.cu and link the library (out: another path, e.g. an A/B variant
    built with extra -D defines; loaded through TSSVD_LIB)."""
    lib_out = out or LIB
    if not force and not out and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(lib_out), exist_ok=True)
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "nvcc")
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(os.path.dirname(lib_out), os.path.basename(src) + (".ab" if out else "") + ".o")
        cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include"), "-I", inc,
               *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out)
        if verbose or "spill" in out.lower() and "0 bytes spill" not in out:
            sys.stdout.write(out)
    tmp = lib_out + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + lib, "-lcudart"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib_out)
    for o in objs:
        os.remove(o)
    return lib_out


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=None, help="A/B variant library path")
    ap.add_argument("-D", action="append", default=[], help="extra preprocessor define")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, defines=tuple(a.D)))
