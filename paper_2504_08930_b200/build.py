"""Build libvlr.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

python -m paper_2504_08930_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvlr.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch-bundled NCCL) not found")
    return list(spec.submodule_search_locations)[0]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "vlr.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile every csrc/*.cu for sm_100a and link libvlr.so. `out`/`defines`
    build a tuning variant elsewhere (tools/variants.py); the product library
    is always LIB with no extra defines."""
    lib_path = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    nd = nccl_dir()
    objs = []
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
              f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}", f"-I{os.path.join(nd, 'include')}",
              "--expt-relaxed-constexpr"]
    common += [f"-D{d}" for d in defines]
    bdir = os.path.join(HERE, "_build") if out is None else out + ".objs"
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        procs.append((src, subprocess.Popen(common + ["-c", src, "-o", obj], stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stdout.write(out)
        if p.returncode:
            failed = True
            sys.stdout.write(f"nvcc failed: {src}\n")
    if failed:
        raise RuntimeError("libvlr build failed")
    tmp = lib_path + ".tmp"
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, f"-L{os.path.join(nd, 'lib')}", "-l:libnccl.so.2",
            f"-Xlinker", f"-rpath={os.path.join(nd, 'lib')}"]
    subprocess.run(link, check=True)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
