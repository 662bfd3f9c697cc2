"""Build libtc.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2006_15512_b200.build

The shared library lands in ``paper_2006_15512_b200/lib/libtc.so`` (git-ignored,
shipped to the GPU box with the working tree).  cudart is linked statically so
the library does not depend on torch's CUDA runtime version.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libtc.so")
FLAT_SRC = os.path.join(CSRC, "flatten_ext.c")

SOURCES = ["plan.cpp", "compile.cpp", "factor.cpp", "decompose.cpp", "runtime.cu"]
HEADERS = ["plan.hpp", "compile.hpp", "program.h", "kernels.cuh", "ograph.hpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def flat_ext_path() -> str:
    import sysconfig

    return os.path.join(PKG, "lib", "_tcflat" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_flat_ext(force: bool = False, verbose: bool = False) -> str:
    """The native host-side flattener (CPython C API, gcc): _tcflat.*.so."""
    import sysconfig

    out = flat_ext_path()
    if not force and not _stale(out, [FLAT_SRC, os.path.abspath(__file__)]):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    import numpy

    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-std=c11", "-Wall",
           "-I", sysconfig.get_paths()["include"], "-I", numpy.get_include(), FLAT_SRC, "-o", out + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    build_flat_ext(force=force and out is None, verbose=verbose)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "tc.h"))
    deps.append(os.path.join(ROOT, "include", "tc_factor.h"))
    deps.append(os.path.join(ROOT, "include", "tc_decompose.h"))
    deps.append(os.path.abspath(__file__))
    lib_out = out or LIB
    os.makedirs(os.path.dirname(lib_out), exist_ok=True)
    # one object per source (compiled in parallel, each rebuilt only when it or a
    # header changed), then one link: editing a host .cpp does not recompile the
    # kernels in runtime.cu
    objdir = os.path.join(os.path.dirname(lib_out), "obj" + ("" if out is None else "_" + os.path.basename(out)))
    os.makedirs(objdir, exist_ok=True)
    defs = os.environ.get("TC_NVCC_DEFS", "").split()
    common = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", *defs, "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-O3",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    hdr = [d for d in deps if not d.endswith(tuple(SOURCES))]
    jobs = []
    objs = []
    import hashlib

    hh = hashlib.sha256()
    for d in hdr:
        with open(d, "rb") as fh:
            hh.update(fh.read())
    for f in SOURCES:
        src = os.path.join(CSRC, f)
        obj = os.path.join(objdir, f + ".o")
        stamp = obj + ".flags"
        # the stamp holds the flags and a hash of the source and headers (an
        # mtime check misses an edit made while the previous compile ran)
        h = hh.copy()
        with open(src, "rb") as fh:
            h.update(fh.read())
        flags = " ".join(common) + "\n" + h.hexdigest()
        objs.append(obj)
        old = open(stamp).read() if os.path.exists(stamp) else None
        if force or old != flags or not os.path.exists(obj):
            jobs.append(([*common, "-c", src, "-o", obj + ".tmp"], obj, stamp, flags))

    def run(job):
        cmd, obj, stamp, flags = job
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(obj + ".tmp", obj)
        with open(stamp, "w") as fh:
            fh.write(flags)

    if jobs:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(len(jobs)) as ex:
            list(ex.map(run, jobs))
    elif not force and os.path.exists(lib_out) and not _stale(lib_out, objs):
        return lib_out
    cmd = [nvcc(), *ARCH, "-shared", *objs, "-o", lib_out + ".tmp", "-lpthread", "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(lib_out + ".tmp", lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
