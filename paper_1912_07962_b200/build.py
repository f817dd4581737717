"""Build the in-tree CUDA library ``libslimb200.so`` for sm_100a.

``python -m paper_1912_07962_b200.build`` (or ``__graft_entry__.build()``)
compiles every ``csrc/*.cu`` with nvcc for ``-gencode
arch=compute_100a,code=sm_100a`` and the host helpers with g++, then links
one shared library next to this file.  Objects are cached by content hash
under ``build/`` so rebuilding after a one-file edit is quick.
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJDIR = os.path.join(ROOT, "build", "obj")
# SLIM_BUILD_TAG=<tag>: an alternate build (e.g. another digit layout via
# SLIM_NVCC_EXTRA) into libslimb200_<tag>.so, loaded with SLIM_LIB=<path>
_TAG = os.environ.get("SLIM_BUILD_TAG", "")
LIB = os.path.join(HERE, f"libslimb200_{_TAG}.so" if _TAG else "libslimb200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills", *GENCODE, f"-I{INCLUDE}", f"-I{CSRC}",
              *os.environ.get("SLIM_NVCC_EXTRA", "").split()]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", f"-I{INCLUDE}"]


def _sources():
    cu = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    cpp = sorted(f for f in os.listdir(CSRC) if f.endswith(".cpp"))
    return cu, cpp


def _digest(path, flags):
    h = hashlib.sha256()
    h.update(" ".join(flags).encode())
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cuh", ".h")):
            with open(os.path.join(CSRC, name), "rb") as fh:
                h.update(fh.read())
    with open(os.path.join(INCLUDE, "slimb200.h"), "rb") as fh:
        h.update(fh.read())
    with open(path, "rb") as fh:
        text = fh.read()
    h.update(text)
    for name in sorted(os.listdir(CSRC)):  # a source that includes another .cu (chol_q6.cu)
        if name.endswith(".cu") and f'#include "{name}"'.encode() in text:
            with open(os.path.join(CSRC, name), "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def _compile(args):
    cmd, obj = args
    if os.path.exists(obj):
        return obj, ""
    tmp = obj + ".tmp.o"
    proc = subprocess.run(cmd + ["-o", tmp], capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    os.replace(tmp, obj)
    return obj, proc.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    cu, cpp = _sources()
    jobs = []
    for f in cu:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJDIR, f"{f}.{_digest(src, NVCC_FLAGS)}.o")
        jobs.append(([NVCC, *NVCC_FLAGS, "-c", src], obj))
    for f in cpp:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJDIR, f"{f}.{_digest(src, CXX_FLAGS)}.o")
        jobs.append((["g++", *CXX_FLAGS, "-c", src], obj))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as pool:
        results = list(pool.map(_compile, jobs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log.strip():
                print(log)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *GENCODE, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-lcudart"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    os.replace(tmp, LIB)
    return LIB


def clean():
    shutil.rmtree(os.path.join(ROOT, "build"), ignore_errors=True)
    if os.path.exists(LIB):
        os.remove(LIB)


if __name__ == "__main__":
    if "--clean" in sys.argv:
        clean()
    print(build(verbose=True))
