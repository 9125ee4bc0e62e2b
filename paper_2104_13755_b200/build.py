"""Build libmg.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2104_13755_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libmg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = GENCODE + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INC}", f"-I{CSRC}"]
# experiment builds only (tools/): extra -D flags; part of the source hash
NVCC_FLAGS += os.environ.get("MG_NVCC_DEFINES", "").split()
CU_SOURCES = ["mg_vcycle.cu", "mg_setup.cu", "mg_krylov.cu"]
CPP_SOURCES = ["mg_host.cpp"]


def _sources():
    return [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES] + \
        [os.path.join(CSRC, "mg_internal.h"), os.path.join(CSRC, "mg_common.cuh"), os.path.join(INC, "mg.h")]


def source_hash():
    """sha256 over every source, header and the compile flags: the library is
    rebuilt whenever this differs from the hash recorded beside it (file
    mtimes do not survive the copy to the GPU box reliably)."""
    import hashlib
    h = hashlib.sha256()
    h.update(" ".join(NVCC_FLAGS + CU_SOURCES + CPP_SOURCES).encode())
    for s in _sources():
        with open(s, "rb") as f:
            h.update(os.path.basename(s).encode())
            h.update(f.read())
    return h.hexdigest()


HASH_FILE = LIB + ".sha256"


def up_to_date():
    if not (os.path.exists(LIB) and os.path.exists(HASH_FILE)):
        return False
    with open(HASH_FILE) as f:
        return f.read().strip() == source_hash()


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    for f in CU_SOURCES + CPP_SOURCES:
        src = os.path.join(CSRC, f)
        obj = os.path.join(LIBDIR, f + ".o")
        extra = ["-Xptxas", "-v"] if (verbose and f.endswith(".cu")) else []
        cmd = [NVCC, *NVCC_FLAGS, *extra, "-c", src, "-o", obj]
        if f.endswith(".cpp"):
            cmd = [NVCC, *NVCC_FLAGS, "-x", "c++", "-c", src, "-o", obj]
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *GENCODE, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    with open(HASH_FILE, "w") as f:
        f.write(source_hash() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
