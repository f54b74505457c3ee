"""Build libbmc.so (sm_100a) in-tree with nvcc.  No JIT cache, no torch extension:
the .so sits next to this file and travels with the repo snapshot."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libbmc.so")
SOURCES = ["cache_kernels.cu", "attn_decode.cu", "attn_tc.cu", "attn_tck.cu", "arena.cpp", "bmc_abi.cpp"]
HEADERS = ["bmc_internal.h", "combine.cuh", "tc_common.cuh", os.path.join("..", "..", "include", "bmc.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = SO, defines=()) -> str:
    """out / defines: experiment builds only (e.g. the -DBMC_TC_TRACE timeline
    library used by tools/tck_trace.py); the product is SO without defines."""
    if out == SO and not defines and not force and not _stale():
        return SO
    objs = []
    bdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(defines))
    os.makedirs(bdir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               *[f"-D{d}" for d in defines],
               "-I", os.path.join(HERE, "..", "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs]
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    if "--trace" in sys.argv:   # clock64 timeline build for tools/tck_trace.py / tc_trace.py
        print(build(out=os.path.join(HERE, "..", "tools", "exp", "libbmc_trace.so"),
                    defines=("BMC_TC_TRACE",)))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(SO)
