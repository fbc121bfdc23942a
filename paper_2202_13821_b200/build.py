"""Build the in-tree CUDA library libhgks_b200.so for sm_100a.

nvcc cross-compiles without a GPU. The library is split into translation
units per (degree, dim) family so the build parallelises; every unit is
compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
LIB = os.environ.get("HGKS_LIB") or os.path.join(HERE, "libhgks_b200.so")
OBJ = os.environ.get("HGKS_OBJ") or os.path.join(HERE, "_obj")
# extra nvcc flags for kernel-variant experiments (e.g. -DHGKS_FACE_MINB=2; tools/ab_lib.sh)
EXTRA = os.environ.get("HGKS_NVCC_EXTRA", "").split()

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr"]

# translation units: (object name, source, extra defines)
UNITS = [
    ("capi", "hgks_capi.cu", []),
    ("k_p2_3d", "hgks_instances.cu", ["-DHGKS_INST_P=2", "-DHGKS_INST_DIM=3"]),
    ("k_p3_3d", "hgks_instances.cu", ["-DHGKS_INST_P=3", "-DHGKS_INST_DIM=3"]),
    ("k_p1_3d", "hgks_instances.cu", ["-DHGKS_INST_P=1", "-DHGKS_INST_DIM=3"]),
    ("k_p2_2d", "hgks_instances.cu", ["-DHGKS_INST_P=2", "-DHGKS_INST_DIM=2"]),
    ("k_p3_2d", "hgks_instances.cu", ["-DHGKS_INST_P=3", "-DHGKS_INST_DIM=2"]),
]


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    raise RuntimeError("nvcc not found")


def _sources():
    return ([os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INC, "hgks_b200.h")] +
            [os.path.join(INC, "hgks_b200", f) for f in os.listdir(os.path.join(INC, "hgks_b200"))
             if f.endswith(".h")])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _sources())


def build(force: bool = False, verbose: bool = False, log: str | None = None) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    nvcc = _nvcc()

    def compile_unit(u):
        name, src, defs = u
        out = os.path.join(OBJ, name + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *EXTRA, *defs, "-I", INC, "-I", CSRC, "-dc" if False else "-c",
               os.path.join(CSRC, src), "-o", out]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr[-4000:]}")
        return out, r.stderr

    with ThreadPoolExecutor(max_workers=min(len(UNITS), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_unit, UNITS))
    objs = [o for o, _ in results]
    ptxas_log = "\n".join(e for _, e in results)
    if log:
        with open(log, "w") as f:
            f.write(ptxas_log)
    if verbose:
        print(ptxas_log)
    cmd = [nvcc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv,
          log=os.path.join(HERE, "_obj", "ptxas.log"))
    print(LIB)
