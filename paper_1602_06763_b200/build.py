"""Build the sm_100a shared library in-tree (no JIT cache): every CUDA
translation unit is compiled by nvcc for `-gencode arch=compute_100a,code=sm_100a`
and linked into paper_1602_06763_b200/librelapack_b200.so (C ABI, include/relapack.h).
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
# RELAPACK_BUILD_OUT / RELAPACK_BUILD_DEFS: an alternative build (A/B experiments,
# tools/ab_bench.py) into another directory with extra -D flags
OUT = os.environ.get("RELAPACK_BUILD_OUT") or os.path.join(HERE, "librelapack_b200.so")
BUILD = os.path.join(os.path.dirname(OUT), "build") if os.environ.get("RELAPACK_BUILD_OUT") else os.path.join(HERE, "build")
EXTRA_DEFS = [f"-D{d}" for d in os.environ.get("RELAPACK_BUILD_DEFS", "").split()]
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = EXTRA_DEFS + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
SOURCES = ["update.cu", "potf2.cu", "trsm.cu", "trsm_fused.cu", "batched.cu", "driver.cu", "dist.cu", "hooks.cu", "xkernels.cu", "xdriver.cu", "plan.cpp", "xplan.cpp"]


def _digest() -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(name.encode() + f.read())
    with open(os.path.join(ROOT, "include", "relapack.h"), "rb") as f:
        h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()[:16]


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr}")
    return obj, p.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    stamp = os.path.join(BUILD, "stamp")
    digest = _digest()
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and open(stamp).read() == digest:
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, SOURCES))
    log = "".join(r[1] for r in results)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        f.write(log)
    if verbose:
        print(log)
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *[r[0] for r in results], "-cudart", "static", "-ldl", "-lpthread",
           "-Xlinker", "--no-undefined"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stderr}")
    os.replace(tmp, OUT)
    with open(stamp, "w") as f:
        f.write(digest)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
