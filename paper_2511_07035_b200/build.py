"""Build libgockpt.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

  kernels.cu         nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
                     (no --use_fast_math: IEEE div/sqrt and denormals are normative)
  gockpt_runtime.cpp g++ -O3 (C ABI, session FSM, ring, pinned arena, streams)
  replay_host.cpp    g++ -O3 -ffp-contract=off -fno-math-errno (bit-exact host replay;
                     AVX-512/AVX2 target clones)
  link               nvcc -shared, static cudart (no dependence on torch's cudart version)
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libgockpt.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["kernels.cu", "gockpt_runtime.cpp", "replay_host.cpp", "persist.cpp", "model.cpp", "internal.h", "adamw_math.cuh"]


def _cuda_home() -> str:
    for c in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if c and os.path.exists(os.path.join(c, "bin", "nvcc")):
            return c
    nvcc = shutil.which("nvcc")
    if nvcc:
        return os.path.dirname(os.path.dirname(nvcc))
    raise RuntimeError("nvcc not found: set CUDA_HOME")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(INCLUDE, "gockpt.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log):
    log.append(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile (if stale) and return the path of libgockpt.so."""
    if not force and not _stale():
        return LIB
    cuda = _cuda_home()
    nvcc = os.path.join(cuda, "bin", "nvcc")
    os.makedirs(BUILD, exist_ok=True)
    log: list[str] = []
    inc = ["-I", INCLUDE, "-I", CSRC]
    objs = {k: os.path.join(BUILD, k + ".o") for k in ("kernels", "runtime", "replay_host", "persist", "model")}
    _run([nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-Xcompiler", "-fPIC", *inc,
          "-c", os.path.join(CSRC, "kernels.cu"), "-o", objs["kernels"]], log)
    gxx = ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function", *inc,
           "-I", os.path.join(cuda, "include")]
    _run(gxx + ["-c", os.path.join(CSRC, "gockpt_runtime.cpp"), "-o", objs["runtime"]], log)
    _run(gxx + ["-ffp-contract=off", "-fno-math-errno",
                "-c", os.path.join(CSRC, "replay_host.cpp"), "-o", objs["replay_host"]], log)
    _run(gxx + ["-c", os.path.join(CSRC, "persist.cpp"), "-o", objs["persist"]], log)
    _run(gxx + ["-c", os.path.join(CSRC, "model.cpp"), "-o", objs["model"]], log)
    tmp = LIB + ".tmp"
    _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, objs["kernels"], objs["runtime"],
          objs["replay_host"], objs["persist"], objs["model"], "-Xcompiler", "-fPIC", "-lpthread", "-lz", "-ldl"], log)
    os.replace(tmp, LIB)
    with open(os.path.join(BUILD, "build.log"), "w") as fh:
        fh.write("\n".join(log))
    if verbose:
        print("\n".join(log), file=sys.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
