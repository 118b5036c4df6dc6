"""In-tree build of libocgpu.so (host C++ + hand-written sm_100a kernels).

nvcc cross-compiles for sm_100a without a GPU; the generated per-model kernels
are compiled at plan creation by NVRTC (-arch=sm_100a) inside the library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
LIB = PKG / "libocgpu.so"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
ARCH = "-gencode=arch=compute_100a,code=sm_100a"

HOST_SRCS = ["graph.cpp", "dsl.cpp", "transcribe.cpp", "codegen.cpp", "jit.cpp", "capi.cpp", "ipm.cpp", "batch.cpp", "refldl.cpp", "shard.cpp"]
CUDA_SRCS = ["kernels.cu", "band.cu", "sepcr.cu", "ipm_kernels.cu", "kktbuild.cu", "batch_kernels.cu", "refldl.cu"]
# the interior-point vector kernels round every product and sum separately,
# as the reference's loops do on x86-64 (no FMA contraction there)
NO_FMA = {"ipm_kernels.cu", "batch_kernels.cu"}
HEADERS = ["model.hpp", "plan.hpp", "jit.hpp", "kernels.hpp", "band.hpp", "ipm_kernels.hpp", "kktbuild.hpp", "batch_kernels.hpp", "handles.hpp", "devmem.hpp", "refldl.hpp", "shard.hpp"]


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ({r.returncode})")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False) -> Path:
    OUT.mkdir(exist_ok=True)
    hdrs = [CSRC / h for h in HEADERS] + [PKG.parent / "include" / "octgpu.h"]
    objs = []
    cxx = os.environ.get("CXX", "g++")
    for s in HOST_SRCS:
        src, obj = CSRC / s, OUT / (Path(s).stem + ".o")
        if _stale(obj, [src] + hdrs):
            cmd = [cxx, "-std=c++20", "-O2", "-fPIC", "-pthread", "-Wall", "-Wno-unused-parameter",
                   f"-I{CUDA / 'include'}", "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
        objs.append(obj)
    for s in CUDA_SRCS:
        src, obj = CSRC / s, OUT / (Path(s).stem + ".cu.o")
        if _stale(obj, [src] + hdrs):
            cmd = [str(CUDA / "bin" / "nvcc"), ARCH, "-O3", "-lineinfo", "-std=c++17",
                   "-Xptxas", "-v", "-Xcompiler", "-fPIC", "-c", str(src), "-o", str(obj)]
            if s in NO_FMA:
                cmd.insert(3, "-fmad=false")
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
        objs.append(obj)
    if _stale(LIB, objs):
        cmd = [cxx, "-shared", "-pthread", "-Wl,--exclude-libs,ALL", "-o", str(LIB)] + [str(o) for o in objs] + [
            f"-L{CUDA / 'lib64'}", "-lcudart", "-lnvrtc", "-ldl", f"-Wl,-rpath,{CUDA / 'lib64'}"]
        if verbose:
            print(" ".join(cmd))
        _run(cmd)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
