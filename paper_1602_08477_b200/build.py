"""In-tree build of libkw_b200.so (sm_100a) and of the C++ drop-in test programs.

Everything is compiled with nvcc / g++ directly (no JIT cache): the built .so files sit in the
package directory so they travel to the GPU box with the repository snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = PKG / "_build"
LIB = PKG / "libkw_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}"]
# measurement builds only (e.g. "-DKW_SPLIT_TRACE"): appended to every library compile
NVCC_FLAGS += os.environ.get("KW_EXTRA_NVCC_FLAGS", "").split()
SOURCES = ["kw_runtime.cu", "kw_axpy.cu", "kw_dgemm.cu", "kw_dgemm_e2e.cu", "kw_comm.cu"]


def _run(cmd: list[str]) -> str:
    p = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"command failed ({p.returncode}): {' '.join(cmd)}\n{p.stdout}")
    return p.stdout


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/*.cu for sm_100a and link libkw_b200.so. NCCL is not linked: kw_comm.cu
    dlopens libnccl.so.2 at first use (the copy torch already loaded, when there is one)."""
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [INCLUDE / "kw_b200.h"]
    objs = []
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *NVCC_FLAGS, "-c", str(s), "-o", str(o)])
    if jobs:
        logs = []
        with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            for cmd, out in zip(jobs, ex.map(_run, jobs)):
                if verbose:
                    print(out)
                logs.append(f"== {Path(cmd[-3]).name}\n{out}")
        # ptxas -v of the objects rebuilt by this call (overwritten, not appended)
        (BUILD / "ptxas.log").write_text("".join(logs))
    if force or jobs or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", "-ldl"])
    return LIB


def build_cpp_tests(force: bool = False) -> list[Path]:
    """Builds the C++ drop-in programs under tests/cpp against include/ and libkw_b200.so."""
    out = []
    cpp_dir = ROOT / "tests" / "cpp"
    hdrs = list((INCLUDE / "kernelweave").rglob("*.hpp")) + [INCLUDE / "kw_b200.h", INCLUDE / "kernelweave" / "cuda_exec.cuh"]
    for src in sorted(cpp_dir.glob("*.cpp")):
        exe = BUILD / src.stem
        if force or _stale(exe, [src, LIB] + hdrs):
            _run(["g++", "-O2", "-std=c++20", "-Wall", "-Wextra", f"-I{INCLUDE}", str(src), "-o", str(exe),
                  f"-L{PKG}", "-lkw_b200", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/..", "-lpthread"])
        out.append(exe)
    # kwbench carries its own plain CUDA kernels (the "native" back-end), so nvcc builds it
    kwb = ROOT / "tools" / "kwbench" / "kwbench.cu"
    exe = BUILD / "kwbench"
    if force or _stale(exe, [kwb, LIB] + hdrs):
        _run([NVCC, *ARCH, "-O2", "-std=c++20", "-lineinfo", f"-I{INCLUDE}", str(kwb), "-o", str(exe), f"-L{PKG}",
              "-lkw_b200", f"-Xlinker=-rpath,{PKG}", "-lcudart"])
    out.append(exe)
    for src in sorted(cpp_dir.glob("*.cu")):
        exe = BUILD / src.stem
        if force or _stale(exe, [src, LIB] + hdrs + [INCLUDE / "kernelweave" / "cuda_exec.cuh"]):
            _run([NVCC, *ARCH, "-O2", "-std=c++20", "-lineinfo", f"-I{INCLUDE}", str(src), "-o", str(exe),
                  f"-L{PKG}", "-lkw_b200", f"-Xlinker=-rpath,{PKG}", "-lcudart"])
        out.append(exe)
    return out


if __name__ == "__main__":
    build_lib(force="--force" in sys.argv, verbose=True)
    print(build_cpp_tests(force="--force" in sys.argv))
