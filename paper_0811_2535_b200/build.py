"""Build libmoa_fft.so in-tree with nvcc for sm_100a (no torch extension machinery).

The pass kernel is instantiated once per FFT length 2^1..2^13 (fft_inst.cu with
-DMOA_INST_LOGF=f); the objects compile in parallel.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build" + os.environ.get("MOA_BUILD_TAG", ""))
LIB = os.environ.get("MOA_FFT_LIB") or os.path.join(HERE, "libmoa_fft.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*os.environ.get("MOA_NVCC_EXTRA", "").split(),
         "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr"]

SOURCES = ["kernels.cu", "plan.cu", "exec.cu", "abi.cu", "dist.cu", "fused.cu"]
INST_LOGF = list(range(1, 14))


def _sources_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "moa_fft.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def needs_build() -> bool:
    return not os.path.exists(LIB) or os.path.getmtime(LIB) < _sources_mtime()


def _compile(src: str, obj: str, extra: list[str]) -> str:
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False, jobs: int | None = None,
          ptxas_verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []
    tasks = []
    for f in INST_LOGF:
        tasks.append((os.path.join(CSRC, "fft_inst.cu"), os.path.join(BUILD, f"fft_inst_{f}.o"),
                      [f"-DMOA_INST_LOGF={f}", *extra]))
    for s in SOURCES:
        tasks.append((os.path.join(CSRC, s), os.path.join(BUILD, s.replace(".cu", ".o")), extra))
    jobs = jobs or min(len(tasks), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda a: _compile(*a), tasks))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="--ptxas" in sys.argv)
