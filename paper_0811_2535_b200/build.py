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
# MOA_BUILD_VARIANTS=1: the ablation library libmoa_fft_variants.so, which also holds the
# pass variants measured slower and kept out of the product (persistent / TMA-staged /
# prefetching passes, the L2-fused pass pair), selected only through the
# MOA_FFT_* knobs under MOA_FFT_ABLATION=1.  The default build is the product library.
VARIANTS = os.environ.get("MOA_BUILD_VARIANTS", "0") not in ("", "0")
BUILD = os.path.join(HERE, "_build" + ("_variants" if VARIANTS else "") + os.environ.get("MOA_BUILD_TAG", ""))
LIB = os.environ.get("MOA_FFT_LIB") or os.path.join(HERE, "libmoa_fft_variants.so" if VARIANTS else "libmoa_fft.so")
VARIANTS_LIB = os.path.join(HERE, "libmoa_fft_variants.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*os.environ.get("MOA_NVCC_EXTRA", "").split(),
         "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr"]

SOURCES = ["kernels.cu", "plan.cu", "exec.cu", "abi.cu", "dist.cu", "redist.cu"] + (["fused.cu", "bigpass.cu"] if VARIANTS else [])
if VARIANTS:
    FLAGS.append("-DMOA_VARIANTS=1")
INST_LOGF = list(range(1, 14))


def _sources_mtime() -> float:
    # the product library does not depend on the variant-only sources
    skip = set() if VARIANTS else {"fused.cu", "bigpass.cu"}
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f not in skip]
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


def build_variants(force: bool = False) -> str:
    """Build libmoa_fft_variants.so (the ablation library) in a child process."""
    env = dict(os.environ, MOA_BUILD_VARIANTS="1")
    env.pop("MOA_FFT_LIB", None)
    cmd = [sys.executable, os.path.abspath(__file__)] + (["--force"] if force else [])
    r = subprocess.run(cmd, env=env, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"variants build failed:\n{r.stdout}\n{r.stderr}")
    return VARIANTS_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="--ptxas" in sys.argv)
