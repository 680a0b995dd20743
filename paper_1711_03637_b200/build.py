"""Build libsnn_b200.so in-tree for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "snn_b200.cu")
OUT = os.path.join(HERE, "libsnn_b200.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("snn_b200.cu", "hidden.cuh", "hidden_gb.cuh", "normad.cuh", "normad_cl.cuh", "normad_spec.cuh",
                                                 "snn_common.cuh", "preprocess.cuh")]
DEPS.append(os.path.join(ROOT, "include", "snn_b200.h"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


PEAKS_SRC = os.path.join(HERE, "csrc", "peaks.cu")
PEAKS_OUT = os.path.join(HERE, "libsnn_peaks.so")


def build_peaks(force: bool = False) -> str:
    """The FP64/FP32 pipe-peak microbenchmark used for roofline denominators."""
    if force or not os.path.exists(PEAKS_OUT) or os.path.getmtime(PEAKS_OUT) < os.path.getmtime(PEAKS_SRC):
        subprocess.run([nvcc(), *NVCC_FLAGS, "-o", PEAKS_OUT, PEAKS_SRC], check=True)
    return PEAKS_OUT


def build(force: bool = False, verbose: bool = False) -> str:
    build_peaks(force)
    if not force and up_to_date():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", OUT + ".tmp", SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


PROFILE_OUT = os.path.join(HERE, "libsnn_b200_profile.so")


def build_profile(force: bool = False) -> str:
    """Profiling-only build (-DSNN_NORMAD_PROFILE): the cluster NormAD kernel
    with phase clocks and phase ablation compiled in.  Never loaded by the
    product path; scripts select it with SNN_B200_LIB (see _native.py)."""
    if force or not os.path.exists(PROFILE_OUT) or any(os.path.getmtime(d) > os.path.getmtime(PROFILE_OUT) for d in DEPS):
        subprocess.run([nvcc(), *NVCC_FLAGS, "-DSNN_NORMAD_PROFILE", "-I", os.path.join(ROOT, "include"),
                        "-o", PROFILE_OUT, SRC], check=True)
    return PROFILE_OUT


if __name__ == "__main__":
    if "--profile" in sys.argv:
        print(build_profile(force="--force" in sys.argv))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
