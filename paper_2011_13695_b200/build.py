"""Build librx.so in-tree for sm_100a (nvcc; no torch extension machinery needed: the
boundary is a plain C ABI, include/rx.h)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "librx.so")
SOURCES = ["csrc/rx_api.cu", "csrc/tx_api.cu"]
DEPS = ["csrc/rx_api.cu", "csrc/common.cuh", "csrc/fft.cuh", "csrc/rx_dev.cuh", "csrc/k_pam.cuh",
        "csrc/k_kk.cuh", "csrc/k_lms.cuh", "csrc/k_shard.cuh", "../include/rx.h", "csrc/tx_api.cu",
        "../include/tx.h"]


def _git_rev() -> str:
    try:
        return subprocess.check_output(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                                       stderr=subprocess.DEVNULL, text=True).strip()
    except Exception:
        return "nogit"


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(os.path.join(HERE, p)) > t for p in DEPS)


PEAK_SO = os.path.join(HERE, "libfp32peak.so")


def build_peak(force: bool = False) -> str:
    """bench.py's FP32 FFMA peak probe (csrc/fp32_peak.cu), a separate library: not part of
    the receiver ABI."""
    src = os.path.join(HERE, "csrc", "fp32_peak.cu")
    if not force and os.path.exists(PEAK_SO) and os.path.getmtime(PEAK_SO) > os.path.getmtime(src):
        return PEAK_SO
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                    "-Xcompiler", "-fPIC", "-o", PEAK_SO + ".tmp", src], check=True, cwd=HERE)
    os.replace(PEAK_SO + ".tmp", PEAK_SO)
    return PEAK_SO


def build(force: bool = False, verbose: bool = False) -> str:
    build_peak(force)
    if not force and not needs_build():
        return SO
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-shared", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
           f"-DRX_GIT=\"{_git_rev()}\"", "-o", SO + ".tmp"] + [os.path.join(HERE, s) for s in SOURCES]
    cmd[1:1] = os.environ.get("RX_NVCC_FLAGS", "").split()     # experiments (e.g. -DLMS_SPC=2)
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
