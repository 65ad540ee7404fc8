"""Build the in-tree shared libraries (no torch extension machinery, plain nvcc / g++).

  libsdv2.so      — the C-ABI library (include/sdv2.h): host control plane + sm_100a kernels
  libsdv2_ctl.so  — the host control plane alone (CPU tests; no CUDA needed)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force=False, verbose_ptxas=False):
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(HERE, "..", "include", "sdv2.h"))
    ctl_srcs = [os.path.join(CSRC, "ctl.cpp"), os.path.join(CSRC, "ctl_abi.cpp"), os.path.join(CSRC, "slo.cpp"),
                os.path.join(CSRC, "balance.cpp")]
    ctl_out = os.path.join(HERE, "libsdv2_ctl.so")
    if force or _stale(ctl_out, ctl_srcs + hdrs):
        _run(["g++", "-std=c++17", "-O2", "-shared", "-fPIC", "-o", ctl_out] + ctl_srcs)
    cu = os.path.join(CSRC, "sdv2.cu")
    out = os.path.join(HERE, "libsdv2.so")
    if force or _stale(out, [cu] + ctl_srcs + hdrs):
        cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-o", out, cu] + ctl_srcs
        if verbose_ptxas:
            cmd += ["-Xptxas", "-v"]
        _run(cmd)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
