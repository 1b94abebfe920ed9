"""Build liblbm19.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2108_13241_b200.build [--verbose] [--experiments]

--experiments builds exp_lib/liblbm19_exp.so with -DLBM_EXPERIMENTS: the
measured-slower dense step variants (warp-uniform select, 128-bit vector
kernel; LBM_STEP_VARIANT=1/2/3/8) next to the product kernels.  Load it with
LBM_LIB=exp_lib/liblbm19_exp.so.  The product library never contains them.
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "liblbm19.so")
SOURCES = [os.path.join(CSRC, "lbm19.cu"), os.path.join(CSRC, "host_copy.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cuh")] + \
    [os.path.join(ROOT, "include", "lbm19.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off,-O3", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force=False, verbose=False, experiments=False):
    lib = os.path.join(ROOT, "exp_lib", "liblbm19_exp.so") if experiments else LIB
    if not force and not experiments and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    cmd = [NVCC] + FLAGS + (["-DLBM_EXPERIMENTS"] if experiments else []) + \
        (["-Xptxas", "-v"] if verbose else []) + SOURCES + ["-o", lib + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv, experiments="--experiments" in sys.argv))
