"""Build libcwreco.so in-tree: host C++ (g++, OpenMP) + sm_100a CUDA (nvcc).

Called by __graft_entry__.build() and by the package on first import when the
library is missing.  Sources: paper_1612_09335_b200/csrc/, header: include/.
"""
import io
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
OUT = os.path.join(HERE, "libcwreco.so")
BUILD = os.path.join(HERE, "build")

CXX_SRCS = ["api.cpp", "mesh.cpp", "stencil.cpp", "basis.cpp", "precompute.cpp", "predictor.cpp"]
CU_SRCS = ["kernels.cu", "rowblk_2d.cu", "rowblk_3d.cu", "matfree.cu", "traces.cu", "halo.cu", "predictor.cu"]
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
# -ffp-contract=off: the IEEE-specified geometry (R29) must not be fused; -mfma
# lets std::fma (exact products in the predicates) use the hardware instruction.
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-fopenmp", "-mfma", "-ffp-contract=off", "-Wall",
            "-Wno-unused-function", "-I", INC, "-I", CSRC]
NVFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
           "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", INC, "-I", CSRC]


# Timing-only experiment switches (CWRECO_EXP_FLAGS, CWRECO_KC, CWRECO_MAX_STAGES, …)
# exist only in a library built with CWRECO_BUILD_EXPERIMENTS=1 (tools/); the product
# build has none of them, and cwreco_version() says which build is loaded.
if os.environ.get("CWRECO_BUILD_EXPERIMENTS") == "1":
    CXXFLAGS = CXXFLAGS + ["-DCWRECO_EXPERIMENTS"]
    NVFLAGS = NVFLAGS + ["-DCWRECO_EXPERIMENTS"]


def _run(cmd, log):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    log.write(" ".join(cmd) + "\n" + r.stdout + "\n")
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r.stdout


def build(verbose=False, out=None, defines=()):
    """Compile every source in parallel (one process each), then link.  out / defines:
    tuning variants only (tools/): another file name and extra -D macros."""
    from concurrent.futures import ThreadPoolExecutor
    out = out or OUT
    bdir = BUILD if out == OUT else os.path.join(BUILD, os.path.basename(out) + ".d")
    os.makedirs(bdir, exist_ok=True)
    dflags = ["-D" + d for d in defines]
    jobs = []
    for s in CXX_SRCS:
        jobs.append((["g++", *CXXFLAGS, *dflags, "-c", os.path.join(CSRC, s), "-o", os.path.join(bdir, s + ".o")],
                     os.path.join(bdir, s + ".o")))
    for s in CU_SRCS:
        jobs.append(([NVCC, *NVFLAGS, *dflags, "-c", os.path.join(CSRC, s), "-o", os.path.join(bdir, s + ".o")],
                     os.path.join(bdir, s + ".o")))
    logs = [io.StringIO() for _ in jobs]
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        futs = [ex.submit(_run, cmd, lg) for (cmd, _), lg in zip(jobs, logs)]
        outs = [f.result() for f in futs]
    objs = [o for _, o in jobs]
    with open(os.path.join(bdir, "build.log"), "w") as log:
        for lg in logs:
            log.write(lg.getvalue())
        if verbose:
            print("\n".join(outs))
        _run(["g++", "-shared", "-o", out + ".tmp", *objs, "-fopenmp", "-L" + os.path.join(CUDA_HOME, "lib64"),
              "-lcudart_static", "-lrt", "-ldl", "-lpthread"], log)
    os.replace(out + ".tmp", out)
    return out


def stale_abi(path):
    """True if the built library lacks an entry point include/cwreco.h declares."""
    import re
    try:
        with open(os.path.join(INC, "cwreco.h")) as f:
            names = set(re.findall(r"\b(cwreco_[a-z_]+)\s*\(", f.read()))
        out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    except OSError:
        return False
    if not out:
        return False
    have = set(re.findall(r" T (cwreco_\w+)", out))
    return bool(names - have)


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INC, "cwreco.h")]
    return any(os.path.getmtime(s) > t for s in srcs)


if __name__ == "__main__":
    # python _build.py [-v] [--out FILE] [-D MACRO=VAL ...]   (variants: tools only)
    args = sys.argv[1:]
    o, ds = None, []
    while args:
        x = args.pop(0)
        if x == "--out":
            o = args.pop(0)
        elif x == "-D":
            ds.append(args.pop(0))
    print(build(verbose="-v" in sys.argv, out=o, defines=ds))
