"""Build libgwas.so in-tree with nvcc for sm_100a (explicit -gencode; no torch arch list involved).

Each translation unit under csrc/ is compiled to an object in parallel (the estimation kernels are instantiated
for p = 1..12 across four units), then nvcc links the shared library against cuSOLVER."""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgwas.so")
SOURCES = ["gwas.cu", "est_p1_3.cu", "est_p4_6.cu", "est_p7_9.cu", "est_p10_12.cu"]
HEADERS = ["ctile.cuh", "estimate.cuh", "estimate_launch.cuh", "gemm_dmma.cuh", "gemm_i8.cuh", "lowrank_k3.cuh", "schur.cuh", "setup_kernels.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
]


def _nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "gwas.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def _compile(src, obj_dir):
    obj = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
    cmd = [_nvcc(), *COMPILE_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, r


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    obj_dir = tempfile.mkdtemp(prefix="gwas_build_")  # objects stay out of the tree (they would travel to the box)
    try:
        return _build(obj_dir, verbose)
    finally:
        shutil.rmtree(obj_dir, ignore_errors=True)


def _build(obj_dir, verbose):
    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(lambda src: _compile(src, obj_dir), SOURCES))
    info = []
    for src, obj, r in results:
        info.append(f"==== {src}\n{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = [_nvcc(), *ARCH, "-shared", *[obj for _, obj, _ in results], "-o", LIB + ".tmp",
           "-L", os.path.join(cuda, "lib64"), "-lcusolver", "-Xlinker", "-rpath=" + os.path.join(cuda, "lib64")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libgwas.so")
    if verbose:
        sys.stderr.write("".join(info))
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write("".join(info))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
