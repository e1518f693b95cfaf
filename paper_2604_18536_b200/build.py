"""Build the sm_100a shared library ``libstagflow_b200.so`` in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a, cudart static, linked against
cuFFT (raw transforms only).  Invoked by ``__graft_entry__.build()`` and by
``python -m paper_2604_18536_b200.build``.
"""

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstagflow_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O3",
         "-Xptxas", "-O3"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(HERE, "..", "include", "*.h"))
    return any(os.path.getmtime(f) > t for f in deps)


def build(force=False, verbose=False, jobs=None):
    if not force and not _stale():
        return LIB
    nvcc = os.path.join(CUDA, "bin", "nvcc")
    objs = []
    procs = []
    os.makedirs(os.path.join(CSRC, "build"), exist_ok=True)
    # nccl.h of the NCCL PyTorch loads (comm.cu dlopens libnccl.so.2 at run time)
    nccl_inc = [f for d in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl",
                                                  "include")) for f in ("-I", d)][:2]
    for src in sources():
        obj = os.path.join(CSRC, "build", os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        extra = os.environ.get("SFB_NVCC_FLAGS", "").split()
        cmd = [nvcc, *ARCH, *FLAGS, *extra, "-I", os.path.join(HERE, "..", "include"), *nccl_inc, "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed.append((src, out))
        elif verbose and out:
            print(out)
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    torch_cufft = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "cufft", "lib"))
    rpaths = [os.path.join(CUDA, "lib64")] + torch_cufft
    link = [nvcc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-L", os.path.join(CUDA, "lib64"), "-lcufft", "-ldl"]
    for r in rpaths:
        link += ["-Xlinker", "-rpath=" + r]
    subprocess.run(link, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
