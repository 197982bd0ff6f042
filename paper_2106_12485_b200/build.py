"""Build libzpic_b200.so in-tree with nvcc for sm_100a (no torch JIT; the .so travels with the repo)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libzpic_b200.so")
SOURCES = ["zpic_api.cu", "zpic_kernels.cu", "zpic_push.cu", "zpic_peer.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# -ftz=true: fp32 denormals flush to zero (no guard code around rsqrt / rcp); -prec-div=false:
# approximate fp32 division (2 ulp) for the cell-crossing fractions.  The fp64 paths (injector RNG,
# energy sums) are unaffected.
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-ftz=true",
         "-prec-div=false", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-O2", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _nccl_dirs():
    """torch's bundled NCCL (the library must share the communicator type and the loaded .so)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl") or importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations or []) if spec else []
    for r in roots:
        base = r if r.endswith("nccl") else os.path.join(r, "nccl")
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            return os.path.join(base, "include"), os.path.join(base, "lib")
    raise RuntimeError("nccl.h not found (expected torch's nvidia/nccl package)")


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "zpic.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return SO
    nccl_inc, nccl_lib = _nccl_dirs()
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC] + FLAGS + ["-I", nccl_inc, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError("nvcc failed for " + src)
        objs.append(obj)
    tmp = SO + ".tmp%d" % os.getpid()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs + [
        "-lcudart", "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib]
    subprocess.check_call(cmd)
    os.replace(tmp, SO)
    for o in objs:
        os.remove(o)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(SO)
