"""Build libmirage.so in-tree with nvcc for sm_100a (the only target)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmirage.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
try:  # NCCL ships with torch (nvidia-nccl wheel); headers + libnccl.so.2
    import nvidia.nccl as _nccl
    NCCL_DIR = list(_nccl.__path__)[0]
except Exception:  # pragma: no cover
    NCCL_DIR = "/usr"
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I" + os.path.join(NCCL_DIR, "include")]
SOURCES = ["attention.cu", "decode_gemm.cu", "layer_kernels.cu", "runtime.cpp", "planner.cpp"]


def _compile(src):
    obj = os.path.join(BUILD, src + ".o")
    path = os.path.join(CSRC, src)
    deps = [path] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "mirage.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj, ""
    lang = ["-x", "cu"] if src.endswith(".cu") else []
    cmd = [NVCC] + ARCH + FLAGS + lang + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        res = list(ex.map(_compile, SOURCES))
    objs = [o for o, _ in res]
    if verbose:
        for _, log in res:
            sys.stderr.write(log)
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUT] + objs + [
            "-L/usr/local/cuda/lib64", "-lcublas", "-lcublasLt", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
            "-L" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(NCCL_DIR, "lib")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
