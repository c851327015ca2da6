"""Build librsr.so (all CUDA sources under csrc/) for sm_100a, in-tree.

Each source compiles to its own object in parallel (the kernels of one file call
no device code of another), then nvcc links the shared library."""
import glob
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "librsr.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + \
        glob.glob(os.path.join(HERE, "csrc", "*.h")) + [os.path.join(HERE, "..", "include", "rsr.h")]
    return all(os.path.getmtime(d) <= t for d in deps)


def _nvcc():
    return os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _compile_link(out, defines=()):
    """Objects in parallel, then one link; returns (ok, log)."""
    with tempfile.TemporaryDirectory() as tmp:
        def one(src):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [_nvcc()] + NVCC_FLAGS + ["-D" + d for d in defines] + ["-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            return obj, r.returncode, " ".join(cmd) + "\n" + r.stdout + r.stderr
        with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
            results = list(ex.map(one, sources()))
        log = "".join(x[2] for x in results)
        if any(x[1] != 0 for x in results):
            return False, log
        cmd = [_nvcc()] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", out] + [x[0] for x in results]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return r.returncode == 0, log + " ".join(cmd) + "\n" + r.stdout + r.stderr


def build(force=False, verbose=False, out=None, defines=()):
    """Compile every csrc/*.cu into one shared library (default: librsr.so)."""
    if out is not None:   # experiment build (tools/): always rebuilt
        ok, log = _compile_link(out, defines)
        if not ok:
            sys.stderr.write(log)
            raise RuntimeError("nvcc failed")
        return out
    if not force and up_to_date():
        return LIB
    ok, log = _compile_link(LIB)
    with open(os.path.join(HERE, "build_ptxas.log"), "w") as f:
        f.write(log)
    if not ok:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed building librsr.so")
    if verbose:
        print(log)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
