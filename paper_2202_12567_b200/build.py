"""Build liblmc.so (the C-ABI library) in-tree for sm_100a with nvcc.

exact.cu and lighttree.cu are compiled with -fmad=false (decision precision: no FMA contraction,
DESIGN.md R30);
complete.cu and lmc_api.cu with the default contraction.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblmc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-ffp-contract=off",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-Xptxas", "-v"]
UNITS = [("exact.cu", ["-fmad=false"]), ("complete.cu", []), ("complete2.cu", []), ("mals.cu", []), ("lighttree.cu", ["-fmad=false"]), ("slice.cu", ["-fmad=false"]), ("lmc_api.cu", [])]


def _nccl_link():
    """Link the NCCL that PyTorch ships (and rpath it): libtorch_cuda and liblmc then share one
    libnccl.so.2 whichever is loaded first (the system NCCL is older than torch's and lacks symbols
    libtorch_cuda needs, so loading it first would break `import torch`)."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia")
        for base in (spec.submodule_search_locations or []) if spec else []:
            d = os.path.join(base, "nccl", "lib")
            if os.path.exists(os.path.join(d, "libnccl.so.2")):
                return ["-L" + d, "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", d]
    except (ImportError, ValueError):
        pass
    return ["-lnccl"]


def _stale(obj, deps):
    return not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(d) for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(ROOT, "include", "lmc.h"))
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    for src, extra in UNITS:
        s = os.path.join(CSRC, src)
        o = os.path.join(HERE, "build", src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s, *hdrs, __file__]):
            cmd = [NVCC, *COMMON, *extra, "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            with open(o + ".ptxas.txt", "w") as f:
                f.write(r.stderr)
    if force or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, "-shared", *ARCH, "-o", tmp, *objs, *_nccl_link()]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link of liblmc.so failed")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
