"""Build libefunc.so in-tree for sm_100a (nvcc, no JIT cache): `python -m paper_2505_21319_b200.build`."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libefunc.so")
SOURCES = ["efunc_api.cu", "k_bin.cu", "k_lists.cu", "k_forward.cu", "k_backward.cu", "k_fit.cu", "k_fit_eik.cu", "k_adamw.cu", "k_mesh.cu", "k_var.cu", "k_cosine.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "efunc.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile + link. `out`/`defines` build a tuning variant (e.g. -DFK_MIN_BLOCKS=20) elsewhere."""
    if not force and out == LIB and not _stale():
        return LIB
    odir = os.path.dirname(out)
    os.makedirs(odir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(odir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs,
           "-Xcompiler", "-fPIC", "-cudart", "static", "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    if "--variant" in args:  # --variant NAME -DX=Y ...: lib/variants/NAME/libefunc.so
        name = args[args.index("--variant") + 1]
        defs = [a for a in args if a.startswith("-D")]
        print(build(force=True, out=os.path.join(LIBDIR, "variants", name, "libefunc.so"), defines=defs))
    else:
        print(build(force="--force" in args, verbose=True))
