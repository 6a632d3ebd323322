"""Build libpst.so (sm_100a) in-tree with nvcc.  `python -m paper_1912_12675_b200.build`."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
BUILD = os.path.join(ROOT, "build", "pst")
LIB = os.path.join(HERE, "libpst.so")
VARIANTS = {"": ("libpst.so", ()),                         # float32 storage, 3xTF32 tensor-core products
            "bf16": ("libpst_bf16.so", ("-DPST_PREC_BF16",)),  # fast variant (see DESIGN.md Precision)
            "f16": ("libpst_f16.so", ("-DPST_ACT_FP16",)),     # diagnostics only
            "exp": ("libpst_exp.so", ("-DPST_EXPERIMENTS",))}  # default precision + experiment switches (tools/)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]
SOURCES = ["common.cpp", "model.cpp", "conv_tc.cu", "conv_ts.cu", "conv_wgrad_ts.cu", "elementwise.cu", "stage.cu", "pst_api.cu", "ops_api.cu"]


def _deps_mtime():
    return max(os.path.getmtime(os.path.join(d, f))
               for d in (CSRC, os.path.join(ROOT, "include"))
               for f in os.listdir(d) if f.endswith((".h", ".cuh")))


def _compile(src, extra):
    obj = os.path.join(BUILD, src + ".o")
    path = os.path.join(CSRC, src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), _deps_mtime()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-x", "cu", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and os.environ.get("PST_BUILD_VERBOSE"):
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, extra=(), variant: str = "") -> str:
    """variant "" -> libpst.so (default precision); "bf16" / "f16" -> the other variants."""
    global BUILD
    name, defs = VARIANTS[variant]
    lib_path = os.path.join(HERE, name)
    build_dir = os.path.join(ROOT, "build", "pst" + (("_" + variant) if variant else ""))
    extra = tuple(extra) + tuple(defs)
    BUILD, saved = build_dir, BUILD
    try:
        return _build(verbose, extra, lib_path)
    finally:
        BUILD = saved


def _build(verbose, extra, lib_path):
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, list(extra)), SOURCES))
    if not os.path.exists(lib_path) or os.path.getmtime(lib_path) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib_path, *objs,
               "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-Xlinker", "-rpath,/usr/lib/x86_64-linux-gnu"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("built", lib_path)
    return lib_path


if __name__ == "__main__":
    build(verbose=True)
    if len(sys.argv) > 1 and sys.argv[1] == "all":
        build(verbose=True, variant="bf16")
