"""Build the native library in-tree: paper_2306_16601_b200/_native/libsparseinfer_b200.so.

nvcc cross-compiles for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``,
no other architecture, no JIT).  Host C++ is compiled with
``-ffp-contract=off`` so the plan builder's epilogue tables follow the
reference's f64 expression trees.  The CUDA runtime is linked statically so
the library does not depend on which libcudart torch happens to load.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_native")
LIB_NAME = "libsparseinfer_b200.so"
LIB_PATH = os.path.join(OUT_DIR, LIB_NAME)
# experiment builds: SI_BUILD_DEFS="-DNAME ..." -> a separate library that
# SI_LIB=<path> selects at load time (never the default product library)
EXTRA_DEFS = os.environ.get("SI_BUILD_DEFS", "").split()

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
              "-Xptxas", "-v", "--expt-relaxed-constexpr"]
SOURCES = ["plan.cpp", "abi.cu", "spmm_gather.cu", "spmm_tc.cu", "spmm_xs.cu", "spmm_ws.cu", "eltwise.cu"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _compile(src: str, obj: str, log_dir: str) -> None:
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *EXTRA_DEFS, "-I", os.path.join(HERE, "..", "include"), "-c",
           os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cpp"):
        cmd.insert(1, "-x")
        cmd.insert(2, "c++")
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(log_dir, os.path.basename(obj) + ".log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr[-4000:]}")


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "sparseinfer_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, out: str | None = None) -> str:
    """Compile (if stale) and return the library path."""
    lib_path = out or LIB_PATH
    if not force and out is None and not _stale():
        return LIB_PATH
    obj_dir = os.path.join(OUT_DIR, "obj" if out is None else "obj_exp")
    os.makedirs(obj_dir, exist_ok=True)
    objs = [os.path.join(obj_dir, s.rsplit(".", 1)[0] + ".o") for s in SOURCES]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "sparseinfer_b200.h"))
    newest_hdr = max(os.path.getmtime(h) for h in headers)

    def needed(so):
        src, obj = so
        if force or not os.path.exists(obj):
            return True
        return os.path.getmtime(obj) < max(os.path.getmtime(os.path.join(CSRC, src)), newest_hdr)

    todo = [so for so in zip(SOURCES, objs) if needed(so)]
    if todo:
        with cf.ThreadPoolExecutor(len(todo)) as ex:
            list(ex.map(lambda so: _compile(so[0], so[1], obj_dir), todo))
    tmp = lib_path + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    import sys
    print(build(force=True, out=sys.argv[1] if len(sys.argv) > 1 else None))
