"""Build the in-tree CUDA C-ABI library ``_lib/libconesplit_b200.so``.

    python -m paper_1905_03748_b200.build      (or __graft_entry__.build())

nvcc cross-compiles for sm_100a only (no GPU needed); objects are rebuilt
when a source or header is newer than the library.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libconesplit_b200.so")
SOURCES = ["runtime.cu", "forward.cu", "backward.cu",
           "staged.cu", "tv.cu", "vector.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"),
                 "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, out_dir: str = OUT_DIR,
          defines: tuple = ()) -> str:
    """Compile every source into out_dir/libconesplit_b200.so; ``defines``
    (e.g. ("DUAL_MINB=1",)) build A/B variants into another out_dir."""
    nvcc = _nvcc()
    os.makedirs(out_dir, exist_ok=True)
    lib_path = os.path.join(out_dir, "libconesplit_b200.so")
    dflags = [f"-D{d}" for d in defines]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
               if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "conesplit_b200.h"))
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [nvcc, *ARCH, *FLAGS, *dflags, "-I", INCLUDE, "-c", path,
                   "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
            if verbose:
                sys.stderr.write(r.stderr)
            with open(obj + ".ptxas.txt", "w") as f:
                f.write(r.stderr)
    if force or _stale(lib_path, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", lib_path, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib_path


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
