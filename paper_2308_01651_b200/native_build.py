"""Build the sm_100a shared library `libmdx.so` in-tree with nvcc.

`python -m paper_2308_01651_b200.native_build` (or `__graft_entry__.build()`)
compiles every `csrc/*.cu` for `-gencode arch=compute_100a,code=sm_100a` and
links `paper_2308_01651_b200/libmdx.so` (git-ignored, travels with the repo
snapshot to the GPU box).  `assembly.cu` is compiled with `--fmad=false` so the
assembled operators round exactly like the reference's numba kernels.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libmdx.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "-I", str(ROOT / "include"), "--expt-relaxed-constexpr"]
PER_FILE = {"assembly.cu": ["--fmad=false"]}


def nvcc_path():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; cannot build libmdx.so")
    return cand


def _stale(target, deps):
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force=False, verbose=False, ptxas_info=False):
    nvcc = nvcc_path()
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "mdx.h"]
    objs, jobs = [], []
    for src in sorted(CSRC.glob("*.cu")):
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *headers, Path(__file__)]):
            cmd = [nvcc, *ARCH, *COMMON, *PER_FILE.get(src.name, []),
                   "-c", str(src), "-o", str(obj)]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append((src, cmd))

    def compile_one(job):
        src, cmd = job
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
        if ptxas_info or verbose:
            print(res.stderr, file=sys.stderr)

    if jobs:       # the translation units are independent: compile them side by side
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
            list(pool.map(compile_one, jobs))
    if force or _stale(LIB, objs):
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static",
               *[str(o) for o in objs], "-o", str(LIB)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link of libmdx.so failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          ptxas_info="--ptxas" in sys.argv)
    print(LIB)
