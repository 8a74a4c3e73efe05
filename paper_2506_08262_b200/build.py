"""Build the sm_100a C-ABI library in-tree: paper_2506_08262_b200/_lib/librrs_b200.so.

    python -m paper_2506_08262_b200.build        (or __graft_entry__.build())

nvcc cross-compiles for sm_100a without a GPU.  gen.cu is compiled with
-fmad=false (its FP64 arithmetic restates the reference's un-contracted
numpy/C sequence); the FP32 contraction keeps FFMA.  Every object is built
with -lineinfo so ncu's source page maps to the .cu lines.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "librrs_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = {  # file -> extra flags
    "gen.cu": ["-fmad=false"],
    "contract.cu": [],
    "contract_tc.cu": [],
    "contract_tcf.cu": [],
    "contract_tcw.cu": [],
    "contract_tcp.cu": [],
    "contract_tcs.cu": [],
    "select.cu": [],
    "center.cu": [],
    "contract64.cu": [],
    "api64.cu": [],
    "engine.cu": [],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(dep) > t for dep in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    objdir = os.path.join(OUT_DIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "rrs_b200.h"))
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v" if verbose else "-O3"]
    objs, jobs = [], []
    for src, extra in SOURCES.items():
        path = os.path.join(CSRC, src)
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path, *headers]):
            jobs.append([*common, *extra, "-c", path, "-o", obj])
    # the translation units are independent: compile them in parallel
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1) or 1) as pool:
        for r in list(pool.map(lambda cmd: subprocess.run(cmd, capture_output=not verbose), jobs)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args, r.stdout, r.stderr)
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        subprocess.run(cmd, check=True, capture_output=not verbose)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
