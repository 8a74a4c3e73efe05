"""Build kernel variants (extra -D flags) into build/variants/<name>/librrs_b200.so
for A/B timing on the GPU box (select with RRS_B200_LIB=...).  Development only."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_08262_b200 import build as b

def build_variant(name, defines):
    out = os.path.join(ROOT, "build", "variants", name)
    os.makedirs(out, exist_ok=True)
    objs = []
    for src, extra in b.SOURCES.items():
        obj = os.path.join(out, src.replace(".cu", ".o"))
        cmd = [b.nvcc(), *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *extra,
               *[f"-D{d}" for d in defines], "-c", os.path.join(b.CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    lib = os.path.join(out, "librrs_b200.so")
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"], check=True)
    return lib

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition("=")
        print(build_variant(name, [d for d in defs.split(",") if d]))
