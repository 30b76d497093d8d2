"""A/B builds: recompile lpic_kernels.cu (the encoder / seam kernels) -- or,
with --all, every unit -- with extra -D flags and link it with the main
build's other objects into paper_2212_01185_b200/ab/<name>.so (select with
LPIC_LIB=...).
usage: python scripts/ab_build.py NAME [--all] [-DFLAG ...]"""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2212_01185_b200 import build as B
from concurrent.futures import ThreadPoolExecutor
name, args = sys.argv[1], sys.argv[2:]
every = "--all" in args
defs = [a for a in args if a != "--all"]
B.build()
out = os.path.join(B.HERE, "ab"); os.makedirs(out, exist_ok=True)
redo = B.SOURCES if every else ["lpic_kernels.cu"]


def one(src):
    obj = os.path.join(B.OBJDIR, f"ab_{name}_" + src.replace(".cu", ".o"))
    subprocess.run([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    return obj


with ThreadPoolExecutor(max_workers=len(redo)) as ex:
    objs = list(ex.map(one, redo))
objs += [os.path.join(B.OBJDIR, s.replace(".cu", ".o")) for s in B.SOURCES if s not in redo]
so = os.path.join(out, f"{name}.so")
subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", so], check=True)
for o in objs:                       # (keep the gpurun snapshot small: variant objects are not reused)
    if os.path.basename(o).startswith("ab_"):
        os.remove(o)
print(so)
