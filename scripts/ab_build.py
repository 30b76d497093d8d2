"""A/B builds: recompile lpic_kernels.cu (the encoder / seam kernels) with
extra -D flags and link it with the main build's other objects into
paper_2212_01185_b200/ab/<name>.so (select with LPIC_LIB=...).
usage: python scripts/ab_build.py NAME [-DFLAG ...]"""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2212_01185_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
B.build()
out = os.path.join(B.HERE, "ab"); os.makedirs(out, exist_ok=True)
obj = os.path.join(B.OBJDIR, f"ab_{name}_kernels.o")
subprocess.run([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, "lpic_kernels.cu"), "-o", obj], check=True)
objs = [obj] + [os.path.join(B.OBJDIR, s.replace(".cu", ".o")) for s in B.SOURCES if s != "lpic_kernels.cu"]
so = os.path.join(out, f"{name}.so")
subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", so], check=True)
print(so)
