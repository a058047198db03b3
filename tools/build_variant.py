"""Build an in-tree variant of the library with extra nvcc flags (developer tool):
    python tools/build_variant.py libl0l2_prof.so -DL0L2_PROF
then run with L0L2_LIB=libl0l2_prof.so."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2602_04551_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
objdir = os.path.join(b.HERE, "build_" + name.replace(".so", ""))
os.makedirs(objdir, exist_ok=True)
nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
common = flags + b.ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", b._nccl_include(),
                           "-I", os.path.join(b.HERE, "..", "include")]
objs = []
for src in b.SOURCES:
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    subprocess.run([nvcc] + common + ["-c", os.path.join(b.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
subprocess.run([nvcc] + b.ARCH + ["-shared", "-o", os.path.join(b.HERE, name)] + objs + ["-ldl"], check=True)
print(os.path.join(b.HERE, name))
