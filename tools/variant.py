"""Build an experimental libdit variant: one source recompiled with extra -D flags, linked with
the regular objects into paper_2604_08123_b200/build/variants/libdit_<name>.so.
usage: python tools/variant.py <name> <source.cu> -DFOO=1 ...   (then DIT_LIB_OVERRIDE=<path>)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as G  # noqa: E402

name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
G.build()
nccl = G._nccl_dir()
vd = os.path.join(G.BUILD, "variants")
os.makedirs(vd, exist_ok=True)
obj = os.path.join(vd, f"{name}_{src}.o")
common = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(nccl, "include"),
          "-I" + os.path.join(G.ROOT, "include")]
G._run([G.NVCC] + G.ARCH + common + flags + ["-x", "cu", "-c", os.path.join(G.CSRC, src), "-o", obj])
objs = [obj if s == src else os.path.join(G.BUILD, s + ".o") for s in G.SOURCES]
lib = os.path.join(vd, f"libdit_{name}.so")
G._run([G.NVCC] + G.ARCH + ["-shared", "-o", lib] + objs +
       ["-L" + os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nccl, "lib")])
print(lib)
