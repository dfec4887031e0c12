"""Build an A/B variant of libenergon.so: recompile one source with extra -D flags and link a copy under
paper_2209_02341_b200/lib/ab/<name>.so (for AB_LIB in scripts/bench_attn.py / gemm_one.py).
Usage: python scripts/build_variant.py <name> <source.cu> -DFOO=1 ..."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import importlib
B = importlib.import_module("paper_2209_02341_b200.build")

name, src = sys.argv[1], sys.argv[2]
defs = sys.argv[3:]
B.build()
inc, libdir = B.nccl_dirs()
objdir = os.path.join(B.LIBDIR, "obj")
abdir = os.path.join(B.LIBDIR, "ab")
os.makedirs(abdir, exist_ok=True)
vobj = os.path.join(abdir, f"{name}_{os.path.basename(src)[:-3]}.o")
subprocess.check_call(["nvcc", "-O3", "-std=c++17", *B.ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler",
                       "-fvisibility=hidden", "--expt-relaxed-constexpr", "-I", os.path.join(B.ROOT, "include"), "-I",
                       inc, *defs, "-c", os.path.join(B.CSRC, src), "-o", vobj])
objs = [vobj if os.path.basename(o) == os.path.basename(src)[:-3] + ".o" else o
        for o in sorted(os.path.join(objdir, f) for f in os.listdir(objdir) if f.endswith(".o"))]
so = os.path.join(abdir, f"{name}.so")
subprocess.check_call(["nvcc", "-shared", *B.ARCH, "-o", so, *objs, "-L", libdir, "-l:libnccl.so.2", "-Xlinker",
                       f"-rpath={libdir}"])
print(so)
