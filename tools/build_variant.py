"""Build a variant of libthermiga_b200.so with extra -D flags on chosen
sources (tuning runs: TG_LIB_VARIANT=<path> selects it at load time).
  python tools/build_variant.py NAME "k5_fused.cu" -DK5_TA=128 -DK5_THREADS=512 -DK5_MINB=1"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_20432_b200 import _build as B
name, files, flags = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build()
out_dir = os.path.join(B.LIBDIR, "variants")
os.makedirs(out_dir, exist_ok=True)
objs = []
for src in B._sources():
    if os.path.basename(src) in files:
        obj = os.path.join(out_dir, f"{name}__{os.path.basename(src)}.o")
        cmd = [B.NVCC, *B.ARCH, *B.COMMON, *flags, "-c", src, "-o", obj]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    else:
        objs.append(B._obj_for(src))
lib = os.path.join(out_dir, f"lib_{name}.so")
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, *B.LINK], check=True)
print(lib)
