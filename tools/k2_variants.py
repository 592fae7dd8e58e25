"""K2 tuning sweep (as tools/k1_variants.py, for k2_kron.cu): build variant
libraries on the CPU side, time the config-4 solve per variant on the GPU.

  python tools/k2_variants.py build
  python tools/k2_variants.py run
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2511_20432_b200", "_lib", "variants_k2")

VARIANTS = {
    "base": dict(),
    "nosweep": dict(K2_STUDY_NOSWEEP=1),
}


def build():
    from paper_2511_20432_b200 import _build as B
    B.build()
    os.makedirs(VDIR, exist_ok=True)
    src = os.path.join(B.CSRC, os.environ.get("TG_VARIANT_SRC", "k2_kron.cu"))
    others = [B._obj_for(s) for s in B._sources() if s != src]
    for name, defs in VARIANTS.items():
        obj = os.path.join(B.OBJDIR, f"k2_{name}.o")
        d = [f"-D{k}={v}" for k, v in defs.items()]
        subprocess.run([B.NVCC, *B.ARCH, *B.COMMON, *d, "-c", src, "-o", obj], check=True)
        subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o",
                        os.path.join(VDIR, f"{name}.so"), obj, *others, *B.LINK], check=True)
        print("built", name)


def run():
    for so in sorted(glob.glob(os.path.join(VDIR, "*.so"))):
        env = dict(os.environ, TG_LIB_VARIANT=so, TG_K2_ALGOS="cg1")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "k2_algos.py"),
                            *sys.argv[2:]],
                           env=env, capture_output=True, text=True)
        for line in (r.stdout.strip() or r.stderr[-1500:]).splitlines():
            print(os.path.basename(so)[:-3], line, flush=True)


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run()
