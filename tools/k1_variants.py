"""K1 tuning sweep. On the CPU side (`build`), compile k1_superpose.cu with
each knob setting and link it with the other objects into
paper_2511_20432_b200/_lib/variants/<name>.so; on the GPU (`run`), time the
config-1 superposition for every variant x points-per-thread (TG_K1_P),
loading each build through TG_LIB_VARIANT.

  python tools/k1_variants.py build
  python tools/k1_variants.py run [P ...]
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2511_20432_b200", "_lib", "variants")

VARIANTS = {
    "planar_sweep": dict(K1_PLANAR_SWEEP=1),
}


def build():
    from paper_2511_20432_b200 import _build as B
    B.build()
    os.makedirs(VDIR, exist_ok=True)
    k1 = os.path.join(B.CSRC, "k1_superpose.cu")
    others = [B._obj_for(s) for s in B._sources() if s != k1]
    for name, defs in VARIANTS.items():
        obj = os.path.join(B.OBJDIR, f"k1_{name}.o")
        d = [f"-D{k}={v}" for k, v in defs.items()]
        subprocess.run([B.NVCC, *B.ARCH, *B.COMMON, *d, "-c", k1, "-o", obj], check=True)
        subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o",
                        os.path.join(VDIR, f"{name}.so"), obj, *others, *B.LINK], check=True)
        print("built", name)


def run(Ps):
    for so in sorted(glob.glob(os.path.join(VDIR, "*.so"))):
        for P in Ps:
            env = dict(os.environ, TG_K1_P=P, TG_LIB_VARIANT=so)
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "k1_sweep.py"), "--one"],
                               env=env, capture_output=True, text=True)
            out = r.stdout.strip() or r.stderr[-1500:]
            try:
                d = json.loads(out)
                d["variant"] = os.path.basename(so)[:-3]
                print(json.dumps(d), flush=True)
            except ValueError:
                print(os.path.basename(so), P, out, flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[2:] or ["4", "6", "8"])
