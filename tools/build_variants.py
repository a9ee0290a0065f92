"""Build A/B variants of libmig.so into build/var/<name>.so: every source compiled once (build/obj), and
one source (VAR_SRC, default simulate_lane.cu; simulate_ff.cu for k_ff_lane / k_base_lane) recompiled per variant
with extra -D flags. Usage:
  python tools/build_variants.py name1='-DFOO=1' name2='-DFOO=2' ...   (then: gpurun -- 'bash tools/gpu_ab.sh')"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402

FLAGS = [ge.NVCC, *ge.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--fmad=false", "-Iinclude"]


def obj(src, out, extra=()):
    subprocess.run(FLAGS + list(extra) + ["-c", src, "-o", out], check=True, cwd=ROOT)
    return out


def main():
    os.makedirs(os.path.join(ROOT, "build/obj"), exist_ok=True)
    os.makedirs(os.path.join(ROOT, "build/var"), exist_ok=True)
    for f in ([] if os.environ.get("VAR_KEEP") else os.listdir(os.path.join(ROOT, "build/var"))):
        os.remove(os.path.join(ROOT, "build/var", f))
    var_src = os.environ.get("VAR_SRC", "paper_2508_18556_b200/csrc/simulate_lane.cu")
    others = [s for s in ge.MIG_SOURCES if s != var_src]
    variants = [a.split("=", 1) for a in sys.argv[1:]]
    with ThreadPoolExecutor(8) as ex:
        futs = [ex.submit(obj, s, f"build/obj/{os.path.basename(s)}.o") for s in others]
        vfuts = [ex.submit(obj, var_src, f"build/obj/var_{n}.o", fl.split())
                 for n, fl in variants]
        objs = [f.result() for f in futs]
        vobjs = [f.result() for f in vfuts]
    for (n, _), vo in zip(variants, vobjs):
        subprocess.run([ge.NVCC, *ge.ARCH, "-shared", "-o", f"build/var/{n}.so", *objs, vo, "-ldl"], check=True,
                       cwd=ROOT)
        print("built", n)


if __name__ == "__main__":
    main()
