"""Build two libmig.so variants for an A/B: build/var/old.so from the committed (HEAD, or REV) sources and
build/var/new.so from the working tree. Usage: python tools/build_ab.py [REV]"""
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402

FLAGS = [ge.NVCC, *ge.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--fmad=false"]


def main():
    rev = sys.argv[1] if len(sys.argv) > 1 else "HEAD"
    old = "/tmp/ab_old"
    shutil.rmtree(old, ignore_errors=True)
    subprocess.run(f"git archive {rev} | tar -x -C {old}" if False else f"mkdir -p {old} && git archive {rev} | tar -x -C {old}",
                   shell=True, check=True, cwd=ROOT)
    os.makedirs(os.path.join(ROOT, "build/var"), exist_ok=True)
    for f in os.listdir(os.path.join(ROOT, "build/var")):
        os.remove(os.path.join(ROOT, "build/var", f))

    def build(tree, name):
        objdir = f"/tmp/ab_obj_{name}"
        shutil.rmtree(objdir, ignore_errors=True)
        os.makedirs(objdir, exist_ok=True)
        with ThreadPoolExecutor(8) as ex:
            srcs = [s for s in ge.MIG_SOURCES if os.path.exists(f"{tree}/{s}")]  # the tree's own sources
            objs = list(ex.map(lambda s: (subprocess.run(FLAGS + [f"-I{tree}/include", "-c", f"{tree}/{s}", "-o",
                                                                  f"{objdir}/{os.path.basename(s)}.o"], check=True),
                                          f"{objdir}/{os.path.basename(s)}.o")[1], srcs))
        subprocess.run([ge.NVCC, *ge.ARCH, "-shared", "-o", os.path.join(ROOT, f"build/var/{name}.so"), *objs, "-ldl"],
                       check=True)
        print("built", name)

    build(old, "old")
    build(ROOT, "new")


if __name__ == "__main__":
    main()
