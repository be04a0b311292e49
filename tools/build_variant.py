"""Experiment builds: compile liblgs.so with extra nvcc flags (e.g. -DLGS_FUSED_NB=128) into
<outdir>/liblgs.so (use variants/var_NAME: gpurun_out/ does not travel to the box), leaving the in-tree library alone.  python tools/build_variant.py OUTDIR FLAG..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_16144_b200 import build as B  # noqa: E402


def main():
    out, flags = sys.argv[1], sys.argv[2:]
    os.makedirs(out, exist_ok=True)
    nvcc = B._nvcc()
    objs, cmds = [], []
    for src in B.sources():
        obj = os.path.join(out, src.replace(".cu", ".o"))
        objs.append(obj)
        cmds.append([nvcc, *B.ARCH, *B.COMMON, *B.PER_FILE.get(src, []), *flags, "-c", os.path.join(B.CSRC, src),
                     "-o", obj])
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
        list(pool.map(lambda c: subprocess.run(c, check=True), cmds))
    subprocess.run([nvcc, *B.ARCH, "-shared", "-cudart", "static", "-o", os.path.join(out, "liblgs.so"), *objs],
                   check=True)


if __name__ == "__main__":
    main()
