"""Build a tuning variant of libvfpi.so: one translation unit recompiled with
extra -D flags, linked with the other objects of the in-tree build.

    python scripts/build_variant.py NAME vfpi_resident.cu -DVFPI_RES_FREE_START=2 ...
    VFPI_LIB=paper_2201_09212_b200/_variants/libvfpi_NAME.so python scripts/cfg1_solve.py

(the variant .so is git-ignored and travels to the GPU box with the snapshot)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09212_b200 import build as B  # noqa: E402


def main():
    name, unit, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    objdir = os.path.join(ROOT, "build", "obj")
    vdir = os.path.join(ROOT, "build", "var_" + name)
    out = os.path.join(B.HERE, "_variants")
    os.makedirs(vdir, exist_ok=True)
    os.makedirs(out, exist_ok=True)
    cflags = [f for f in B.NVCC_FLAGS if f != "-shared"]
    vobj = os.path.join(vdir, unit.replace(".cu", ".o"))
    subprocess.run([B._nvcc(), *cflags, *defs, "-c", "-o", vobj, os.path.join(B.CSRC, unit)], check=True)
    objs = [vobj if s == unit else os.path.join(objdir, s.replace(".cu", ".o")) for s in B.SOURCES]
    lib = os.path.join(out, f"libvfpi_{name}.so")
    subprocess.run([B._nvcc(), *B.NVCC_FLAGS, "-o", lib, *objs], check=True)
    print(lib)


if __name__ == "__main__":
    main()
