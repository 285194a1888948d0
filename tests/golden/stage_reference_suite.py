"""Stage the reference's own test suite next to the reference install so the
GPU box can run it against the drop-in (``tests/test_gpu_dropin_suite.py``).

    python tests/golden/stage_reference_suite.py   # in the build container

Copies ``/root/reference/pkg/tests`` and ``pkg/scenarios`` into
``baseline/_ref/condsim_suite/`` -- git-ignored like the rest of
``baseline/_ref`` (the ``pip install --target baseline/_ref`` of the
reference), never committed, but shipped to the GPU box with the snapshot.
The reference tree is only read here; nothing on the GPU box reads
``/root/reference``.
"""

import os
import shutil
import sys

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
DST = os.path.join(ROOT, "baseline", "_ref", "condsim_suite")


def main():
    if not os.path.isdir(REF):
        sys.exit("the reference tree is not present here")
    if os.path.isdir(DST):
        shutil.rmtree(DST)
    os.makedirs(DST)
    for sub in ("tests", "scenarios"):
        shutil.copytree(os.path.join(REF, sub), os.path.join(DST, sub))
    print("staged", sorted(os.listdir(os.path.join(DST, "tests"))), sorted(os.listdir(os.path.join(DST, "scenarios"))))


if __name__ == "__main__":
    main()
