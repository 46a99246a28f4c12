"""Build the library of an earlier commit as an A/B variant (experiment tooling):

    python scripts/build_base.py <git-rev> <tag>   ->  paper_2508_15010_b200/lib/variants/libtoast_<tag>.so

The commit's csrc/ and include/ are exported to a scratch directory and
compiled with the current build flags; scripts/gpu_ab_lib_n.sh <tag> then
times it beside the working tree's library on one box.
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_15010_b200 import build as b  # noqa: E402


def main():
    rev, tag = sys.argv[1], sys.argv[2]
    tmp = tempfile.mkdtemp(prefix="toast_base_")
    arc = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_2508_15010_b200/csrc", "include"],
                         check=True, capture_output=True).stdout
    subprocess.run(["tar", "-x", "-C", tmp], input=arc, check=True)
    src, inc = os.path.join(tmp, "paper_2508_15010_b200", "csrc"), os.path.join(tmp, "include")
    b.SRC, b.INC = src, inc
    b.CU_FLAGS = [f for f in b.CU_FLAGS if not f.startswith("-I")] + [f"-I{inc}", f"-I{src}"]
    b.CXX_FLAGS = [f for f in b.CXX_FLAGS if not f.startswith("-I")] + [f"-I{b.CUDA}/include", f"-I{inc}", f"-I{src}"]
    var = os.path.join(ROOT, "paper_2508_15010_b200", "lib", "variants")
    os.makedirs(var, exist_ok=True)
    print(b.build(force=True, lib=os.path.join(var, f"libtoast_{tag}.so"),
                  obj=os.path.join(ROOT, "paper_2508_15010_b200", "build", tag)))


if __name__ == "__main__":
    main()
