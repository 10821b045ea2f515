"""Tuning builds: python tools/build_variant.py NAME -DFOO=1 ... -> tools/variants/libkitc_NAME.so
(selected at run time with KITC_LIB=...; the product build is paper_1902_02250_b200/build.py)."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_02250_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "tools", "variants"), exist_ok=True)
out = os.path.join(ROOT, "tools", "variants", f"libkitc_{name}.so")
cus = sorted(glob.glob(os.path.join(ROOT, "paper_1902_02250_b200", "csrc", "*.cu")))
subprocess.check_call(["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, *defs, "-o", out, *cus])
print(out)
