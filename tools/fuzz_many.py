"""Extended GPU-vs-oracle fuzz (the tests/test_gpu_fuzz.py case generator over more seeds).
python tools/fuzz_many.py [first] [last]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as F  # noqa: E402

from paper_1902_02250_b200 import kitc  # noqa: E402

a, b = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (100, 250)
bad = 0
for case in range(a, b):
    try:
        F.test_fuzz(kitc, case)
    except AssertionError as e:
        bad += 1
        print("FAIL", case, str(e)[:300], flush=True)
print(f"cases {a}..{b - 1}: failures {bad}")
