"""B200-native hot path of the barycentric Lagrange KITC (arXiv:1902.02250).

The compute lives in libkitc.so (csrc/, C ABI in include/kitc.h); `kitc` is
its ctypes binding.  Importing `paper_1902_02250_b200.kitc` raises if the
library has not been built -- there is no CPU fallback.
"""
