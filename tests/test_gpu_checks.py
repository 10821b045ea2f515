"""Device-side invariant checks, the stand-in for compute-sanitizer (closed on the GPU pool):
the GPU parity cases and an exercise of every entry point run on libkitc_checks.so, the same
sources built with -DKITC_CHECKS (csrc/kitc_internal.cuh).  That build checks, in every
launch, the index bounds the kernels rely on: batch and target positions, popped cluster ids
and their topology (particle ranges inside [0, N), children after their parent), the lane
masks of the traversal stack, the DFS stack capacity, the TMA stage sizes against the warp's
shared-memory carve-out, near-field source ranges, output rows, the tree scatter positions
(children partition their parent's range) and the modified-weights work items.  A violation
prints its location and traps, which fails the subprocess.  The product library has the
checks compiled out."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def checks_env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1902_02250_b200 import build as B
    lib = B.build(checks=True)  # built by __graft_entry__.build(); rebuilt here only if stale
    return dict(os.environ, KITC_LIB=lib)


def _run(cmd, env, timeout):
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    out = r.stdout + r.stderr
    assert "KITC_CHECKS" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    return out


def test_every_entry_point_under_checks(checks_env):
    """Tree build, modified weights (direct, per-peer replicas), eval (stats, size check, interleaved
    part), separate targets, direct sum, sampled direct sum, E: three kernels, uniform / sphere / rods,
    n = 2 .. 12 (the runtime-degree kernel included), N from 7 to 3775."""
    out = _run([sys.executable, "tools/sanitize_run.py"], checks_env, 900)
    assert out.count(" E ") >= 5, out[-2000:]
    assert "build flags 1 " in out, out[-2000:]  # the checks are compiled into the library that ran


def test_parity_suite_under_checks(checks_env):
    """The GPU-vs-oracle parity, fuzz and separate-target cases, unchanged, on the checked build."""
    _run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu and not slow",
          "tests/test_gpu_parity.py", "tests/test_gpu_fuzz.py", "tests/test_gpu_targets.py"], checks_env, 1800)
