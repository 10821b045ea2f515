"""C-ABI checks that need no GPU: libkitc.so builds for sm_100a, loads, and
exports every symbol include/kitc.h declares; argument validation paths that
return before any CUDA call."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1902_02250_b200 import build as B
    B.build()
    return C.CDLL(B.LIB)


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kitc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kitc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("kitc_build_tree", "kitc_modified_weights", "kitc_eval", "kitc_direct"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_1902_02250_b200 import build as B
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (kitc_\w+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(lib, s)


def test_binding_names_match_header():
    from paper_1902_02250_b200 import kitc
    assert sorted(kitc.EXPORTS) == declared_symbols()


def test_sm100a_code_present():
    from paper_1902_02250_b200 import build as B
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validation_without_gpu():
    from paper_1902_02250_b200 import kitc
    assert kitc.kitc_kernel_dims(kitc.STOKESLET) == (3, 3)
    assert kitc.kitc_kernel_dims(kitc.ROTLET) == (3, 6)
    assert kitc.kitc_kernel_dims(kitc.STOKESLET_ROTLET) == (6, 6)
    with pytest.raises(kitc.KitcError) as e:
        kitc.kitc_kernel_dims(5)
    assert e.value.status == kitc.KITC_EINVAL
    # direct: unknown kernel, SELF_OMIT with distinct target/source arrays, negative eps
    fake = C.c_void_p(16)
    with pytest.raises(kitc.KitcError):
        kitc.kitc_direct(9, 0.01, kitc.SELF_INCLUDE, fake, 1, fake, fake, 1, fake, None)
    with pytest.raises(kitc.KitcError):
        kitc.kitc_direct(0, 0.01, kitc.SELF_OMIT, fake, 1, C.c_void_p(32), fake, 1, fake, None)
    with pytest.raises(kitc.KitcError):
        kitc.kitc_direct(0, -1.0, kitc.SELF_INCLUDE, fake, 1, fake, fake, 1, fake, None)
    h = kitc.kitc_tree_create()
    with pytest.raises(kitc.KitcError) as e:
        kitc.kitc_build_tree(h, fake, 0, 10, None)           # N < 1
    assert e.value.status == kitc.KITC_EINVAL
    with pytest.raises(kitc.KitcError) as e:
        kitc.kitc_tree_info(h)                                # not built
    assert e.value.status == kitc.KITC_ESTATE
    kitc.kitc_tree_free(h)


def test_fhat_cluster_len(lib):
    # [round][k3][comp][8 rows], rounds = ceil((n+1)^2 / 8)  (include/kitc.h)
    ln = C.c_int64()
    for kern, m in ((0, 3), (1, 3), (2, 6)):
        for n in (1, 4, 8, 16):
            P = n + 1
            assert lib.kitc_fhat_cluster_len(kern, n, C.byref(ln)) == 0
            assert ln.value == -(-P * P // 8) * P * m * 8
    assert lib.kitc_fhat_cluster_len(0, 0, C.byref(ln)) == -1
    assert lib.kitc_fhat_cluster_len(0, 17, C.byref(ln)) == -1
    assert lib.kitc_fhat_cluster_len(7, 4, C.byref(ln)) == -1


def test_rods_generator_matches_paper_example2():
    # N = N_r (M + 1); slab ~16^2 x 9 at N_r = 15^2, ~85^2 x 9 at 80^2
    import numpy as np
    import kitc_inputs as KI
    X, W = KI.particles(15 * 15 * 151, "rods", m=6)
    assert X.shape == (33975, 3) and W.shape == (33975, 6)       # the paper's smallest N
    ext = X.max(0) - X.min(0)
    assert abs(ext[0] - 16) < 1 and abs(ext[1] - 16) < 1 and ext[2] == 9.0
    X, _ = KI.config_particles("X2")
    assert X.shape[0] == 966400                                   # Table 5's N
    ext = X.max(0) - X.min(0)
    assert abs(ext[0] - 85) < 1 and ext[2] == 9.0
    # rod 0 follows (x0 + 0.3 cos 2z, y0 + 0.3 sin 2z, z)
    z = X[:151, 2]
    assert np.allclose(X[:151, 0] - X[0, 0], 0.3 * (np.cos(2 * z) - 1), atol=1e-12)


def test_binding_declares_every_signature():
    # every exported call has ctypes argtypes (no implicit int/float conversion)
    from paper_1902_02250_b200 import kitc
    assert sorted(kitc.SIGNATURES) == sorted(kitc.EXPORTS)
    src = open(os.path.join(ROOT, "include", "kitc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    for name, args in kitc.SIGNATURES.items():
        m = re.search(r"\b" + name + r"\s*\(([^)]*)\)", src)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name


def test_organisms_generator_matches_paper_example1():
    # pairs (body, flagellum) at distance 0.02 in a side-10 cube, unit forces +-t
    import numpy as np
    import kitc_inputs as KI
    X, W = KI.particles(10000, "organisms", seed=3)
    d = X[1::2] - X[0::2]
    assert np.allclose(np.linalg.norm(d, axis=1), 0.02, rtol=1e-12)
    assert np.allclose(W[0::2], d / 0.02, atol=1e-12) and np.array_equal(W[1::2], -W[0::2])
    assert X[0::2].min() >= 0 and X[0::2].max() <= 10
    assert KI.CONFIGS["X1"]["N"] == 640_000 and KI.CONFIGS["X1L"]["N"] == 5_120_000   # Table 1 rows


def test_plain_c_client(lib, tmp_path):
    # the boundary is a C ABI: a C99 program includes kitc.h, links libkitc.so and calls it
    # (no torch, no Python), exercising the argument checks that need no GPU
    from paper_1902_02250_b200 import build as B
    src = tmp_path / "client.c"
    src.write_text(r"""
#include "kitc.h"
#include <stdio.h>
int main(void) {
    int64_t len = 0;
    int32_t m = 0, p = 0;
    if (kitc_fhat_cluster_len(KITC_ROTLET, 8, &len) != KITC_OK || len != 11 * 9 * 3 * 8) return 1;
    if (kitc_kernel_dims(KITC_STOKESLET_ROTLET, &m, &p) != KITC_OK || m != 6 || p != 6) return 2;
    if (kitc_fhat_cluster_len(KITC_STOKESLET, 17, &len) != KITC_EINVAL) return 3;
    if (kitc_last_error()[0] == 0) return 4;
    puts("ok");
    return 0;
}
""")
    exe = tmp_path / "client"
    libdir = os.path.dirname(B.LIB)
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                           "-L", libdir, "-lkitc", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", (out.returncode, out.stdout, out.stderr)


def test_tree_workspace_bytes():
    # kitc_tree_workspace_bytes: an upper bound that covers at least the sorted
    # coordinates + scratch, the worst-case (2N - 1 clusters) table, and grows with N and n
    from paper_1902_02250_b200 import kitc
    b1 = kitc.kitc_tree_workspace_bytes(10_000, 100, kitc.STOKESLET, 8)
    b2 = kitc.kitc_tree_workspace_bytes(20_000, 100, kitc.STOKESLET, 8)
    assert b2 > b1 > 10_000 * (6 * 8 + 2 * 4)
    assert kitc.kitc_tree_workspace_bytes(10_000, 100, kitc.STOKESLET, 10) > b1
    assert kitc.kitc_tree_workspace_bytes(10_000, 100, kitc.STOKESLET_ROTLET, 8) > b1
    for bad in ((0, 100, 0, 8), (10, 0, 0, 8), (10, 5, 7, 8), (10, 5, 0, 17)):
        with pytest.raises(kitc.KitcError) as e:
            kitc.kitc_tree_workspace_bytes(*bad)
        assert e.value.status == kitc.KITC_EINVAL


def test_product_library_has_the_checks_compiled_out():
    # libkitc.so is the product build (KITC_BUILD_CHECKS clear); libkitc_checks.so, the
    # verification build tests/test_gpu_checks.py loads, sets it.  No CUDA call is made.
    import ctypes
    from paper_1902_02250_b200 import build as B, kitc
    if os.environ.get("KITC_LIB"):
        pytest.skip("a tuning / verification library is loaded")
    assert kitc.kitc_build_flags() == 0
    if os.path.exists(B.CHECKS_LIB):
        lib = ctypes.CDLL(B.CHECKS_LIB)
        lib.kitc_build_flags.restype = ctypes.c_uint32
        assert lib.kitc_build_flags() == 1
