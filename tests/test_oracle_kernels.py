"""Oracle pins: MRS kernels (§7, Eqs. MRS_kernels / Velocity_1 /
Velocity_2 / AngularVelocity).

Pinned by closed forms (r = 0 and eps = 0), and by two identities the
mathematics fixes (checked by central differences in the target position,
independent of how the oracle writes the formulas):
  * div u = 0 for the regularized Stokeslet and rotlet velocities;
  * w = 1/2 curl u (rotlet: across its own outputs; Stokeslet: 1/2 curl u_S
    equals the 1/2 [f x d] Q term of Eq. AngularVelocity).
A wrong H1/H2/Q/D1/D2 coefficient or a dropped / mis-signed term breaks one.
"""
import numpy as np
import pytest

import oracle as O

NAMES = ["H1", "H2", "Q", "D1", "D2"]


def test_r0_closed_forms(golden):
    g = golden("mrs_closed_forms.json")
    for eps, key in [(0.01, "r0_eps_0.01"), (1.0, "r0_eps_1")]:
        v = O.mrs_scalars(0.0, eps)
        for i, nm in enumerate(NAMES):
            assert abs(v[i] / g[key][nm] - 1) < 4e-16


def test_eps0_textbook_limit(golden):
    g = golden("mrs_closed_forms.json")["eps0_r_1.7"]
    v = O.mrs_scalars(1.7, 0.0)
    for i, nm in enumerate(NAMES):
        assert abs(v[i] / g[nm] - 1) < 1e-15


def test_eps_to_zero_continuity():
    ref = O.mrs_scalars(1.0, 0.0)
    prev = None
    for eps in [1e-2, 1e-4, 1e-6]:
        d = np.max(np.abs(O.mrs_scalars(1.0, eps) / ref - 1))
        if prev is not None:
            assert d < prev
        prev = d
    assert prev < 1e-10


def _u(kernel, eps, x, y, f):
    return O.pair(kernel, eps, x, y, f)


def _jac(kernel, eps, x, y, f, h=1e-5):
    p = O.DIMS[kernel][1]
    J = np.zeros((p, 3))
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        J[:, a] = (_u(kernel, eps, x + e, y, f) - _u(kernel, eps, x - e, y, f)) / (2 * h)
    return J


def _curl(J):
    return np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]])


@pytest.mark.parametrize("eps", [0.3, 1.0])
def test_divergence_free_and_curl_identities(eps):
    rng = np.random.default_rng(3)
    for _ in range(10):
        x, y = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
        f = rng.uniform(-1, 1, 3)
        # Stokeslet: div u = 0; 1/2 curl u = 1/2 [f x d] Q  (Eq. AngularVelocity, f-term)
        J = _jac(O.STOKESLET, eps, x, y, f)
        scale = np.max(np.abs(J)) + 1e-300
        assert abs(np.trace(J)) < 1e-8 * scale
        d = x - y
        Q = O.mrs_scalars(np.linalg.norm(d), eps)[2]
        assert np.max(np.abs(0.5 * _curl(J) - 0.5 * np.cross(f, d) * Q)) < 1e-8 * scale
        # rotlet (reading A10): div u = 0, w = 1/2 curl u  (reading A9 for d D2)
        uw = _u(O.ROTLET, eps, x, y, f)
        Jr = _jac(O.ROTLET, eps, x, y, f)[:3]
        sc = np.max(np.abs(Jr)) + 1e-300
        assert abs(np.trace(Jr)) < 1e-8 * sc
        assert np.max(np.abs(0.5 * _curl(Jr) - uw[3:])) < 1e-8 * max(sc, np.max(np.abs(uw[3:])))


def test_combined_kernel_is_sum_of_parts():
    # Eqs. Velocity_2 / AngularVelocity with (f, n)
    rng = np.random.default_rng(5)
    for _ in range(10):
        x, y = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
        f, g = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
        eps = 0.2
        c = O.pair(O.STOKESLET_ROTLET, eps, x, y, np.concatenate([f, g]))
        s = O.pair(O.STOKESLET, eps, x, y, f)
        r = O.pair(O.ROTLET, eps, x, y, g)
        Q = O.mrs_scalars(np.linalg.norm(x - y), eps)[2]
        assert np.allclose(c[:3], s + r[:3], rtol=1e-14, atol=1e-15)
        assert np.allclose(c[3:], r[3:] + 0.5 * np.cross(f, x - y) * Q, rtol=1e-14, atol=1e-15)


def test_symmetries_and_linearity():
    rng = np.random.default_rng(11)
    for _ in range(20):
        x, y = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
        f, g = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
        a, b = rng.uniform(-2, 2, 2)
        eps = 0.05
        for K in [O.STOKESLET, O.ROTLET]:
            lhs = O.pair(K, eps, x, y, a * f + b * g)
            rhs = a * O.pair(K, eps, x, y, f) + b * O.pair(K, eps, x, y, g)
            assert np.allclose(lhs, rhs, rtol=1e-13, atol=1e-13 * np.max(np.abs(rhs)))
        # Stokeslet even in d; rotlet u odd, w even
        assert np.allclose(O.pair(O.STOKESLET, eps, x, y, f), O.pair(O.STOKESLET, eps, y, x, f), rtol=1e-15)
        r1, r2 = O.pair(O.ROTLET, eps, x, y, f), O.pair(O.ROTLET, eps, y, x, f)
        assert np.allclose(r1[:3], -r2[:3], rtol=1e-15) and np.allclose(r1[3:], r2[3:], rtol=1e-15)
        # Stokeslet reciprocity: f_a . u_b(x_a) = f_b . u_a(x_b) (symmetric tensor)
        assert abs(f @ O.pair(O.STOKESLET, eps, x, y, g) - g @ O.pair(O.STOKESLET, eps, y, x, f)) < 1e-13


def test_self_term_values(golden):
    g = golden("mrs_closed_forms.json")["r0_eps_1"]
    f = np.array([0.0, 1.0, 0.0])
    u = O.pair(O.STOKESLET, 1.0, np.zeros(3), np.zeros(3), f)
    assert np.allclose(u, [0, g["H1"], 0], rtol=1e-15, atol=0)
    uw = O.pair(O.ROTLET, 1.0, np.zeros(3), np.zeros(3), np.array([0, 0, 1.0]))
    assert np.allclose(uw, [0, 0, 0, 0, 0, g["D1"] / 4], rtol=1e-15, atol=0)


def test_non_homogeneous_for_eps_positive():
    # for eps != 0 no single power law across scales
    x, y, f = np.array([0.3, 0.1, -0.2]), np.zeros(3), np.array([1.0, 0.5, -0.25])
    u1 = O.pair(O.STOKESLET, 0.1, x, y, f)
    u2 = O.pair(O.STOKESLET, 0.1, 2 * x, y, f)
    u4 = O.pair(O.STOKESLET, 0.1, 4 * x, y, f)
    lam1 = np.log2(np.linalg.norm(u2) / np.linalg.norm(u1))
    lam2 = np.log2(np.linalg.norm(u4) / np.linalg.norm(u2))
    assert abs(lam1 - lam2) > 1e-6
