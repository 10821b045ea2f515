"""Oracle pins: Chebyshev nodes, barycentric weights, mapped grids and the
barycentric Lagrange basis (§2-§3; Algorithm 1 flag path
P:540-547).  Pinned against closed forms and the product-form Lagrange
polynomials (Eq. Lagrange_polynomial) evaluated in 50-digit mpmath.
"""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle as O

ULP1 = 2.3e-16


def test_nodes_closed_form(golden):
    g = golden("nodes_weights.json")
    for n, vals in g["nodes"].items():
        t = O.cheb_nodes(int(n))
        assert np.max(np.abs(t - np.array(vals))) <= ULP1
        assert t[0] == 1.0 and t[-1] == -1.0


@pytest.mark.parametrize("n", range(1, 17))
def test_nodes_vs_cos_and_symmetry(n):
    t = O.cheb_nodes(n)
    mp.mp.dps = 30
    for k in range(n + 1):
        assert abs(t[k] - float(mp.cos(k * mp.pi / n))) <= ULP1   # Eq. Chebyshev_points
        assert t[k] == -t[n - k]                                  # reading A12: exact symmetry
    if n % 2 == 0:
        assert t[n // 2] == 0.0
    assert np.all(np.diff(t) < 0)                                # descending in k


def test_weights_closed_form(golden):
    g = golden("nodes_weights.json")
    for n, vals in g["weights"].items():
        assert list(O.bary_weights(int(n))) == vals


@pytest.mark.parametrize("n", [1, 2, 5, 8, 13])
def test_weights_are_scaled_true_barycentric_weights(n):
    # Eq. Barycentric-1D: w_k = 1/prod_{j!=k}(s_k - s_j); the simple weights are
    # these times one common constant (scale invariance).
    mp.mp.dps = 50
    s = [mp.cos(k * mp.pi / n) for k in range(n + 1)]
    true = [1 / mp.fprod(s[k] - s[j] for j in range(n + 1) if j != k) for k in range(n + 1)]
    w = O.bary_weights(n)
    ratio = [true[k] / w[k] for k in range(n + 1)]
    for r in ratio:
        assert abs(r / ratio[0] - 1) < 1e-25


def test_grid_mapping_and_pinned_endpoints():
    for n in [1, 2, 4, 7, 8]:
        for lo, hi in [(-1.0, 1.0), (0.3, 0.9), (3.0, 5.0), (-7.25, -7.0)]:
            s = O.grid(n, lo, hi)
            assert s[0] == hi and s[n] == lo                       # reading A13
            mp.mp.dps = 30
            for k in range(1, n):
                exact = (mp.mpf(lo) + mp.mpf(hi)) / 2 + mp.cos(k * mp.pi / n) * (mp.mpf(hi) - mp.mpf(lo)) / 2
                assert abs(s[k] - float(exact)) <= 4e-16 * max(1.0, abs(lo), abs(hi))
    assert list(O.grid(2, 3.0, 5.0)) == [5.0, 4.0, 3.0]


def test_basis_worked_values(golden):
    g = golden("nodes_weights.json")
    assert np.allclose(O.basis(2, O.grid(2, -1, 1), 0.5), g["basis_n2_t05"]["value"], rtol=0, atol=1e-16)
    assert np.allclose(O.basis(1, O.grid(1, -1, 1), 0.5), g["basis_n1_t05"]["value"], rtol=0, atol=1e-16)


def _product_form(s, k, t):
    # Eq. Lagrange_polynomial in mpmath
    num = mp.fprod(mp.mpf(t) - mp.mpf(s[j]) for j in range(len(s)) if j != k)
    den = mp.fprod(mp.mpf(s[k]) - mp.mpf(s[j]) for j in range(len(s)) if j != k)
    return num / den


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 8, 10, 12])
def test_basis_vs_product_form(n):
    mp.mp.dps = 50
    rng = np.random.default_rng(n)
    for lo, hi in [(-1.0, 1.0), (0.25, 0.75), (-3.0, 11.0)]:
        s = O.grid(n, lo, hi)
        for t in rng.uniform(lo, hi, 12):
            L = O.basis(n, s, t)
            ref = np.array([float(_product_form(s, k, t)) for k in range(n + 1)])
            assert np.max(np.abs(L - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("n", [1, 2, 5, 8, 11])
def test_basis_node_reproduction_is_exact(n):
    s = O.grid(n, -0.3, 0.8)
    for j in range(n + 1):
        e = np.zeros(n + 1)
        e[j] = 1.0
        assert np.array_equal(O.basis(n, s, s[j]), e)                # flag path


@pytest.mark.parametrize("n", [1, 3, 8, 10])
def test_partition_of_unity_and_polynomial_reproduction(n):
    rng = np.random.default_rng(7)
    lo, hi = -0.4, 1.3
    s = O.grid(n, lo, hi)
    coef = rng.standard_normal(n + 1)
    for t in rng.uniform(lo, hi, 40):
        L = O.basis(n, s, t)
        assert abs(L.sum() - 1.0) <= 1e-14
        q = np.polynomial.polynomial.polyval(s, coef)
        assert abs(L @ q - np.polynomial.polynomial.polyval(t, coef)) <= 1e-12 * np.abs(coef).sum() * 2 ** n


def test_scale_invariance():
    # same simple weights on any interval: basis on [a,b] at the
    # mapped point equals basis on [-1,1] at the preimage
    n = 7
    a, b = 2.0, 5.0
    s = O.grid(n, a, b)
    s0 = O.grid(n, -1, 1)
    for u in np.linspace(-0.95, 0.95, 11):
        t = 0.5 * (a + b + u * (b - a))
        assert np.max(np.abs(O.basis(n, s, t) - O.basis(n, s0, u))) <= 1e-13


def test_runge_convergence():
    f = lambda t: 1.0 / (1.0 + 25.0 * t * t)
    errs = []
    for n in [10, 20, 40]:
        s = O.grid(n, -1, 1)
        ts = np.linspace(-1, 1, 301)
        errs.append(max(abs(O.basis(n, s, t) @ f(s) - f(t)) for t in ts))
    assert errs[0] > errs[1] > errs[2]
    # Chebyshev interpolation of a function analytic in the Bernstein ellipse
    # rho = (1 + sqrt(26))/5 converges like rho^-n
    rho = (1 + math.sqrt(26)) / 5
    assert errs[2] < 10 * rho ** -40
