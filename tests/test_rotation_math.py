"""Derivation check for the rotation-based M2L (point-and-shoot, PAPER.md:3485-3500;
SPEC.md:120-123) in this code's solid-harmonic basis, independent of the C++/CUDA:
rotate the multipole so the offset lies on +z (W), translate along z with the
scalar coefficients (-1)^{n+m} (j+n)!/rho^{j+n+1}, rotate the local back (V).
W and V come from Wigner small-d via
  W_{k k'} = (-1)^{k+k'} A_{n|k|}/A_{n|k'|} d^n_{k'k}(-theta) e^{i k phi},
  V_{k k'} = (-1)^{k+k'} A_{n|k'|}/A_{n|k|} e^{-i k' phi} d^n_{k'k}(theta),
A_{n,a} = sqrt((n-a)!(n+a)!); the product must equal the dense M2L operator."""
from math import factorial as F

import numpy as np
import pytest

scipy_special = pytest.importorskip("scipy.special")


def _P(n, m, x):
    return (-1) ** m * scipy_special.lpmv(m, n, x)  # no Condon-Shortley phase


def _sph(v):
    r = np.linalg.norm(v)
    return r, np.arccos(np.clip(v[2] / r, -1, 1)), np.arctan2(v[1], v[0])


def _R(n, m, v):
    r, th, ph = _sph(v)
    a = abs(m)
    if a > n:
        return 0
    val = r ** n * _P(n, a, np.cos(th)) * np.exp(1j * a * ph) / F(n + a)
    return val if m >= 0 else (-1) ** a * np.conj(val)


def _I(n, m, v):
    r, th, ph = _sph(v)
    a = abs(m)
    if a > n:
        return 0
    val = F(n - a) * _P(n, a, np.cos(th)) * np.exp(1j * a * ph) / r ** (n + 1)
    return val if m >= 0 else (-1) ** a * np.conj(val)


def _d(l, mp, m, b):
    s = 0.0
    for k in range(max(0, m - mp), min(l + m, l - mp) + 1):
        num = np.sqrt(F(l + m) * F(l - m) * F(l + mp) * F(l - mp))
        den = F(l + m - k) * F(k) * F(l - k - mp) * F(k - m + mp)
        s += (-1) ** (k - m + mp) * num / den * np.cos(b / 2) ** (2 * l - 2 * k + m - mp) * \
            np.sin(b / 2) ** (2 * k - m + mp)
    return s


def _A(n, a):
    return np.sqrt(F(n - a) * F(n + a))


@pytest.mark.parametrize("v", [(2.0, -4.0, 6.0), (0.0, 0.0, -6.0), (-8.0, 2.0, 0.0), (4.0, 4.0, 4.0)])
def test_rotation_m2l_equals_dense(v):
    p = 6
    v = np.array(v)
    rho = np.linalg.norm(v)
    th, ph = np.arccos(v[2] / rho), np.arctan2(v[1], v[0])

    def W(n):
        return np.array([[(-1) ** (k + kp) * _A(n, abs(k)) / _A(n, abs(kp)) * _d(n, kp, k, -th) * np.exp(1j * k * ph)
                          for kp in range(-n, n + 1)] for k in range(-n, n + 1)])

    def V(n):
        return np.array([[(-1) ** (k + kp) * _A(n, abs(kp)) / _A(n, abs(k)) * np.exp(-1j * kp * ph) * _d(n, kp, k, th)
                          for kp in range(-n, n + 1)] for k in range(-n, n + 1)])

    rng = np.random.default_rng(1)
    src = rng.normal(size=(3, 3)) * 0.3
    M = {(j, k): sum(np.conj(_R(j, k, s)) for s in src) for j in range(p + 1) for k in range(-j, j + 1)}
    Mp = {}
    for j in range(p + 1):
        w = W(j)
        for kp in range(-j, j + 1):
            Mp[j, kp] = sum(M[j, k] * w[k + j, kp + j] for k in range(-j, j + 1))
    Lp = {(n, m): (-1) ** (n + m) * sum(Mp[j, m] * F(j + n) / rho ** (j + n + 1) for j in range(abs(m), p + 1))
          for n in range(p + 1) for m in range(-n, n + 1)}
    L = {}
    for n in range(p + 1):
        vv = V(n)
        for mp in range(-n, n + 1):
            L[n, mp] = sum(Lp[n, m] * vv[m + n, mp + n] for m in range(-n, n + 1))
    dense = {(n, m): (-1) ** (n + m) * sum(M[j, k] * _I(j + n, k - m, v) for (j, k) in M)
             for n in range(p + 1) for m in range(-n, n + 1)}
    scale = max(abs(x) for x in dense.values())
    assert max(abs(L[k] - dense[k]) for k in L) <= 1e-13 * scale
