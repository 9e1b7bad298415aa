"""Riemannian geometry of U(4) and U(2) x U(2) (host 4x4 math).

Same semantics as the reference ``gatefit.manifold`` (reference
manifold.py:42-172): metric Re Tr[X^dag Y], tangent projection
``V asym(V^dag X)``, polar retraction via the SVD, holomorphic -> Euclidean
gradient ``-conj(D)``, the Riemannian Hessian action, and parity-block
handling where U(2) x U(2) gates are treated blockwise (odd block rows/cols
{1, 2}, even block {0, 3}).  O(n_logical) 4x4 operations -- no kernels.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "DegenerateRetractionError",
    "asym",
    "project_tangent",
    "retract_polar",
    "inner",
    "euclid_gradient_from_holomorphic",
    "riemannian_hessian_apply",
    "parity_split",
    "parity_join",
    "project_tangent_gate",
    "retract_gate",
    "hessian_apply_gate",
    "random_unitary",
]

PARITY_ODD = (1, 2)
PARITY_EVEN = (0, 3)
_OFF = np.array([1, 2, 4, 7, 8, 11, 13, 14])


class DegenerateRetractionError(ValueError):
    """V + X is numerically rank deficient: the polar factor is not unique."""


def _dag(a):
    return np.conj(a).T


def asym(a: np.ndarray) -> np.ndarray:
    return (a - _dag(a)) / 2.0


def project_tangent(v, x):
    return v @ asym(_dag(v) @ x)


def retract_polar(v, x):
    w, s, vh = np.linalg.svd(v + x)
    if s[-1] <= 1e-14 * max(s[0], 1.0):
        raise DegenerateRetractionError(f"retraction point is rank deficient (smallest singular value {s[-1]:.3e})")
    return w @ vh


def inner(x, y) -> float:
    t = np.sum(np.conj(x) * y)  # Tr[X^dag Y]
    if abs(t.imag) > 1e-10 * max(1.0, abs(t)):
        raise ValueError(f"inner product has non-negligible imaginary part {t.imag:.3e}")
    return float(t.real)


def euclid_gradient_from_holomorphic(d):
    return -np.conj(d)


def riemannian_hessian_apply(v, euclid_grad, euclid_grad_derivative, x):
    """P_V( X asym(V^dag g) + V asym(X^dag g + V^dag Dg[X]) )."""
    vg = asym(_dag(v) @ euclid_grad)
    term = asym(_dag(x) @ euclid_grad + _dag(v) @ euclid_grad_derivative)
    return project_tangent(v, x @ vg + v @ term)


def parity_split(g, tol: float = 1e-12):
    g = np.asarray(g)
    flat = g.reshape(16)
    bad = np.abs(flat[_OFF]) > tol
    if np.any(bad):
        e = int(_OFF[np.argmax(bad)])
        raise ValueError(f"matrix entry ({e // 4},{e % 4}) = {flat[e]:.3e} violates the parity pattern")
    return g[np.ix_(PARITY_ODD, PARITY_ODD)].copy(), g[np.ix_(PARITY_EVEN, PARITY_EVEN)].copy()


def parity_join(odd, even):
    g = np.zeros((4, 4), dtype=np.complex128)
    g[np.ix_(PARITY_ODD, PARITY_ODD)] = odd
    g[np.ix_(PARITY_EVEN, PARITY_EVEN)] = even
    return g


def _by_blocks(fn, v, *rest):
    vo, ve = parity_split(v)
    blocks = [parity_split(m, tol=np.inf) for m in rest]
    return parity_join(fn(vo, *(b[0] for b in blocks)), fn(ve, *(b[1] for b in blocks)))


def project_tangent_gate(v, x, parity: bool = False):
    return _by_blocks(project_tangent, v, x) if parity else project_tangent(v, x)


def retract_gate(v, x, parity: bool = False):
    return _by_blocks(retract_polar, v, x) if parity else retract_polar(v, x)


def hessian_apply_gate(v, euclid_grad, euclid_grad_derivative, x, parity: bool = False):
    if parity:
        return _by_blocks(riemannian_hessian_apply, v, euclid_grad, euclid_grad_derivative, x)
    return riemannian_hessian_apply(v, euclid_grad, euclid_grad_derivative, x)


def random_unitary(m: int, rng: np.random.Generator):
    """QR of a complex Gaussian with R's diagonal phases removed (Haar);
    same draw order as reference manifold.py:166-172 so seeds reproduce."""
    z = rng.normal(size=(m, m)) + 1j * rng.normal(size=(m, m))
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return np.ascontiguousarray(q * ph)
