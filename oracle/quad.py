"""Collocation and element quadrature tables (oracle restatement).

Restates ``collocation.py`` of the reference: Radau-right / Lobatto /
equidistant node sets (``collocation.py:110-147``), Gauss-Legendre and
Gauss-Lobatto-Legendre rules (``:150-167``), Lagrange evaluation matrices
(``:170-180``) and the node-to-node / zero-to-node weight matrices
(``:190-217``); plus the barycentric derivative matrix and the delta(P)
time-step normaliser of ``dgsem.py:33-69``.

Roots are found with a different method from the reference (companion-matrix
eigenvalues of the Legendre series, then Newton polish in the Legendre
recurrence), so agreement with the reference's golden tables is a genuine
cross-check rather than a copy.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as L


def _leg(n, x):
    """(P_n(x), P_n'(x)) by the three-term recurrence, x array."""
    x = np.asarray(x, dtype=float)
    p0 = np.ones_like(x)
    if n == 0:
        return p0, np.zeros_like(x)
    p1 = x.copy()
    d0, d1 = np.zeros_like(x), np.ones_like(x)
    for k in range(1, n):
        p0, p1 = p1, ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
        d0, d1 = d1, d0 + (2 * k + 1) * p0
    return p1, d1


def _polish(fun, x, iters=6):
    for _ in range(iters):
        f, d = fun(x)
        step = np.where(d != 0.0, f / np.where(d != 0.0, d, 1.0), 0.0)
        x = x - step
        if np.all(np.abs(step) < 1e-16):
            break
    return x


def _series_roots(coef):
    r = L.legroots(coef)
    return np.sort(np.real(r))


def radau_right(M: int) -> np.ndarray:
    """Nodes on (0,1] of the right Radau rule (roots of P_M - P_{M-1});
    restates ``collocation.py:119-131``."""
    if M == 1:
        return np.array([1.0])
    c = np.zeros(M + 1)
    c[M] = 1.0
    c[M - 1] = -1.0
    x = _series_roots(c)
    x = x[x < 1.0 - 1e-8]

    def fun(z):
        a, da = _leg(M, z)
        b, db = _leg(M - 1, z)
        return a - b, da - db

    x = _polish(fun, x)
    return np.concatenate([(x + 1.0) / 2.0, [1.0]])


def lobatto(M: int) -> np.ndarray:
    """Lobatto nodes on [0,1]; restates ``collocation.py:132-143``."""
    if M < 2:
        raise ValueError("lobatto needs M >= 2")
    n = M - 1
    if n == 1:
        return np.array([0.0, 1.0])
    c = np.zeros(n + 1)
    c[n] = 1.0
    x = _series_roots(L.legder(c))

    def fun(z):
        # derivative of P_n and its derivative via the Legendre ODE
        p, dp = _leg(n, z)
        d2 = (2.0 * z * dp - n * (n + 1) * p) / (1.0 - z * z)
        return dp, d2

    x = _polish(fun, x)
    return np.concatenate([[0.0], (x + 1.0) / 2.0, [1.0]])


def make_tau(kind: str, M: int) -> np.ndarray:
    if kind == "radau_right":
        return radau_right(M)
    if kind == "lobatto":
        return lobatto(M)
    if kind == "equidistant":
        return np.arange(1, M + 1) / M
    raise ValueError(kind)


def gauss_legendre(n: int):
    """Gauss-Legendre rule on [-1,1]; restates ``collocation.py:150-160``."""
    x, w = L.leggauss(n)
    return x, w


def gll(n: int):
    """Gauss-Lobatto-Legendre nodes/weights (n points) on [-1,1];
    restates ``collocation.py:163-167``."""
    x = 2.0 * lobatto(n) - 1.0
    p, _ = _leg(n - 1, x)
    w = 2.0 / (n * (n - 1) * p * p)
    return x, w


def lagrange(src, dst) -> np.ndarray:
    """A[i,j] = ell_j(dst_i) on src nodes; restates ``collocation.py:170-180``."""
    src = np.asarray(src, dtype=float)
    dst = np.asarray(dst, dtype=float)
    n = len(src)
    A = np.ones((len(dst), n))
    for j in range(n):
        for k in range(n):
            if k != j:
                A[:, j] *= (dst - src[k]) / (src[j] - src[k])
    return A


def weights_nn(tau) -> np.ndarray:
    """w_nn[m,i] = int_{tau_{m-1}}^{tau_m} ell_i; restates ``collocation.py:190-207``."""
    tau = np.asarray(tau, dtype=float)
    M = len(tau)
    gx, gw = gauss_legendre(M + 2)
    edges = np.concatenate([[0.0], tau])
    w = np.zeros((M, M))
    for m in range(M):
        a, b = edges[m], edges[m + 1]
        if b == a:
            continue
        pts = 0.5 * (b - a) * gx + 0.5 * (a + b)
        w[m] = 0.5 * (b - a) * (gw @ lagrange(tau, pts))
    return w


def weights_0n(w_nn) -> np.ndarray:
    """Cumulative rows; restates ``collocation.py:210-212``."""
    return np.cumsum(np.asarray(w_nn, dtype=float), axis=0)


def diff_matrix(x) -> np.ndarray:
    """Barycentric collocation derivative D[i,j] = ell_j'(x_i), diagonal as
    negative row sum; restates ``dgsem.py:33-43``."""
    x = np.asarray(x, dtype=float)
    n = len(x)
    diff = x[:, None] - x[None, :]
    np.fill_diagonal(diff, 1.0)
    lam = 1.0 / np.prod(diff, axis=1)
    D = (lam[None, :] / lam[:, None]) / diff
    np.fill_diagonal(D, 0.0)
    D[np.arange(n), np.arange(n)] = -D.sum(axis=1)
    return D


def delta_of_degree(P: int) -> float:
    """Spectral radius of -D with inflow row/col removed; ``dgsem.py:46-59``."""
    x, _ = gll(P + 1)
    A = -diff_matrix(x)[1:, 1:]
    return float(np.max(np.abs(np.linalg.eigvals(A))))


def dt_from_cfl(cfl, dx_elem, lam_max, P):
    """``dgsem.py:67-69``."""
    return cfl * dx_elem / (2.0 * delta_of_degree(P) * lam_max)
