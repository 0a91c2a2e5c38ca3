"""Collocation node sets and quadrature weights (host-side precompute).

Same API as the reference's ``collocation.py`` (``make_nodes`` ``:110-147``,
``gauss_legendre`` ``:150-160``, ``gauss_lobatto`` ``:163-167``,
``lagrange_matrix`` ``:170-180``, weight matrices ``:190-217``).  These are
setup-time tables of at most 16x16 entries that are uploaded once; the
roots are found by Newton's method from Chebyshev-type initial guesses.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Literal

import numpy as np

NodeKind = Literal["radau_right", "lobatto", "equidistant"]


def _legendre_all(n: int, x: float):
    """P_n, P_n', P_{n-1}, P_{n-1}' at x."""
    p_prev, p = 1.0, x
    d_prev, d = 0.0, 1.0
    if n == 0:
        return 1.0, 0.0, 0.0, 0.0
    for k in range(1, n):
        p_prev, p = p, ((2 * k + 1) * x * p - k * p_prev) / (k + 1)
        d_prev, d = d, d_prev + (2 * k + 1) * p_prev
    return p, d, p_prev, d_prev


def _newton(fun, x0, tol=1e-16, maxit=100):
    x = float(x0)
    for _ in range(maxit):
        f, df = fun(x)
        if df == 0.0:
            break
        step = f / df
        x -= step
        if abs(step) <= tol * max(1.0, abs(x)):
            break
    return x


@dataclass(frozen=True)
class CollocationRule:
    """A node family on (0, 1] with tau_M = 1 (``collocation.py:83-99``)."""
    kind: str
    M: int
    tau: np.ndarray
    includes_left: bool

    def __post_init__(self):
        if len(self.tau) != self.M:
            raise ValueError("node count mismatch")
        if not np.all(np.diff(self.tau) > 0):
            raise ValueError("nodes must be strictly increasing")
        if abs(self.tau[-1] - 1.0) > 1e-14:
            raise ValueError("last node must be 1")


@dataclass(frozen=True)
class QuadratureWeights:
    w_nn: np.ndarray
    w_0n: np.ndarray


def make_nodes(kind: NodeKind, M: int) -> CollocationRule:
    if M < 1:
        raise ValueError("M must be positive")
    if kind == "radau_right":
        if M == 1:
            return CollocationRule(kind, 1, np.array([1.0]), False)

        def f(x):
            a, da, b, db = _legendre_all(M, x)
            return a - b, da - db
        # right-Radau points ~ cos(2 pi j / (2M - 1)), j = 1..M-1
        xs = sorted(_newton(f, math.cos(2.0 * math.pi * j / (2 * M - 1))) for j in range(1, M))
        return CollocationRule(kind, M, np.array([(x + 1.0) / 2.0 for x in xs] + [1.0]), False)
    if kind == "lobatto":
        if M < 2:
            raise ValueError("lobatto needs M >= 2")
        n = M - 1

        def f(x):
            p, dp, _, _ = _legendre_all(n, x)
            return dp, (2.0 * x * dp - n * (n + 1) * p) / (1.0 - x * x)
        xs = sorted(_newton(f, -math.cos(math.pi * j / n)) for j in range(1, n))
        return CollocationRule(kind, M, np.array([0.0] + [(x + 1.0) / 2.0 for x in xs] + [1.0]), True)
    if kind == "equidistant":
        return CollocationRule(kind, M, np.arange(1, M + 1) / M, False)
    raise ValueError(f"unknown node kind {kind!r}")


def gauss_legendre(n: int):
    return np.polynomial.legendre.leggauss(n)


def gauss_lobatto(n: int):
    x = 2.0 * make_nodes("lobatto", n).tau - 1.0
    w = np.array([2.0 / (n * (n - 1) * _legendre_all(n - 1, xi)[0] ** 2) for xi in x])
    return x, w


def lagrange_matrix(src, dst) -> np.ndarray:
    src = np.asarray(src, dtype=float)
    dst = np.asarray(dst, dtype=float)
    A = np.ones((len(dst), len(src)))
    for j, sj in enumerate(src):
        for k, sk in enumerate(src):
            if k != j:
                A[:, j] *= (dst - sk) / (sj - sk)
    return A


def compute_nn_weights(rule: CollocationRule) -> np.ndarray:
    M = rule.M
    gx, gw = gauss_legendre(M + 2)
    edges = np.concatenate([[0.0], rule.tau])
    w = np.zeros((M, M))
    for m in range(M):
        a, b = edges[m], edges[m + 1]
        if b > a:
            pts = 0.5 * (b - a) * gx + 0.5 * (a + b)
            w[m] = 0.5 * (b - a) * gw @ lagrange_matrix(rule.tau, pts)
    return w


def compute_0n_weights(w_nn) -> np.ndarray:
    return np.cumsum(np.asarray(w_nn, dtype=float), axis=0)


def make_weights(rule: CollocationRule) -> QuadratureWeights:
    w = compute_nn_weights(rule)
    return QuadratureWeights(w, compute_0n_weights(w))
