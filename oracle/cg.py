"""Pinned Jacobi-preconditioned CG for the implicit substep -- TEST INFRASTRUCTURE.

The reference solves (M + a B[C]) x = M rhs with SuperLU (``dgsem.py:503-533``)
and has no CG; the north star asks for CG with identical iteration counts, so
this module *defines* the iteration the CUDA path reproduces.  The pinned
iteration is ``pcg`` = the Chronopoulos-Gear form (``pcg_cg1``): the
Hestenes-Stiefel Krylov iterates with one fused reduction per iteration;
``pcg_hs`` keeps the two-reduction textbook form (same iteration counts on
every BASELINE solve, checked in tests/test_oracle_golden.py).  Common pins:

* operator A x = M x - a M apply_diffusion(C, x)   (= (M + a B[C]) x, SPD for C >= 0)
* right-hand side b = M rhs, initial guess x0 = rhs
* Jacobi preconditioner z = r / diag(M + a B[C])
* Hestenes-Stiefel recurrences, recursive residual
* stop at the first k with ||r_k||_2 <= rtol ||b||_2 (checked before each
  iteration, so k = 0 is possible); k > maxit -> failure (returns it = -1)

Returns (x, iterations, margin) with margin = ||r_k|| / (rtol ||b||) at exit,
which makes any +-1 iteration flip against the GPU diagnosable.
"""
import numpy as np


def pcg_hs(A, diag, b, x0, rtol=1e-14, maxit=1000):
    x = x0.copy()
    r = b - A(x)
    z = r / diag
    p = z.copy()
    rz = float(r @ z)
    rr = float(r @ r)
    thr = rtol * rtol * float(b @ b)
    k = 0
    while rr > thr:
        if k >= maxit:
            return x, -1, np.sqrt(rr / thr)
        Ap = A(p)
        alpha = rz / float(p @ Ap)
        x += alpha * p
        r -= alpha * Ap
        z = r / diag
        rz_new = float(r @ z)
        rr = float(r @ r)
        p = z + (rz_new / rz) * p
        rz = rz_new
        k += 1
    return x, k, float(np.sqrt(rr / thr)) if thr > 0 else 0.0


def pcg_cg1(A, diag, b, x0, rtol=1e-14, maxit=1000):
    """Chronopoulos-Gear Jacobi-PCG: the same Krylov iterates as ``pcg`` in
    exact arithmetic with ONE fused reduction per iteration,
    (gamma, delta, rho) = ((r,u), (w,u), (r,r)), u = D^-1 r, w = A u.
    Same pins: x0 = rhs, recursive residual, stop at the first k with
    rho_k <= rtol^2 (b,b).  Returns (x, iterations, margin)."""
    x = x0.copy()
    r = b - A(x)
    u = r / diag
    w = A(u)
    gamma, delta, rho = float(r @ u), float(w @ u), float(r @ r)
    thr = rtol * rtol * float(b @ b)
    p, s = u.copy(), w.copy()
    alpha = gamma / delta
    rgamma, ralpha = 1.0 / gamma, 1.0 / alpha
    k = 0
    while rho > thr:
        if k >= maxit:
            return x, -1, np.sqrt(rho / thr)
        x += alpha * p
        r -= alpha * s
        u = r / diag
        w = A(u)
        g_new, delta, rho = float(r @ u), float(w @ u), float(r @ r)
        k += 1
        if rho <= thr:
            break
        beta = g_new * rgamma
        alpha = g_new / (delta - beta * (g_new * ralpha))
        ralpha = 1.0 / alpha
        p = u + beta * p
        s = w + beta * s
        gamma = g_new
        rgamma = 1.0 / gamma
    return x, k, float(np.sqrt(rho / thr)) if thr > 0 else 0.0


pcg = pcg_cg1
