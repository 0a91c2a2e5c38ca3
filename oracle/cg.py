"""Pinned Jacobi-preconditioned CG for the implicit substep -- TEST INFRASTRUCTURE.

The reference solves (M + a B[C]) x = M rhs with SuperLU (``dgsem.py:503-533``)
and has no CG; the north star asks for CG with identical iteration counts, so
this module *defines* the iteration the CUDA path reproduces:

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


def pcg(A, diag, b, x0, rtol=1e-14, maxit=1000):
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
