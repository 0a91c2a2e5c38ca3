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


def element_block_preconditioner(Amat, nc, ne, p1):
    """Element-block Jacobi: y = inv(A_ee) v per element e, A_ee the
    (nc (P+1))^2 diagonal block of the assembled M + a B[C] with rows/cols
    ordered (field, node); y_r = sum_j inv(A_ee)[r, j] v_j."""
    A = Amat.tocsr()
    blocks = []
    for e in range(ne):
        ids = np.concatenate([(c * ne + e) * p1 + np.arange(p1) for c in range(nc)])
        blocks.append((ids, np.linalg.inv(A[ids][:, ids].toarray())))

    def prec(v):
        out = np.empty_like(v)
        for ids, Bi in blocks:
            out[ids] = Bi @ v[ids]
        return out
    return prec


RESTART_ETA = 1e-10


def bicgstab(A, prec, b, x0, rtol=1e-14, maxit=1000):
    """Pinned right-preconditioned BiCGStab for the NON-symmetric
    implicit systems of the 1-D CNS problem (matrix-valued SI coefficient
    (dt_m/2) A_c(u_b)^2 + A_d(u_b), ``dgsem.py:356-396``; the reference
    factorises them with splu, ``dgsem.py:503-533``).  The CUDA kernel
    (``csrc/cns1d.cu``) reproduces this iteration:

    * A x = M x - a M apply_diffusion(C, x), b = M rhs, x0 = rhs,
      y = K^-1 p, z = K^-1 s with K the element-block diagonal of M + a B[C]
      (``element_block_preconditioner``; point Jacobi stagnates at the
      reference's own CFL-256 acoustic test, cond ~ 1e10)
    * shadow residual r^ = r0; rho_0 = (r^, r0)
    * per iteration k: [k > 0: beta = (rho_k / rho_{k-1}) (alpha / omega),
      p = r + beta (p - omega v)]; v = A y; alpha = rho / (r^, v);
      s = r - alpha v; t = A z; omega = (t, s) / (t, t) (0 if (t, t) == 0);
      x = x + alpha y + omega z; r = s - omega t;
      rho_{k+1} = (r^, s) - omega (r^, t)   (== (r^, r), fused reduction)
    * restart (r^ = p = r, rho = (r, r), same k) when |rho| <= 1e-10 |r^| |r|
      after the p update: the shadow residual has become orthogonal to r
      (Lanczos breakdown; without it the CFL-256 acoustic solves stagnate
      in ~1 of 6 runs perturbed at 1e-14, with it all converge)
    * stop at the first k with (r_k, r_k) <= rtol^2 (b, b) (checked before
      each iteration); k > maxit or a non-finite (r_k, r_k) (breakdown,
      overflow) -> failure (it = -1).

    Returns (x, iterations, margin) like ``pcg``."""
    x = x0.copy()
    r = b - A(x)
    rh = r.copy()
    rr = float(r @ r)
    rho = rr
    rhrh = rr                  # (r^, r^)
    thr = rtol * rtol * float(b @ b)
    p = r.copy()
    v = np.zeros_like(r)
    alpha = omega = 1.0
    rho_new = rho
    k = 0
    fresh = True
    while rr > thr or not np.isfinite(rr):
        if k >= maxit or not np.isfinite(rr):   # breakdown / overflow is a failure
            return x, -1, np.sqrt(rr / thr)
        if not fresh:
            beta = (rho_new / rho) * (alpha / omega)
            p = r + beta * (p - omega * v)
            rho = rho_new
        fresh = False
        if abs(rho) <= RESTART_ETA * np.sqrt(rhrh * rr):   # Lanczos breakdown: r^ _|_ r
            rh = r.copy()
            rhrh = rr
            rho = rr
            p = r.copy()
        y = prec(p)
        v = A(y)
        alpha = rho / float(rh @ v)
        s = r - alpha * v
        z = prec(s)
        t = A(z)
        tt = float(t @ t)
        omega = float(t @ s) / tt if tt != 0.0 else 0.0
        x = x + alpha * y + omega * z
        r = s - omega * t
        rho_new = float(rh @ s) - omega * float(rh @ t)
        rr = float(r @ r)
        k += 1
    return x, k, float(np.sqrt(rr / thr)) if thr > 0 else 0.0
