"""1-D nodal DG-SEM operator (oracle restatement of ``dgsem.py`` + ``problems.py``).

States are flat float64 vectors in the reference layout (ncomp, n_elem, P+1)
(``dgsem.py:12-13``).  Coefficients use the reference's four kinds
(``dgsem.py:229-239``): None, python float ("const"), (n_elem, P+1) array
("scalar") and (n_elem, P+1, nc, nc) array ("matrix").

The implicit solve offers the reference's algorithm (mode "lu": sparse LU of
M + a B[C] with a per-shift cache and defect iterations, ``dgsem.py:492-533``)
and the pinned Jacobi-PCG (mode "pcg", ``oracle/cg.py``) that the CUDA path
reproduces.  TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from . import quad
from .cg import bicgstab, element_block_preconditioner, pcg


class SolverError(RuntimeError):
    """Mirror of ``dgsem.SolverError`` (``dgsem.py:29-30``)."""


# ----------------------------------------------------------------- physics
class ConvDiff:
    """u_t + v u_x = nu u_xx (``problems.py:25-52``)."""
    ncomp = 1
    linear = True

    def __init__(self, speed=1.0, nu=0.0, boundary=None):
        self.v, self.nu = float(speed), float(nu)
        self.boundary = boundary

    def flux(self, u):
        return self.v * u

    def speed(self, u):
        return np.full(u.shape[1:], abs(self.v))

    def jac(self, u3):
        return self.v

    def dcoef(self, u3):
        return self.nu if self.nu > 0 else None


class Burgers:
    """u_t + (u^2/2)_x = nu u_xx (``problems.py:55-82``)."""
    ncomp = 1
    linear = False

    def __init__(self, nu=0.0, boundary=None, source=None):
        self.nu = float(nu)
        self.boundary = boundary   # t -> (left state, right state), problems.py:66
        self.source = source       # (x, t, u3) -> values, problems.py:61-65

    def flux(self, u):
        return 0.5 * u * u

    def speed(self, u):
        return np.abs(u[0])

    def jac(self, u3):
        return np.array(u3[0])

    def dcoef(self, u3):
        return self.nu if self.nu > 0 else None


class CNS1D:
    """1-D compressible Navier-Stokes, conservative (rho, rho v, rho E)
    (``problems.py:160-240``)."""
    ncomp = 3
    linear = False

    def __init__(self, gamma=1.4, R_gas=287.28, eta=0.0, Pr=0.75):
        self.g, self.R, self.eta, self.Pr = float(gamma), float(R_gas), float(eta), float(Pr)

    def _prim(self, u):
        rho = u[0]
        v = u[1] / rho
        p = (self.g - 1.0) * (u[2] - 0.5 * u[1] * v)
        return rho, v, p

    def flux(self, u):
        rho, v, p = self._prim(u)
        return np.stack([u[1], u[1] * v + p, v * (u[2] + p)])

    def speed(self, u):
        rho, v, p = self._prim(u)
        return np.abs(v) + np.sqrt(self.g * p / rho)

    def jac(self, u3):
        g = self.g
        rho, v, p = self._prim(u3)
        H = (u3[2] + p) / rho
        A = np.zeros(v.shape + (3, 3))
        A[..., 0, 1] = 1.0
        A[..., 1, 0] = 0.5 * (g - 3.0) * v * v
        A[..., 1, 1] = (3.0 - g) * v
        A[..., 1, 2] = g - 1.0
        A[..., 2, 0] = (0.5 * (g - 1.0) * v * v - H) * v
        A[..., 2, 1] = H - (g - 1.0) * v * v
        A[..., 2, 2] = g * v
        return A

    def dcoef(self, u3):
        if self.eta <= 0:
            return None
        rho, v, p = self._prim(u3)
        E = u3[2] / rho
        nu = self.eta / rho
        gk = self.g * nu / self.Pr
        mu = 4.0 / 3.0 * nu
        A = np.zeros(v.shape + (3, 3))
        A[..., 1, 0] = -mu * v
        A[..., 1, 1] = mu
        A[..., 2, 0] = -(mu - gk) * v * v - gk * E
        A[..., 2, 1] = (mu - gk) * v
        A[..., 2, 2] = gk
        return A


def kind_of(c):
    """``dgsem.py:229-239``."""
    if c is None:
        return "none"
    if np.isscalar(c):
        return "const"
    nd = np.ndim(c)
    if nd == 2:
        return "scalar"
    if nd == 4:
        return "matrix"
    raise ValueError("bad coefficient")


# ---------------------------------------------------------------- operator
class Op1D:
    """Oracle DG operator on a uniform 1-D mesh (``dgsem.py:117-151``),
    periodic or Dirichlet faces (``:179-201``): with ``bc="dirichlet"`` the
    outer faces take the problem's boundary states g(t) on the outside, the
    one-sided interior flux q and coefficient, and face weight 1 in the
    adjoint lift; the diffusion operator is then affine in u."""

    def __init__(self, x_left, x_right, n_elem, degree, problem, penalty=2.0,
                 solver="pcg", rtol=1e-14, maxit=1000, av=None, cg_log=None, bc="periodic"):
        self.xl, self.xr = float(x_left), float(x_right)
        self.ne, self.P = int(n_elem), int(degree)
        self.p1 = self.P + 1
        self.dx = (self.xr - self.xl) / self.ne
        self.prob = problem
        self.nc = problem.ncomp
        self.xi, self.w = quad.gll(self.p1)
        self.D = quad.diff_matrix(self.xi)
        self.mass = 0.5 * self.dx * self.w               # dgsem.py:135
        self.mu0 = penalty * self.p1 ** 2 / self.dx       # dgsem.py:137
        self.n = self.nc * self.ne * self.p1
        self.mflat = np.tile(self.mass, self.nc * self.ne)
        self.solver, self.rtol, self.maxit = solver, rtol, maxit
        self.av = av                                      # (kappa_s, c_s) or None
        self.nu_art = None
        self.cg_log = [] if cg_log is None else cg_log    # (iters, |r|/(rtol|b|)), call order
        self._lu = {}
        self._last_dt = None
        V = np.stack([quad._leg(k, self.xi)[0] for k in range(self.p1)], axis=1)
        self._vinv = np.linalg.inv(V)
        if bc not in ("periodic", "dirichlet"):
            raise ValueError(bc)
        if bc == "dirichlet" and getattr(problem, "boundary", None) is None:
            raise ValueError("dirichlet mesh needs a problem with boundary_state(t)")   # dgsem.py:150-151
        self.bc = bc

    def _bstate(self, t):
        gl, gr = self.prob.boundary(t)
        return np.asarray(gl, dtype=float).reshape(self.nc), np.asarray(gr, dtype=float).reshape(self.nc)

    # layout -------------------------------------------------------------
    def u3(self, u):
        return np.asarray(u).reshape(self.nc, self.ne, self.p1)

    @property
    def x_nodes(self):
        e = self.xl + self.dx * np.arange(self.ne)
        return e[:, None] + 0.5 * self.dx * (self.xi + 1.0)[None, :]

    # traces: periodic neighbours (dgsem.py:179-194)
    @staticmethod
    def _left_nb(a):   # value from element e-1 (wrapped)
        return np.roll(a, 1, axis=-2)

    @staticmethod
    def _right_nb(a):  # value from element e+1 (wrapped)
        return np.roll(a, -1, axis=-2)

    # convection (dgsem.py:205-225) --------------------------------------
    def apply_convection(self, u, t=0.0):
        u3 = self.u3(u)
        f = self.prob.flux(u3)
        out = np.einsum("ki,k,cek->cei", self.D, self.w, f)
        # face e+1/2 between element e (minus side, node P) and e+1 (plus, node 0)
        um = u3[:, :, -1]
        up = self._right_nb(u3)[:, :, 0]
        lam = np.maximum(self.prob.speed(um[:, :, None])[..., 0],
                         self.prob.speed(up[:, :, None])[..., 0])
        fh = 0.5 * (self.prob.flux(um[:, :, None])[..., 0] + self.prob.flux(up[:, :, None])[..., 0]) \
            - 0.5 * lam[None] * (up - um)
        if self.bc == "periodic":
            out[:, :, -1] -= fh
            out[:, :, 0] += np.roll(fh, 1, axis=-1)
            return (out / self.mass).reshape(-1)
        # Dirichlet (dgsem.py:212-216): faces 0..ne, outside states g_l(t), g_r(t)
        gl, gr = self._bstate(t)
        um_f = np.concatenate([gl[:, None], u3[:, :, -1]], axis=1)
        up_f = np.concatenate([u3[:, :, 0], gr[:, None]], axis=1)
        lam = np.maximum(self.prob.speed(um_f[:, :, None])[..., 0], self.prob.speed(up_f[:, :, None])[..., 0])
        fh = 0.5 * (self.prob.flux(um_f[:, :, None])[..., 0] + self.prob.flux(up_f[:, :, None])[..., 0]) \
            - 0.5 * lam[None] * (up_f - um_f)
        out[:, :, -1] -= fh[:, 1:]
        out[:, :, 0] += fh[:, :-1]
        return (out / self.mass).reshape(-1)

    # diffusion (dgsem.py:251-309) ---------------------------------------
    def _coef_field(self, c):
        k = kind_of(c)
        if k == "const":
            return np.full((self.ne, self.p1), float(c)), k
        return np.asarray(c, dtype=float), k

    def apply_diffusion(self, coeff, u, t=0.0):
        k = kind_of(coeff)
        if k == "none" or (k == "const" and coeff == 0.0):
            return np.zeros(self.n)
        u3 = self.u3(u)
        C, k = self._coef_field(coeff)
        s = 2.0 / self.dx
        g = s * np.einsum("ij,cej->cei", self.D, u3)
        if k == "matrix":
            q = np.einsum("epab,bep->aep", C, g)
        else:
            q = C[None] * g
        B = np.einsum("ki,k,cek->cei", self.D, self.w, q)
        # face e+1/2: minus = element e node P, plus = element e+1 node 0
        um, up = u3[:, :, -1], self._right_nb(u3)[:, :, 0]
        qm, qp = q[:, :, -1], self._right_nb(q)[:, :, 0]
        jump = um - up
        if k == "matrix":
            Cm, Cp = C[:, -1], np.roll(C, -1, axis=0)[:, 0]           # (ne, nc, nc)
            pen = self.mu0 * np.einsum("eab,be->ae", 0.5 * (Cm + Cp), jump)
            lm = 0.5 * np.einsum("eab,be->ae", Cm, jump)
            lp = 0.5 * np.einsum("eab,be->ae", Cp, jump)
        else:
            Cm, Cp = C[:, -1], np.roll(C, -1, axis=0)[:, 0]
            pen = self.mu0 * 0.5 * (Cm + Cp)[None] * jump
            lm = 0.5 * Cm[None] * jump
            lp = 0.5 * Cp[None] * jump
        G = pen - 0.5 * (qm + qp)
        if self.bc == "periodic":
            B[:, :, -1] += G
            B[:, :, 0] -= np.roll(G, 1, axis=-1)
            # adjoint lift with each side's own coefficient (dgsem.py:296-308)
            B -= s * lm[:, :, None] * self.D[-1][None, None, :]
            B -= s * np.roll(lp, 1, axis=-1)[:, :, None] * self.D[0][None, None, :]
            return (-B / self.mass).reshape(-1)
        # Dirichlet (dgsem.py:282-308): faces 0..ne; outside states g(t), q and C
        # one-sided at the outer faces, adjoint-lift weight 1 there
        gl, gr = self._bstate(t)
        uf_m = np.concatenate([gl[:, None], u3[:, :, -1]], axis=1)
        uf_p = np.concatenate([u3[:, :, 0], gr[:, None]], axis=1)
        qf_m = np.concatenate([q[:, :1, 0], q[:, :, -1]], axis=1)
        qf_p = np.concatenate([q[:, :, 0], q[:, -1:, -1]], axis=1)
        cf_m = np.concatenate([C[:1, 0], C[:, -1]])
        cf_p = np.concatenate([C[:, 0], C[-1:, -1]])
        wf = np.full(self.ne + 1, 0.5)
        wf[0] = wf[-1] = 1.0
        jump = uf_m - uf_p
        if k == "matrix":   # (nf, nc, nc) face coefficients acting on the jump vectors
            pen = self.mu0 * np.einsum("fab,bf->af", 0.5 * (cf_m + cf_p), jump)
            lift_m = np.einsum("f,fab,bf->af", wf, cf_m, jump)
            lift_p = np.einsum("f,fab,bf->af", wf, cf_p, jump)
        else:
            pen = self.mu0 * (0.5 * (cf_m + cf_p))[None] * jump
            lift_m = (wf * cf_m)[None] * jump
            lift_p = (wf * cf_p)[None] * jump
        Gf = -0.5 * (qf_m + qf_p) + pen
        B[:, :, -1] += Gf[:, 1:]
        B[:, :, 0] -= Gf[:, :-1]
        B -= s * lift_m[:, 1:, None] * self.D[-1][None, None, :]
        B -= s * lift_p[:, :-1, None] * self.D[0][None, None, :]
        return (-B / self.mass).reshape(-1)

    # rhs (dgsem.py:313-352) ---------------------------------------------
    def physical_coeff(self, u3):
        base = self.prob.dcoef(u3)
        eps = self.nu_art
        if eps is None:
            return base
        k = kind_of(base)
        if k == "none":
            return eps[:, None] * np.ones((1, self.p1))
        if k == "const":
            return float(base) + eps[:, None] * np.ones((1, self.p1))
        if k == "scalar":
            return np.asarray(base) + eps[:, None]
        return np.asarray(base) + eps[:, None, None, None] * np.eye(self.nc)

    def eval_rhs(self, u, t=0.0):
        out = self.apply_convection(u, t).copy()
        c = self.physical_coeff(self.u3(u))
        if kind_of(c) != "none":
            out = out + self.apply_diffusion(c, u, t)
        src = getattr(self.prob, "source", None)   # dgsem.py:343-347
        if src is not None:
            vals = src(self.x_nodes, t, self.u3(u))
            if vals is not None:
                out = out + (np.asarray(vals) + np.zeros((self.nc, 1, 1))).reshape(-1)
        bad = ~np.isfinite(out.reshape(self.nc, self.ne, self.p1))
        if bad.any():
            e = int(np.nonzero(bad.any(axis=(0, 2)))[0][0])
            raise SolverError(f"non-finite right-hand side in element {e}")
        return out

    # SI coefficient (dgsem.py:356-396) ----------------------------------
    def modified_coeff(self, u_b, dt_m, scheme="si2"):
        u3 = self.u3(u_b)
        phys = self.physical_coeff(u3)
        if scheme == "euler":
            return phys
        J = self.prob.jac(u3)
        pk = kind_of(phys)
        if kind_of(J) == "matrix":
            c = 0.5 * dt_m * np.einsum("epij,epjk->epik", J, J)
            if pk == "none":
                return c
            if pk == "matrix":
                return c + phys
            fld = np.full((self.ne, self.p1), float(phys)) if pk == "const" else phys
            return c + fld[:, :, None, None] * np.eye(self.nc)
        half = 0.5 * dt_m * (float(J) ** 2 if np.isscalar(J) else np.asarray(J) ** 2)
        if pk == "none":
            c = half
        elif pk in ("const", "scalar"):
            c = half + (float(phys) if pk == "const" else phys)
        else:
            hf = np.full((self.ne, self.p1), float(half)) if np.isscalar(half) else half
            c = phys + hf[:, :, None, None] * np.eye(self.nc)
        return float(c) if np.isscalar(c) else c

    # SIP stiffness diagonal and assembly (dgsem.py:414-490) --------------
    def _cmat(self, coeff):
        k = kind_of(coeff)
        eye = np.eye(self.nc)
        if k == "const":
            return np.broadcast_to(float(coeff) * eye, (self.ne, self.p1, self.nc, self.nc)).copy()
        if k == "scalar":
            return np.asarray(coeff)[:, :, None, None] * eye
        if k == "matrix":
            return np.asarray(coeff)
        raise ValueError("cannot assemble a zero coefficient")

    def stiffness(self, coeff):
        """B[C] (no mass) as CSC, periodic; restates ``dgsem.py:414-490``
        (vectorised over faces instead of a per-face Python loop)."""
        C = self._cmat(coeff)
        ne, p1, nc = self.ne, self.p1, self.nc
        s = 2.0 / self.dx
        D, w = self.D, self.w
        gid = (np.arange(nc)[:, None, None] * ne + np.arange(ne)[None, :, None]) * p1 \
            + np.arange(p1)[None, None, :]
        V = s * np.einsum("ki,ekab,k,kj->eaibj", D, C, w, D)
        rows = [np.broadcast_to(gid.transpose(1, 0, 2)[:, :, :, None, None], V.shape).ravel()]
        cols = [np.broadcast_to(gid.transpose(1, 0, 2)[:, None, None, :, :], V.shape).ravel()]
        vals = [V.ravel()]
        # face between eL=e and eR=e+1: local ordering [a, eL node] + [a, eR node]
        eL = np.arange(ne) if self.bc == "periodic" else np.arange(ne - 1)
        eR = (eL + 1) % ne
        CL, CR = C[eL, -1], C[eR, 0]                     # (ne, nc, nc)
        npair = 2 * nc * p1
        J = np.zeros((nc, npair))
        for a in range(nc):
            J[a, a * p1 + p1 - 1] = 1.0
            J[a, nc * p1 + a * p1] = -1.0
        Q = np.zeros((len(eL), nc, npair))
        QT = np.zeros((len(eL), nc, npair))
        for b in range(nc):
            Q[:, :, b * p1:(b + 1) * p1] = 0.5 * s * CL[:, :, b, None] * D[-1][None, None, :]
            Q[:, :, nc * p1 + b * p1:nc * p1 + (b + 1) * p1] = 0.5 * s * CR[:, :, b, None] * D[0][None, None, :]
            QT[:, :, b * p1:(b + 1) * p1] = 0.5 * s * CL[:, b, :, None] * D[-1][None, None, :]
            QT[:, :, nc * p1 + b * p1:nc * p1 + (b + 1) * p1] = 0.5 * s * CR[:, b, :, None] * D[0][None, None, :]
        muC = self.mu0 * 0.5 * (CL + CR)
        blk = -(np.einsum("ai,eaj->eij", J, Q) + np.einsum("eai,aj->eij", QT, J)) \
            + np.einsum("ai,eab,bj->eij", J, muC, J)
        nfc = len(eL)
        ids = np.concatenate([gid[:, eL, :].transpose(1, 0, 2).reshape(nfc, -1),
                              gid[:, eR, :].transpose(1, 0, 2).reshape(nfc, -1)], axis=1)
        rows.append(np.repeat(ids, npair, axis=1).ravel())
        cols.append(np.tile(ids, (1, npair)).ravel())
        vals.append(blk.ravel())
        if self.bc == "dirichlet":   # outer faces, one-sided (dgsem.py:460-481)
            nh = nc * p1
            for e, Cb, drow, sgn, endpos in ((0, C[0, 0], D[0], -1.0, 0), (ne - 1, C[ne - 1, -1], D[-1], 1.0, p1 - 1)):
                Jb = np.zeros((nc, nh))
                Qb = np.zeros((nc, nh))
                QTb = np.zeros((nc, nh))
                for a in range(nc):
                    Jb[a, a * p1 + endpos] = sgn
                    for b2 in range(nc):
                        Qb[a, b2 * p1:(b2 + 1) * p1] = s * Cb[a, b2] * drow
                        QTb[a, b2 * p1:(b2 + 1) * p1] = s * Cb[b2, a] * drow
                blkb = -(Jb.T @ Qb + QTb.T @ Jb) + Jb.T @ (self.mu0 * Cb) @ Jb
                idb = gid[:, e, :].ravel()
                rows.append(np.repeat(idb, nh))
                cols.append(np.tile(idb, nh))
                vals.append(blkb.ravel())
        B = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n, self.n))
        return B.tocsc()

    def stiffness_diag(self, coeff):
        """diag(B[C]) for scalar/const coefficients, closed form of the
        assembly above; feeds the Jacobi preconditioner."""
        C, k = self._coef_field(coeff)
        if k == "matrix":
            return np.asarray(self.stiffness(coeff).diagonal())
        s = 2.0 / self.dx
        d = s * np.einsum("ki,k,ek->ei", self.D ** 2, self.w, C)
        Cm = C[:, -1]
        Cp = np.roll(C, -1, axis=0)[:, 0]
        muC = self.mu0 * 0.5 * (Cm + Cp)                # face e+1/2
        if self.bc == "periodic":
            d[:, -1] += muC - s * Cm * self.D[-1, -1]
            d[:, 0] += np.roll(muC + s * Cp * self.D[0, 0], 1)
        else:   # interior faces, then the outer faces with weight 1 (dgsem.py:460-481)
            d[:-1, -1] += (muC - s * Cm * self.D[-1, -1])[:-1]
            d[1:, 0] += (muC + s * Cp * self.D[0, 0])[:-1]
            d[0, 0] += self.mu0 * C[0, 0] + 2.0 * s * C[0, 0] * self.D[0, 0]
            d[-1, -1] += self.mu0 * C[-1, -1] - 2.0 * s * C[-1, -1] * self.D[-1, -1]
        return np.tile(d.reshape(-1), self.nc)

    # implicit solve (dgsem.py:503-533) ----------------------------------
    def implicit_solve(self, coeff, a, rhs, t=0.0):
        if a == 0.0:
            return rhs
        rhs = np.asarray(rhs)
        b = self.mflat * rhs.reshape(-1)
        if not b.any():
            return np.zeros_like(rhs)
        if self.solver == "lu":
            return self._solve_lu(coeff, a, b, t).reshape(rhs.shape)
        diag = self.mflat + a * self.stiffness_diag(coeff) if self.nc == 1 else None
        m = self.mflat
        if self.bc == "dirichlet":
            # affine SIP: D(x; t) = D_lin(x) + d_bc(t), d_bc = D(0; t).  Solve the
            # linear system (M + a B_lin) x = M rhs + a M d_bc (the solution of the
            # reference's defect iteration, dgsem.py:517-529)
            dbc = self.apply_diffusion(coeff, np.zeros(self.n), t)
            b = b + a * m * dbc

            def A(x):
                return m * x - a * m * (self.apply_diffusion(coeff, x, t) - dbc)
        else:
            def A(x):
                return m * x - a * m * self.apply_diffusion(coeff, x, t)

        if self.nc > 1:   # systems (1-D CNS): non-symmetric -> pinned element-block BiCGStab
            prec = element_block_preconditioner(sp.diags(self.mflat) + a * self.stiffness(coeff), self.nc,
                                                self.ne, self.p1)
            x, it, margin = bicgstab(A, prec, b, rhs.reshape(-1).copy(), self.rtol, self.maxit)
        else:
            x, it, margin = pcg(A, diag, b, rhs.reshape(-1).copy(), self.rtol, self.maxit)
        if it < 0:
            raise SolverError("implicit CG solve did not converge")
        self.cg_log.append((it, margin))
        return x.reshape(rhs.shape)

    def _factor(self, coeff, a):
        return splu((sp.diags(self.mflat) + a * self.stiffness(coeff)).tocsc())

    def _solve_lu(self, coeff, a, b, t):
        ent = self._lu.get(a)
        if ent is None:
            ent = (self._factor(coeff, a), coeff)
            self._lu[a] = ent
        x = ent[0].solve(b)
        same = (np.isscalar(coeff) and np.isscalar(ent[1]) and float(coeff) == float(ent[1])) \
            or coeff is ent[1]
        if same and self.bc == "periodic":
            return x
        bn = np.linalg.norm(b)
        m = self.mflat
        refreshed = False
        for it in range(40):
            r = b - m * x + a * m * self.apply_diffusion(coeff, x, t)
            if np.linalg.norm(r) <= 1e-12 * bn:
                return x
            if it >= 4 and not refreshed:
                ent = (self._factor(coeff, a), coeff)
                self._lu[a] = ent
                refreshed = True
            x = x + ent[0].solve(r)
        raise SolverError("implicit solve stalled after 40 iterations")

    # artificial viscosity + slab hook (dgsem.py:537-571) -----------------
    def persson_viscosity(self, u):
        if self.av is None:
            return np.zeros(self.ne)
        kap, cs = self.av
        P = self.P
        u3 = self.u3(u)
        modal = u3[0] @ self._vinv.T
        en = modal ** 2 * (2.0 / (2.0 * np.arange(self.p1) + 1.0))[None]
        tot = en.sum(axis=1)
        with np.errstate(divide="ignore", invalid="ignore"):
            sv = np.where(tot > 0.0, np.log10(np.maximum(en[:, -1], 1e-300) / tot), -np.inf)
        s0 = -4.0 * np.log10(P)
        lam_e = self.prob.speed(u3).max(axis=1)
        eps0 = cs * self.dx * lam_e / P
        ramp = np.where(sv < s0 - kap, 0.0,
                        np.where(sv > s0 + kap, 1.0, 0.5 * (1.0 + np.sin(0.5 * np.pi * (sv - s0) / kap))))
        return eps0 * ramp

    def begin_slab(self, u0, t0, dt):
        if self.av is not None:
            self.nu_art = self.persson_viscosity(u0)
        if dt != self._last_dt:
            self._lu.clear()
            self._last_dt = dt
