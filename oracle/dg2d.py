"""2-D tensor-product DG-SEM operators (oracle restatement) -- TEST INFRASTRUCTURE.

The reference is 1-D only; BASELINE configs 3-5 are 2-D Euler /
Navier-Stokes.  This module generalises the reference's 1-D operators by
tensor product on a uniform periodic Cartesian mesh with GLL collocation,
where the weak-form convection (``dgsem.py:205-225``) and the interior-penalty
diffusion with a scalar coefficient field (``dgsem.py:251-309``) are exactly
sums of the 1-D operators applied along x-lines and along y-lines (the
transverse quadrature weight cancels against the lumped mass).  A y-invariant
field with no y-flux therefore reproduces the 1-D reference, which
``tests/test_oracle2d.py`` checks against the reference's own goldens.

State layout: (ncomp, ney, nex, P+1 [y], P+1 [x]), C order, flattened.

Physics (documented departures from the reference):
* flux: 2-D compressible Euler in conservative variables (rho, rho u, rho v,
  rho E), ideal gas; Rusanov face flux with lambda = max(|v.n| + c) of the
  two traces (the 1-D rule ``dgsem.py:219`` with the normal speed);
* viscous term (configs 4-5): isotropic constant kinematic viscosity nu on
  all four conservative fields, discretised with the same SIP operator;
* semi-implicit coefficient: the reference's (dt_m/2) A_c^2 + A_d (3x3 /
  4x4 field, non-symmetric -> not CG-solvable) is replaced by
  the isotropic SPD scalar (dt_m/2) lambda(u_b)^2 + nu, lambda = |v| + c,
  shared by the four fields; the SDC fixed point (the collocation solution
  of the full f) is unchanged, only the stabilising implicit part differs.
"""
from __future__ import annotations

import numpy as np

from . import quad
from .cg import pcg


class Euler2D:
    ncomp = 4
    linear = False

    def __init__(self, gamma=1.4, nu=0.0):
        self.g, self.nu = float(gamma), float(nu)

    def prim(self, u):
        rho = u[0]
        vx = u[1] / rho
        vy = u[2] / rho
        p = (self.g - 1.0) * (u[3] - 0.5 * (u[1] * vx + u[2] * vy))
        return rho, vx, vy, p

    def flux(self, u, axis):
        rho, vx, vy, p = self.prim(u)
        vn = vx if axis == 0 else vy
        f = np.empty_like(u)
        f[0] = u[1 + axis]
        f[1] = u[1] * vn + (p if axis == 0 else 0.0)
        f[2] = u[2] * vn + (p if axis == 1 else 0.0)
        f[3] = vn * (u[3] + p)
        return f

    def speed(self, u, axis):
        rho, vx, vy, p = self.prim(u)
        vn = vx if axis == 0 else vy
        return np.abs(vn) + np.sqrt(self.g * p / rho)

    def max_speed(self, u):
        rho, vx, vy, p = self.prim(u)
        return np.sqrt(vx * vx + vy * vy) + np.sqrt(self.g * p / rho)


class NS2D(Euler2D):
    """2-D compressible Navier-Stokes in conservative variables: the Euler
    flux plus the physical viscous flux (Stokes stress with dynamic viscosity
    eta, Fourier heat flux with kappa = eta c_p / Pr), the 2-D generalisation
    of the reference's ``CompressibleFlow.diffusion_coeff`` (``problems.py:
    221-237``: nu = eta / rho, mu = 4/3 nu, gamma kappa = gamma nu / Pr, heat
    flux in terms of the specific internal energy, R cancels).

    F^x = (0, t_xx, t_xy, u t_xx + v t_xy + k rho e_x),
    F^y = (0, t_xy, t_yy, u t_xy + v t_yy + k rho e_y),  k = gamma nu / Pr,
    t_xx = nu (4/3 (m_x - u rho_x) - 2/3 (n_y - v rho_y)), t_yy likewise,
    t_xy = nu ((m_y - u rho_y) + (n_x - v rho_x)),
    rho e_. = E_. - E/rho rho_. - u (m_. - u rho_.) - v (n_. - v rho_.).
    With v = 0 and y-invariant data this is the reference's 1-D A_d u_x.

    The implicit (semi-implicit) part stays the isotropic SPD scalar
    (dt_m/2) lambda^2 + nu_b, nu_b = eta / rho max(4/3, gamma / Pr) (the
    spectral bound of the viscous matrices), shared by the four fields."""

    viscous = True

    def __init__(self, gamma=1.4, eta=0.0, prandtl=0.72):
        super().__init__(gamma, 0.0)
        self.eta, self.pr = float(eta), float(prandtl)

    def _p(self, u):
        rho = u[0]
        return rho, u[1] / rho, u[2] / rho, u[3] / rho, self.eta / rho

    def visc_flux(self, u, gx, gy):
        rho, vx, vy, Es, nu = self._p(u)
        k = self.g * nu / self.pr
        dxm, dym = gx[1] - vx * gx[0], gy[1] - vx * gy[0]   # rho u_x, rho u_y (velocity u)
        dxn, dyn = gx[2] - vy * gx[0], gy[2] - vy * gy[0]   # rho v_x, rho v_y
        txx = nu * ((4.0 / 3.0) * dxm - (2.0 / 3.0) * dyn)
        tyy = nu * ((4.0 / 3.0) * dyn - (2.0 / 3.0) * dxm)
        txy = nu * (dym + dxn)
        ex = gx[3] - Es * gx[0] - vx * dxm - vy * dxn
        ey = gy[3] - Es * gy[0] - vx * dym - vy * dyn
        z = np.zeros_like(rho)
        Fx = np.stack([z, txx, txy, vx * txx + vy * txy + k * ex])
        Fy = np.stack([z, txy, tyy, vx * txy + vy * tyy + k * ey])
        return Fx, Fy

    def apply_gnn(self, u, v, axis):
        """G_nn v: the normal-normal viscous block at state u applied to v
        (penalty and adjoint terms; the 1-D reference's A_d for axis 0)."""
        rho, vx, vy, Es, nu = self._p(u)
        k = self.g * nu / self.pr
        a = v[1] - vx * v[0]
        b = v[2] - vy * v[0]
        r1 = nu * ((4.0 / 3.0) * a if axis == 0 else a)
        r2 = nu * (b if axis == 0 else (4.0 / 3.0) * b)
        r3 = vx * r1 + vy * r2 + k * (v[3] - Es * v[0] - vx * a - vy * b)
        return np.stack([np.zeros_like(rho), r1, r2, r3])

    def nu_si(self, u):
        rho = u[0]
        return (self.eta / rho) * max(4.0 / 3.0, self.g / self.pr)


class Advection2D:
    """Scalar u_t + a.grad u = nu lap u (cross-dimension checks)."""
    ncomp = 1
    linear = True

    def __init__(self, ax=1.0, ay=0.0, nu=0.0):
        self.a, self.nu = (float(ax), float(ay)), float(nu)

    def flux(self, u, axis):
        return self.a[axis] * u

    def speed(self, u, axis):
        return np.full(u.shape[1:], abs(self.a[axis]))

    def max_speed(self, u):
        return np.full(u.shape[1:], np.hypot(*self.a))


class Burgers2D:
    """Scalar u_t + (u^2/2)_x = nu lap u (x-flux only): the 2-D embedding of
    the reference's Burgers problem (``problems.py:55-82``)."""
    ncomp = 1
    linear = False

    def __init__(self, nu=0.0):
        self.nu = float(nu)

    def flux(self, u, axis):
        return 0.5 * u * u if axis == 0 else np.zeros_like(u)

    def speed(self, u, axis):
        return np.abs(u[0]) if axis == 0 else np.zeros(u.shape[1:])

    def max_speed(self, u):
        return np.abs(u[0])


class Op2D:
    """Oracle 2-D operator on a periodic nex x ney mesh of [x0,x1] x [y0,y1]."""

    def __init__(self, x0, x1, y0, y1, nex, ney, degree, problem, penalty=2.0, rtol=1e-14, maxit=1000,
                 cg_log=None, av=None):
        self.av = av            # (kappa_s, c_s): Persson-Peraire artificial viscosity, frozen per slab
        self.nu_art = None      # (ney, nex) once begin_slab has run
        self.nex, self.ney, self.P = int(nex), int(ney), int(degree)
        self.p1 = self.P + 1
        self.dx, self.dy = (x1 - x0) / nex, (y1 - y0) / ney
        self.x0, self.y0 = x0, y0
        self.prob = problem
        self.nc = problem.ncomp
        self.xi, self.w = quad.gll(self.p1)
        self.D = quad.diff_matrix(self.xi)
        self.penalty = penalty
        self.n = self.nc * self.ney * self.nex * self.p1 * self.p1
        # lumped mass per node (dx/2 w_i)(dy/2 w_j)
        self.m2 = (0.5 * self.dy * self.w)[:, None] * (0.5 * self.dx * self.w)[None, :]
        self.rtol, self.maxit = rtol, maxit
        self.cg_log = [] if cg_log is None else cg_log

    # layout ------------------------------------------------------------
    def u5(self, u):
        return np.asarray(u).reshape(self.nc, self.ney, self.nex, self.p1, self.p1)

    def nodes(self):
        ex = self.x0 + self.dx * np.arange(self.nex)
        ey = self.y0 + self.dy * np.arange(self.ney)
        xs = ex[:, None] + 0.5 * self.dx * (self.xi + 1.0)[None, :]     # (nex, p1)
        ys = ey[:, None] + 0.5 * self.dy * (self.xi + 1.0)[None, :]     # (ney, p1)
        X = np.broadcast_to(xs[None, :, None, :], (self.ney, self.nex, self.p1, self.p1))
        Y = np.broadcast_to(ys[:, None, :, None], (self.ney, self.nex, self.p1, self.p1))
        return X, Y

    # direction helpers: bring (element, node) of the direction to the end --
    @staticmethod
    def _to_end(a, axis):
        # a: (..., ney, nex, p1y, p1x); axis 0 = x -> (.., ney, p1y, nex, p1x); axis 1 = y -> (.., nex, p1x, ney, p1y)
        nd = a.ndim
        if axis == 0:
            return np.moveaxis(a, (nd - 3, nd - 1), (nd - 2, nd - 1))
        return np.moveaxis(a, (nd - 4, nd - 2), (nd - 2, nd - 1))

    @staticmethod
    def _from_end(a, axis):
        nd = a.ndim
        if axis == 0:
            return np.moveaxis(a, (nd - 2, nd - 1), (nd - 3, nd - 1))
        return np.moveaxis(a, (nd - 2, nd - 1), (nd - 4, nd - 2))

    # convection (dgsem.py:205-225 along each direction) -------------------
    def apply_convection(self, u, t=0.0):
        u5 = self.u5(u)
        out = np.zeros_like(u5)
        for axis, h in ((0, self.dx), (1, self.dy)):
            ue = self._to_end(u5, axis)                     # (nc, ..., ne, p1)
            f = self.prob.flux(ue, axis)
            vol = np.einsum("ki,k,...ek->...ei", self.D, self.w, f)
            um = ue[..., :, -1]
            up = np.roll(ue, -1, axis=-2)[..., :, 0]
            lam = np.maximum(self.prob.speed(um, axis), self.prob.speed(up, axis))
            fh = 0.5 * (self.prob.flux(um, axis) + self.prob.flux(up, axis)) - 0.5 * lam[None] * (up - um)
            vol[..., -1] -= fh
            vol[..., 0] += np.roll(fh, 1, axis=-1)
            out += self._from_end(vol * (2.0 / h) / self.w, axis)
        return out.reshape(-1)

    # SIP diffusion with a scalar field C (ney, nex, p1, p1) ---------------
    def _coef5(self, C):
        if np.isscalar(C):
            return np.full((self.ney, self.nex, self.p1, self.p1), float(C))
        return np.asarray(C).reshape(self.ney, self.nex, self.p1, self.p1)

    def apply_diffusion(self, C, u, t=0.0):
        if C is None:
            return np.zeros(self.n)
        u5 = self.u5(u)
        C5 = self._coef5(C)
        out = np.zeros_like(u5)
        for axis, h in ((0, self.dx), (1, self.dy)):
            ue = self._to_end(u5, axis)
            Ce = self._to_end(C5[None], axis)[0]
            s = 2.0 / h
            mu0 = self.penalty * self.p1 ** 2 / h
            g = s * np.einsum("ij,...ej->...ei", self.D, ue)
            q = Ce[None] * g
            B = np.einsum("ki,k,...ek->...ei", self.D, self.w, q)
            um, up = ue[..., :, -1], np.roll(ue, -1, axis=-2)[..., :, 0]
            qm, qp = q[..., :, -1], np.roll(q, -1, axis=-2)[..., :, 0]
            Cm, Cp = Ce[..., :, -1], np.roll(Ce, -1, axis=-2)[..., :, 0]
            jump = um - up
            G = mu0 * 0.5 * (Cm + Cp)[None] * jump - 0.5 * (qm + qp)
            B[..., -1] += G
            B[..., 0] -= np.roll(G, 1, axis=-1)
            B -= s * (0.5 * Cm[None] * jump)[..., None] * self.D[-1]
            B -= s * np.roll(0.5 * Cp[None] * jump, 1, axis=-1)[..., None] * self.D[0]
            out += self._from_end(-B / (0.5 * h * self.w), axis)
        return out.reshape(-1)

    # physical viscous operator of NS2D (tensor SIP, see NS2D) -------------
    def apply_viscous(self, u, t=0.0):
        """f_visc = -M^-1 (B_x + B_y): per direction the reference's matrix
        SIP (``dgsem.py:251-309``) with the full viscous flux (cross terms
        included) as q, the normal-normal block G_nn in the penalty
        mu0 {G_nn}[u] and in the adjoint lift (each side's own G_nn)."""
        pr = self.prob
        u5 = self.u5(u)
        gx = (2.0 / self.dx) * np.einsum("ij,...bj->...bi", self.D, u5)
        gy = (2.0 / self.dy) * np.einsum("ij,...jb->...ib", self.D, u5)
        Fx, Fy = pr.visc_flux(u5, gx, gy)
        out = np.zeros_like(u5)
        for axis, h, F in ((0, self.dx, Fx), (1, self.dy, Fy)):
            ue = self._to_end(u5, axis)
            Fe = self._to_end(F, axis)
            s = 2.0 / h
            mu0 = self.penalty * self.p1 ** 2 / h
            B = np.einsum("ki,k,...ek->...ei", self.D, self.w, Fe)
            um, up = ue[..., :, -1], np.roll(ue, -1, axis=-2)[..., :, 0]
            qm, qp = Fe[..., :, -1], np.roll(Fe, -1, axis=-2)[..., :, 0]
            jump = um - up
            gm, gp = pr.apply_gnn(um, jump, axis), pr.apply_gnn(up, jump, axis)
            G = mu0 * (0.5 * (gm + gp)) - 0.5 * (qm + qp)
            B[..., -1] += G
            B[..., 0] -= np.roll(G, 1, axis=-1)
            B -= s * (0.5 * gm)[..., None] * self.D[-1]
            B -= s * np.roll(0.5 * gp, 1, axis=-1)[..., None] * self.D[0]
            out += self._from_end(-B / (0.5 * h * self.w), axis)
        return out.reshape(-1)

    def stiffness_diag(self, C):
        """diag of M * (-apply_diffusion) per node (shape (n,)), closed form."""
        C5 = self._coef5(C)
        d = np.zeros((self.ney, self.nex, self.p1, self.p1))
        for axis, h, hperp in ((0, self.dx, self.dy), (1, self.dy, self.dx)):
            Ce = self._to_end(C5[None], axis)[0]
            s = 2.0 / h
            mu0 = self.penalty * self.p1 ** 2 / h
            dd = s * np.einsum("ki,k,...ek->...ei", self.D ** 2, self.w, Ce)
            Cm = Ce[..., :, -1]
            Cp = np.roll(Ce, -1, axis=-2)[..., :, 0]
            muC = mu0 * 0.5 * (Cm + Cp)
            dd[..., -1] += muC - s * Cm * self.D[-1, -1]
            dd[..., 0] += np.roll(muC + s * Cp * self.D[0, 0], 1, axis=-1)
            # line stiffness scaled by the transverse mass factor (hperp/2) w_perp
            dd = self._from_end(dd[None], axis)[0]
            wperp = (0.5 * hperp * self.w)
            d += dd * (wperp[None, None, None, :] if axis == 1 else wperp[None, None, :, None])
        return np.tile(d.reshape(-1), self.nc)

    # rhs / SI coefficient / implicit solve --------------------------------
    def _av_field(self):
        """nu_art broadcast to the nodes, or None."""
        if self.nu_art is None:
            return None
        return np.broadcast_to(self.nu_art[:, :, None, None], (self.ney, self.nex, self.p1, self.p1))

    def persson_viscosity(self, u):
        """Tensor-product generalisation of the reference's modal sensor (``dgsem.py:537-559``):
        Legendre modes m_kl of field 0, energies m_kl^2 (2/(2k+1)) (2/(2l+1)), sensor = log10 of the
        share of the modes with max(k, l) = P, the reference's ramp around s0 = -4 log10 P, and
        eps0 = c_s h lam_max / P with h = max(dx, dy).  On y-invariant data only l = 0 survives and
        the value is the reference's 1-D one (tests/test_oracle2d.py)."""
        if self.av is None:
            return np.zeros((self.ney, self.nex))
        kap, cs = self.av
        P = self.P
        u5 = self.u5(u)
        V = np.polynomial.legendre.legvander(self.xi, P)
        Vi = np.linalg.inv(V)
        modal = np.einsum("kj,li,...ji->...kl", Vi, Vi, u5[0])
        nk = 2.0 / (2.0 * np.arange(self.p1) + 1.0)
        en = modal ** 2 * (nk[:, None] * nk[None, :])
        tot = en.sum(axis=(-1, -2))
        top = en[..., -1, :].sum(axis=-1) + en[..., :-1, -1].sum(axis=-1)
        with np.errstate(divide="ignore", invalid="ignore"):
            sv = np.where(tot > 0.0, np.log10(np.maximum(top, 1e-300) / tot), -np.inf)
        s0 = -4.0 * np.log10(P)
        lam = self.prob.max_speed(u5).max(axis=(-1, -2))
        eps0 = cs * max(self.dx, self.dy) * lam / P
        with np.errstate(invalid="ignore"):
            ramp = np.where(sv < s0 - kap, 0.0,
                            np.where(sv > s0 + kap, 1.0, 0.5 * (1.0 + np.sin(0.5 * np.pi * (sv - s0) / kap))))
        return eps0 * ramp

    def eval_rhs(self, u, t=0.0):
        out = self.apply_convection(u, t)
        av = self._av_field()
        if getattr(self.prob, "viscous", False):
            out = out + self.apply_viscous(u, t)
            if av is not None:
                out = out + self.apply_diffusion(av, u, t)
        elif av is not None:
            out = out + self.apply_diffusion(max(self.prob.nu, 0.0) + av, u, t)
        elif self.prob.nu > 0:
            out = out + self.apply_diffusion(self.prob.nu, u, t)
        if not np.all(np.isfinite(out)):
            bad = ~np.isfinite(out.reshape(self.nc, self.ney * self.nex, -1))
            e = int(np.nonzero(bad.any(axis=(0, 2)))[0][0])
            raise RuntimeError(f"non-finite right-hand side in element {e}")
        return out

    def modified_coeff(self, u_b, dt_m, scheme="si2"):
        lam = self.prob.max_speed(self.u5(u_b))
        c = 0.5 * dt_m * (lam * lam)
        av = self._av_field()
        if getattr(self.prob, "viscous", False):
            c = c + self.prob.nu_si(self.u5(u_b))
            return c + av if av is not None else c
        if av is not None:
            return c + (max(self.prob.nu, 0.0) + av)
        return c + self.prob.nu if self.prob.nu > 0 else c

    def implicit_solve(self, C, a, rhs, t=0.0):
        if a == 0.0:
            return rhs
        m = np.tile(self.m2.reshape(1, 1, self.p1, self.p1), (self.ney, self.nex, 1, 1)).reshape(-1)
        m = np.tile(m, self.nc)
        b = m * np.asarray(rhs).reshape(-1)
        if not b.any():
            return np.zeros_like(rhs)
        diag = m + a * self.stiffness_diag(C)
        A = lambda x: m * x - a * m * self.apply_diffusion(C, x, t)
        x, it, margin = pcg(A, diag, b, np.asarray(rhs).reshape(-1).copy(), self.rtol, self.maxit)
        if it < 0:
            raise RuntimeError("implicit CG solve did not converge")
        self.cg_log.append((it, margin))
        return x

    def begin_slab(self, u0, t0, dt):
        if self.av is not None:
            self.nu_art = self.persson_viscosity(u0)


class PTransfer2D:
    """Spatial p-transfer as the tensor product of the 1-D GLL Lagrange
    matrices (``transfer.py:213-245`` per direction) with the temporal
    Lagrange transfer (``transfer.py:61-121``), SpaceTimeTransfer order."""

    def __init__(self, ctx_c, ctx_f, rule_c, rule_f):
        self.nc, self.ney, self.nex = ctx_f.nc, ctx_f.ney, ctx_f.nex
        self.pc, self.pf = ctx_c.p1, ctx_f.p1
        xc, xf = quad.gll(self.pc)[0], quad.gll(self.pf)[0]
        self.I = quad.lagrange(xc, xf)
        self.Pm = quad.lagrange(xf, xc)
        # mass-consistent residual restriction M_c^-1 I^T M_f (the 2-D
        # formulation; the reference's I^T over-injects)
        wc, wf = quad.gll(self.pc)[1], quad.gll(self.pf)[1]
        self.R = (1.0 / wc)[:, None] * self.I.T * wf[None, :]
        self.It = quad.lagrange(rule_c.tau, rule_f.tau)
        self.Pt = quad.lagrange(rule_f.tau, rule_c.tau)

    def sp(self, A, u, n_in):
        u = u.reshape(self.nc, self.ney, self.nex, n_in, n_in)
        return np.einsum("ab,ij,cyxbj->cyxai", A, A, u).reshape(-1)

    def project_u0(self, u0f):
        return self.sp(self.Pm, u0f, self.pf)

    def project_solution(self, uf):
        return np.tensordot(self.Pt, np.stack([self.sp(self.Pm, x, self.pf) for x in uf]), axes=(1, 0))

    def restrict_residual(self, rf):
        return np.tensordot(self.It.T, np.stack([self.sp(self.R, x, self.pf) for x in rf]), axes=(1, 0))

    def interp(self, dc):
        t = np.tensordot(self.It, dc, axes=(1, 0))
        return np.stack([self.sp(self.I, x, self.pc) for x in t])
