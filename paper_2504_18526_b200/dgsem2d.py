"""GPU 2-D tensor-product DG-SEM operator (BASELINE configs 3-5).

The reference is 1-D only.  ``DGOperator2D`` exposes the same
``OperatorContext`` methods as ``dgsem.DGOperator`` on a uniform periodic
nex x ney mesh, so the unchanged sweeper (``sdc.py``) and multilevel engine
(``mlsdc.py``) drive it.  Operators are the reference's 1-D operators applied
along x- and y-lines (``dgsem.py:205-225, 251-309``); the semi-implicit
coefficient is the isotropic SPD (dt_m/2) lambda(u_b)^2 + nu, lambda = |v| + c
(DESIGN.md "2-D formulation").  State layout (ncomp, ney, nex, P+1, P+1).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import _lib
from ._lib import Coef
from .collocation import gauss_lobatto
from .dgsem import SICoefficient
from .runtime import get_runtime


@dataclass(frozen=True)
class Mesh2D:
    x_left: float
    x_right: float
    y_bottom: float
    y_top: float
    nex: int
    ney: int
    degree: int

    def __post_init__(self):
        if self.x_right <= self.x_left or self.y_top <= self.y_bottom:
            raise ValueError("empty domain")
        if self.nex < 1 or self.ney < 1 or self.degree < 1:
            raise ValueError("need elements and degree >= 1")

    @property
    def dx(self):
        return (self.x_right - self.x_left) / self.nex

    @property
    def dy(self):
        return (self.y_top - self.y_bottom) / self.ney

    @property
    def n_elem(self):
        return self.nex * self.ney

    @cached_property
    def ref_nodes(self):
        return gauss_lobatto(self.degree + 1)[0]

    @cached_property
    def nodes_xy(self):
        """(X, Y) node coordinates, each (ney, nex, P+1, P+1)."""
        xi = self.ref_nodes
        xs = (self.x_left + self.dx * np.arange(self.nex))[:, None] + 0.5 * self.dx * (xi + 1.0)[None, :]
        ys = (self.y_bottom + self.dy * np.arange(self.ney))[:, None] + 0.5 * self.dy * (xi + 1.0)[None, :]
        p1 = self.degree + 1
        X = np.broadcast_to(xs[None, :, None, :], (self.ney, self.nex, p1, p1))
        Y = np.broadcast_to(ys[:, None, :, None], (self.ney, self.nex, p1, p1))
        return X, Y


class CompressibleEuler2D:
    """2-D compressible Euler / Navier-Stokes (isotropic constant kinematic
    viscosity nu on the conservative fields), ideal gas."""
    ncomp = 4
    is_linear = False
    source = None
    kind = "euler2d"

    def __init__(self, gamma: float = 1.4, nu: float = 0.0):
        if gamma <= 1.0:
            raise ValueError("gamma must exceed 1")
        if nu < 0:
            raise ValueError("viscosity must be nonnegative")
        self.gamma, self.nu = float(gamma), float(nu)


class Advection2D:
    ncomp = 1
    is_linear = True
    source = None
    kind = "advection2d"

    def __init__(self, ax: float = 1.0, ay: float = 0.0, nu: float = 0.0):
        self.ax, self.ay, self.nu = float(ax), float(ay), float(nu)


class Burgers2D:
    ncomp = 1
    is_linear = False
    source = None
    kind = "burgers2d"

    def __init__(self, nu: float = 0.0):
        self.nu = float(nu)


_KIND = {"euler2d": _lib.EULER2D, "advection2d": _lib.ADVECTION2D, "burgers2d": _lib.BURGERS2D}


class DGOperator2D:
    is2d = True

    def __init__(self, mesh: Mesh2D, problem, penalty_const: float = 2.0, device: int = 0, eager_checks: bool = True):
        self.mesh = mesh
        self.problem = problem
        self.av = None
        self.ncomp = problem.ncomp
        self.p1 = mesh.degree + 1
        self.ndof = self.ncomp * mesh.n_elem * self.p1 * self.p1
        self.rt = get_runtime(device)
        self.lib = self.rt.lib
        self.eager_checks = eager_checks
        d = _lib.Op2DDesc(mesh.nex, mesh.ney, mesh.degree, self.ncomp, _KIND[problem.kind],
                          float(mesh.x_left), float(mesh.x_right), float(mesh.y_bottom), float(mesh.y_top),
                          float(getattr(problem, "gamma", 1.4)), float(problem.nu),
                          float(getattr(problem, "ax", 0.0)), float(getattr(problem, "ay", 0.0)), float(penalty_const))
        self._desc = d
        h = C.c_void_p()
        self.rt.check(self.lib.sisdc_op2d_create(self.rt.h, C.byref(d), C.byref(h)), "op2d_create")
        self.h = h
        self._scratch = None
        self.nu_art = None

    def __del__(self):
        try:
            self.lib.sisdc_op1d_destroy(self.h)
        except Exception:
            pass

    def as_nodes(self, u):
        return self.rt.to_device(u).reshape(self.ncomp, self.mesh.ney, self.mesh.nex, self.p1, self.p1)

    def scratch(self):
        if self._scratch is None:
            self._scratch = {k: self.rt.empty(self.ndof) for k in ("rhs", "stage", "conv")}
        return self._scratch

    def _out(self, out):
        self.rt.bind_stream()
        return self.rt.empty(self.ndof) if out is None else out

    def _coef(self, coeff, keep):
        if coeff is None:
            return Coef(_lib.COEF_NONE, 0.0, None)
        if isinstance(coeff, SICoefficient):
            return coeff.c()
        if np.isscalar(coeff):
            return Coef(_lib.COEF_CONST, float(coeff), None)
        t = self.rt.to_device(coeff)
        keep.append(t)
        return Coef(_lib.COEF_FIELD, 0.0, t.data_ptr())

    def modified_diffusion_matrix(self, u_b, dt_m: float, scheme: str):
        if scheme == "euler":
            return self.problem.nu if self.problem.nu > 0 else None
        if scheme not in ("si1", "si2"):
            raise ValueError(f"unknown scheme {scheme!r}")
        return SICoefficient(self.rt.to_device(u_b).clone(), dt_m)

    def apply_convection(self, u, t: float = 0.0, out=None):
        u = self.rt.to_device(u)
        out = self._out(out)
        self.rt.check(self.lib.sisdc_apply_convection(self.h, u.data_ptr(), float(t), out.data_ptr()), "apply_convection")
        return out

    def apply_diffusion(self, coeff, u, t: float = 0.0, out=None):
        keep = []
        c = self._coef(coeff, keep)
        u = self.rt.to_device(u)
        out = self._out(out)
        self.rt.check(self.lib.sisdc_apply_diffusion(self.h, c, u.data_ptr(), float(t), out.data_ptr()), "apply_diffusion")
        return out

    def eval_rhs(self, u, t: float = 0.0, out=None):
        u = self.rt.to_device(u)
        out = self._out(out)
        if self.eager_checks:
            self.rt.reset_status()
        self.rt.check(self.lib.sisdc_eval_rhs(self.h, u.data_ptr(), float(t), out.data_ptr()), "eval_rhs")
        if self.eager_checks:
            self.rt.raise_on_failure()
        return out

    def apply_source(self, u, t: float):
        return self.rt.zeros(self.ndof)

    def coefficient_field(self, coeff):
        keep = []
        c = self._coef(coeff, keep)
        out = self.rt.empty(self.mesh.n_elem * self.p1 * self.p1)
        self.rt.bind_stream()
        self.rt.check(self.lib.sisdc_coef_field(self.h, c, out.data_ptr()), "coef_field")
        return out

    def implicit_solve(self, coeff, a: float, rhs, t: float = 0.0, out=None):
        if a == 0.0:
            return rhs
        keep = []
        c = self._coef(coeff, keep)
        rhs = self.rt.to_device(rhs)
        out = self._out(out)
        if self.eager_checks:
            self.rt.reset_status()
        self.rt.check(self.lib.sisdc_implicit_solve(self.h, c, float(a), rhs.data_ptr(), float(t), out.data_ptr()),
                      "implicit_solve")
        if self.eager_checks:
            self.rt.raise_on_failure()
        return out

    def begin_slab(self, u0, t0: float, dt: float) -> None:
        pass
