"""GPU nodal DG-SEM operator: the reference's ``DGOperator`` on sm_100a.

Mirrors ``dgsem.py`` of the reference (``Mesh1D`` ``:72-106``, ``DGOperator``
``:117-571``, ``compute_delta``/``dt_from_cfl`` ``:46-69``) with the
``OperatorContext`` methods executed by ``libsisdc_b200.so``:

* ``apply_convection``  -> weak volume term + Rusanov faces   (``:205-225``)
* ``apply_diffusion``   -> matrix-free SIP                     (``:251-309``)
* ``eval_rhs``          -> convection + physical diffusion     (``:337-352``)
* ``implicit_solve``    -> cluster-resident Jacobi-PCG         (replaces ``:503-533``)
* ``persson_viscosity`` -> modal sensor                        (``:537-559``)

States are torch float64 CUDA tensors (numpy inputs are uploaded); results
are returned as new CUDA tensors unless ``out=`` is given.  Scope of the
built path: scalar problems (ConvectionDiffusion, Burgers) on periodic and
Dirichlet meshes; 1-D CompressibleFlow (3 fields, matrix coefficients) on
periodic meshes.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from functools import cached_property, lru_cache
from typing import Any, Optional

import numpy as np

from . import _lib
from ._lib import Coef, SolverError
from .collocation import gauss_lobatto
from .runtime import get_runtime


def torch_isfinite(t):
    import torch
    return torch.isfinite(t)

__all__ = ["Mesh1D", "DGOperator", "SolverError", "ArtificialViscosityParams", "SICoefficient",
           "compute_delta", "cfl_number", "dt_from_cfl", "max_wave_speed", "smooth_start"]


def _diff_matrix(x) -> np.ndarray:
    x = np.asarray(x, dtype=float)
    n = len(x)
    lam = np.array([1.0 / np.prod([x[j] - x[k] for k in range(n) if k != j]) for j in range(n)])
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i, j] = (lam[j] / lam[i]) / (x[i] - x[j])
        D[i, i] = -D[i].sum()
    return D


@lru_cache(maxsize=None)
def compute_delta(degree: int) -> float:
    """delta(P): spectral radius of the inflow-stripped derivative (``dgsem.py:46-59``)."""
    if degree < 1:
        raise ValueError("degree must be >= 1")
    x, _ = gauss_lobatto(degree + 1)
    return float(np.max(np.abs(np.linalg.eigvals(-_diff_matrix(x)[1:, 1:]))))


def cfl_number(dt, dx_elem, lam_max, degree):
    return dt * lam_max * 2.0 * compute_delta(degree) / dx_elem


def dt_from_cfl(cfl, dx_elem, lam_max, degree):
    return cfl * dx_elem / (2.0 * compute_delta(degree) * lam_max)


@dataclass(frozen=True)
class Mesh1D:
    """Uniform 1-D mesh of n_elem elements with degree-P GLL nodes."""

    x_left: float
    x_right: float
    n_elem: int
    degree: int
    bc: str = "periodic"

    def __post_init__(self):
        if self.x_right <= self.x_left:
            raise ValueError("empty domain")
        if self.n_elem < 1 or self.degree < 1:
            raise ValueError("need at least one element and degree >= 1")
        if self.bc not in ("periodic", "dirichlet"):
            raise ValueError(f"unknown bc {self.bc!r}")

    @property
    def dx(self) -> float:
        return (self.x_right - self.x_left) / self.n_elem

    @cached_property
    def ref_nodes(self) -> np.ndarray:
        return gauss_lobatto(self.degree + 1)[0]

    @cached_property
    def ref_weights(self) -> np.ndarray:
        return gauss_lobatto(self.degree + 1)[1]

    @cached_property
    def nodes_x(self) -> np.ndarray:
        edges = self.x_left + self.dx * np.arange(self.n_elem)
        return edges[:, None] + 0.5 * self.dx * (self.ref_nodes + 1.0)[None, :]


@dataclass(frozen=True)
class ArtificialViscosityParams:
    kappa_s: float
    c_s: float


class SICoefficient:
    """Opaque semi-implicit coefficient (dt_m/2) A_c(u_b)^2 + A_d (+nu_art)
    frozen at u_b (``dgsem.py:356-396``); evaluated on the fly in-kernel.
    ``u_b`` is owned (a snapshot) unless created by the fused sweeper."""

    __slots__ = ("u_b", "dt_m", "kind")

    def __init__(self, u_b, dt_m: float, kind: int = _lib.COEF_SI):
        self.u_b = u_b
        self.dt_m = float(dt_m)
        self.kind = kind

    def c(self) -> Coef:
        return Coef(self.kind, self.dt_m, self.u_b.data_ptr() if self.u_b is not None else None)


class DGOperator:
    """Spatial operator bundle on one mesh/problem pair, executed on the GPU."""

    def __init__(self, mesh: Mesh1D, problem, av: Optional[ArtificialViscosityParams] = None,
                 penalty_const: float = 2.0, device: int = 0, eager_checks: bool = True):
        if mesh.bc == "dirichlet" and getattr(problem, "boundary_state", None) is None:
            raise ValueError("dirichlet mesh needs a problem with boundary_state(t)")   # dgsem.py:150-151
        self.mesh = mesh
        self.problem = problem
        self.av = av
        self.ncomp = problem.ncomp
        self.p1 = mesh.degree + 1
        self.ndof = self.ncomp * mesh.n_elem * self.p1
        self.rt = get_runtime(device)
        self.lib = self.rt.lib
        self.eager_checks = eager_checks
        kind = {"convdiff": _lib.CONVDIFF, "burgers": _lib.BURGERS, "cns": _lib.CNS1D}[problem.kind]
        self.is_cns = problem.kind == "cns"
        self.dirichlet = mesh.bc == "dirichlet"
        self._btimes = {}   # insertion-ordered mirror of the library's trace table (abi.cu set_boundary)
        self._desc = _lib.Op1DDesc(mesh.n_elem, mesh.degree, self.ncomp,
                                   _lib.DIRICHLET if self.dirichlet else _lib.PERIODIC, kind,
                                   float(mesh.x_left), float(mesh.x_right), float(getattr(problem, "speed", 0.0)),
                                   float(problem.nu), float(penalty_const),
                                   float(getattr(problem, "gamma", 1.4)), float(getattr(problem, "eta", 0.0)),
                                   float(getattr(problem, "Pr", 0.75)))
        h = C.c_void_p()
        self.rt.check(self.lib.sisdc_op1d_create(self.rt.h, C.byref(self._desc), C.byref(h)), "op1d_create")
        self.h = h
        nodes = np.zeros(self.p1)
        wts = np.zeros(self.p1)
        Dm = np.zeros(self.p1 * self.p1)
        self.lib.sisdc_op1d_tables(h, nodes.ctypes.data_as(_lib.DP), wts.ctypes.data_as(_lib.DP),
                                   Dm.ctypes.data_as(_lib.DP))
        self.ref_nodes, self.ref_weights, self.D = nodes, wts, Dm.reshape(self.p1, self.p1)
        self.mass_node = 0.5 * mesh.dx * wts
        self.inv_mass = 1.0 / self.mass_node
        self.mu0 = penalty_const * self.p1 ** 2 / mesh.dx
        # source(x, t, u3) (dgsem.py:328-352): a host callable, evaluated on the host
        # at the node coordinates and added to f on the device (no graph capture)
        self.source_fn = getattr(problem, "source", None)
        # a known forcing src(x, t): device tables keyed by time (no device -> host copy of the state,
        # one upload per distinct node time; cleared every slab)
        self.source_tabulated = self.source_fn is not None and not getattr(problem, "source_depends_on_state", True)
        self._src_tab = {}
        self.nu_art = None            # device tensor (n_elem,) when AV is active
        self._last_dt = None
        self._scratch = None

    def __del__(self):
        try:
            self.lib.sisdc_op1d_destroy(self.h)
        except Exception:
            pass

    # ------------------------------------------------------------- layout
    def as_nodes(self, u):
        return self.rt.to_device(u).reshape(self.ncomp, self.mesh.n_elem, self.p1)

    def flat(self, u3):
        return self.rt.to_device(u3).reshape(-1)

    def nodal_field(self, fn):
        vals = np.asarray(fn(self.mesh.nodes_x))
        if vals.shape != (self.ncomp, self.mesh.n_elem, self.p1):
            raise ValueError("initial data has the wrong shape")
        return self.rt.to_device(vals.reshape(-1))

    def scratch(self):
        """Per-operator device scratch used by the fused sweeper."""
        if self._scratch is None:
            self._scratch = {k: self.rt.empty(self.ndof) for k in ("rhs", "stage", "conv")}
        return self._scratch

    # ------------------------------------------------------- coefficients
    def _coef(self, coeff, keep: list) -> Coef:
        if coeff is None:
            return Coef(_lib.COEF_NONE, 0.0, None)
        if isinstance(coeff, SICoefficient):
            return coeff.c()
        if np.isscalar(coeff):
            return Coef(_lib.COEF_CONST, float(coeff), None)
        t = self.rt.to_device(coeff).contiguous()
        nn = self.mesh.n_elem * self.p1
        if self.is_cns and t.numel() == nn * self.ncomp * self.ncomp:   # (n_elem, P+1, nc, nc)
            keep.append(t)
            return Coef(_lib.COEF_MATRIX, 0.0, t.data_ptr())
        if t.numel() != nn:
            raise NotImplementedError("matrix-valued coefficients are built for CompressibleFlow only")
        keep.append(t)
        return Coef(_lib.COEF_FIELD, 0.0, t.data_ptr())

    def _phys(self):
        """Physical coefficient as the reference returns it (``dgsem.py:313-326``)."""
        nu = self.problem.nu
        if self.nu_art is None:
            return nu if nu > 0 else None
        return SICoefficient(None, 0.0, _lib.COEF_PHYS)

    def modified_diffusion_matrix(self, u_b, dt_m: float, scheme: str) -> Any:
        if self.is_cns:   # matrix-valued, frozen at u_b (dgsem.py:356-396)
            if scheme == "euler":
                if not self.problem.viscous and self.nu_art is None:
                    return None
                return SICoefficient(self.rt.to_device(u_b).clone(), 0.0, _lib.COEF_PHYS)
            if scheme not in ("si1", "si2"):
                raise ValueError(f"unknown scheme {scheme!r}")
            return SICoefficient(self.rt.to_device(u_b).clone(), dt_m)
        if scheme == "euler":
            return self._phys()
        if scheme not in ("si1", "si2"):
            raise ValueError(f"unknown scheme {scheme!r}")
        if self.problem.is_linear and self.nu_art is None:
            # constant: exactly the reference's float (dgsem.py:382-393)
            half = 0.5 * dt_m * float(self.problem.speed) ** 2
            return half + self.problem.nu if self.problem.nu > 0 else half
        return SICoefficient(self.rt.to_device(u_b).clone(), dt_m)

    # --------------------------------------------------- Dirichlet trace data
    def boundary_at(self, *times):
        """Register problem.boundary_state(t) for the given times with the
        library (dgsem.py:212-216): host evaluation, no device work."""
        if not self.dirichlet:
            return
        new = list(dict.fromkeys(float(t) for t in times if float(t) not in self._btimes))
        if not new:
            return
        gl, gr = zip(*[self.problem.boundary_state(t) for t in new])
        ta, tp = _lib.darr(new)
        nc = self.ncomp   # (n, ncomp) outside states
        la, lp = _lib.darr([float(v) for g in gl for v in np.asarray(g, dtype=float).reshape(-1)[:nc]])
        ra, rp = _lib.darr([float(v) for g in gr for v in np.asarray(g, dtype=float).reshape(-1)[:nc]])
        self.rt.check(self.lib.sisdc_op1d_set_boundary(self.h, len(new), tp, lp, rp), "set_boundary")
        for t in new:
            self._btimes[t] = None
        if len(self._btimes) > 4096:   # the library keeps its 1024 most recent times past 4096 (same rule)
            self._btimes = dict.fromkeys(list(self._btimes)[-1024:])

    # ---------------------------------------------------------- operators
    def _out(self, out):
        self.rt.bind_stream()
        return self.rt.empty(self.ndof) if out is None else out

    def apply_convection(self, u, t: float = 0.0, out=None):
        u = self.rt.to_device(u)
        out = self._out(out)
        self.boundary_at(t)
        self.rt.check(self.lib.sisdc_apply_convection(self.h, u.data_ptr(), float(t), out.data_ptr()),
                      "apply_convection")
        return out

    def apply_diffusion(self, coeff, u, t: float = 0.0, out=None):
        keep = []
        c = self._coef(coeff, keep)
        u = self.rt.to_device(u)
        out = self._out(out)
        self.boundary_at(t)
        self.rt.check(self.lib.sisdc_apply_diffusion(self.h, c, u.data_ptr(), float(t), out.data_ptr()),
                      "apply_diffusion")
        return out

    def eval_rhs(self, u, t: float = 0.0, out=None):
        u = self.rt.to_device(u)
        out = self._out(out)
        if self.eager_checks:
            self.rt.reset_status()
        self.boundary_at(t)
        self.rt.check(self.lib.sisdc_eval_rhs(self.h, u.data_ptr(), float(t), out.data_ptr()), "eval_rhs")
        if self.source_fn is not None:
            self.add_source(out, u, t)
            self._check_finite(out)
        if self.eager_checks:
            self.rt.raise_on_failure()
        return out

    def _source_values(self, u, t: float):
        """src(x, t, u3) on the host (dgsem.py:328-335), broadcast over the
        components, as a device vector; None when the source returns None."""
        if self.source_tabulated:
            key = float(t)
            if key not in self._src_tab:
                if len(self._src_tab) >= 64:   # standalone eval_rhs at many times: keep the cache bounded
                    self._src_tab.clear()
                vals = self.source_fn(self.mesh.nodes_x, key, None)
                self._src_tab[key] = None if vals is None else self.rt.to_device(np.ascontiguousarray(
                    (np.asarray(vals, dtype=np.float64) + np.zeros((self.ncomp, 1, 1))).reshape(-1)))
            return self._src_tab[key]
        u3 = self.as_nodes(u).detach().cpu().numpy()
        vals = self.source_fn(self.mesh.nodes_x, float(t), u3)
        if vals is None:
            return None
        v = np.asarray(vals, dtype=np.float64) + np.zeros((self.ncomp, 1, 1))
        return self.rt.to_device(np.ascontiguousarray(v.reshape(-1)))

    def add_source(self, f, u, t: float) -> None:
        """f += src(x, t, u) (the source term of eval_rhs, dgsem.py:343-347)."""
        if self.source_fn is None:
            return
        v = self._source_values(u, t)
        if v is not None:
            f.add_(v)

    def _check_finite(self, out) -> None:
        bad = ~torch_isfinite(out.reshape(self.ncomp, self.mesh.n_elem, self.p1))
        if bool(bad.any()):
            e = int(bad.any(dim=0).any(dim=1).nonzero()[0, 0])
            raise SolverError(f"non-finite right-hand side in element {e}")

    def apply_source(self, u, t: float):
        if self.source_fn is None:
            return self.rt.zeros(self.ndof)
        v = self._source_values(self.rt.to_device(u), t)
        return self.rt.zeros(self.ndof) if v is None else v.clone()

    def coefficient_field(self, coeff):
        """Materialise a coefficient as an (n_elem, P+1) device field
        ((n_elem, P+1, 3, 3) for CompressibleFlow)."""
        keep = []
        c = self._coef(coeff, keep)
        per = self.ncomp * self.ncomp if self.is_cns else 1
        out = self.rt.empty(self.mesh.n_elem * self.p1 * per)
        self.rt.bind_stream()
        self.rt.check(self.lib.sisdc_coef_field(self.h, c, out.data_ptr()), "coef_field")
        if self.is_cns:
            return out.reshape(self.mesh.n_elem, self.p1, self.ncomp, self.ncomp)
        return out.reshape(self.mesh.n_elem, self.p1)

    def implicit_solve(self, coeff, a: float, rhs, t: float = 0.0, out=None):
        """Solve (M + a B[coeff]) x = M rhs with the pinned Jacobi-PCG
        (CompressibleFlow: the pinned element-block-Jacobi BiCGStab)."""
        if a == 0.0:
            return rhs
        keep = []
        c = self._coef(coeff, keep)
        rhs = self.rt.to_device(rhs)
        out = self._out(out)
        if self.eager_checks:
            self.rt.reset_status()
        self.boundary_at(t)
        self.rt.check(self.lib.sisdc_implicit_solve(self.h, c, float(a), rhs.data_ptr(), float(t), out.data_ptr()),
                      "implicit_solve")
        if self.eager_checks:
            self.rt.raise_on_failure()
        return out

    # ---------------------------------------------------- shock sensor / slab
    def persson_viscosity(self, u):
        out = self.rt.zeros(self.mesh.n_elem)
        if self.av is None:
            return out
        u = self.rt.to_device(u)
        self.rt.bind_stream()
        self.rt.check(self.lib.sisdc_persson_viscosity(self.h, u.data_ptr(), float(self.av.kappa_s),
                                                       float(self.av.c_s), out.data_ptr()), "persson")
        return out

    def begin_slab(self, u0, t0: float, dt: float) -> None:
        """Freeze per-slab data (``dgsem.py:563-571``): the AV field."""
        self._src_tab.clear()
        if self.av is not None:
            if self.nu_art is None:
                self.nu_art = self.rt.zeros(self.mesh.n_elem)
            u0 = self.rt.to_device(u0)
            self.rt.bind_stream()
            self.rt.check(self.lib.sisdc_persson_viscosity(self.h, u0.data_ptr(), float(self.av.kappa_s),
                                                           float(self.av.c_s), self.nu_art.data_ptr()), "persson")
            self.lib.sisdc_op1d_set_nu_art(self.h, self.nu_art.data_ptr())
        self._last_dt = dt

    # ------------------------------------------------------------ helpers
    def total_integral(self, u):
        u3 = self.as_nodes(u)
        return (u3 * self.rt.to_device(self.mass_node)).sum(dim=(1, 2))

    def norm_l2(self, u) -> float:
        u3 = self.as_nodes(u)
        return float(((u3 ** 2) * self.rt.to_device(self.mass_node)).sum().sqrt())


def smooth_start(op: DGOperator, u, out=None):
    """Average the two trace values at every interior interface
    (``dgsem.py:574-589``; the periodic wrap too); u may be one state or an
    (M, N) node array."""
    import torch
    u = op.rt.to_device(u)
    M = u.numel() // op.ndof
    if out is None:
        out = torch.empty_like(u)
    op.rt.bind_stream()
    op.rt.check(op.lib.sisdc_smooth_start(op.h, M, u.data_ptr(), out.data_ptr()), "smooth_start")
    return out


def max_wave_speed(op: DGOperator, u) -> float:
    if op.problem.kind == "convdiff":
        return abs(op.problem.speed)
    if op.problem.kind == "cns":   # max(|v| + c), problems.py:194-196
        u3 = op.as_nodes(u)
        g = op.problem.gamma
        v = u3[1] / u3[0]
        p = (g - 1.0) * (u3[2] - 0.5 * u3[1] * v)
        return float((v.abs() + (g * p / u3[0]).sqrt()).max())
    return float(op.rt.to_device(u).abs().max())
