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


class CompressibleNS2D:
    """2-D compressible Navier-Stokes, ideal gas: the Euler flux plus the
    physical viscous flux with dynamic viscosity ``eta`` (Stokes stress) and
    Fourier heat flux with Prandtl number ``prandtl`` -- the 2-D
    generalisation of the reference's ``CompressibleFlow`` viscous term
    (``problems.py:221-237``; restated in ``oracle/dg2d.py`` ``NS2D``).  The
    semi-implicit coefficient is the isotropic scalar (dt_m/2) lambda^2 +
    eta/rho max(4/3, gamma/Pr) shared by the four fields (SPD: CG-solvable)."""
    ncomp = 4
    is_linear = False
    source = None
    kind = "ns2d"

    def __init__(self, gamma: float = 1.4, eta: float = 0.0, prandtl: float = 0.72):
        if gamma <= 1.0:
            raise ValueError("gamma must exceed 1")
        if eta < 0:
            raise ValueError("viscosity must be nonnegative")
        if prandtl <= 0:
            raise ValueError("Prandtl number must be positive")
        self.gamma, self.eta, self.prandtl = float(gamma), float(eta), float(prandtl)
        self.nu = self.eta   # the descriptor's viscosity slot carries eta for NS2D


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


_KIND = {"euler2d": _lib.EULER2D, "ns2d": _lib.NS2D, "advection2d": _lib.ADVECTION2D, "burgers2d": _lib.BURGERS2D}


def rank_rows(ney: int, nranks: int, rank: int):
    """(first row, row count) of ``rank`` when ``ney`` element rows are split
    into contiguous blocks (the split ``sisdc_op2d_create_part`` uses)."""
    if not 1 <= nranks <= ney:
        raise ValueError(f"cannot split {ney} element rows over {nranks} ranks")
    if not 0 <= rank < nranks:
        raise ValueError("rank out of range")
    base, rem = divmod(ney, nranks)
    return rank * base + min(rank, rem), base + (1 if rank < rem else 0)


def part_layout(ney: int, nex: int, p1: int, ncomp: int, nranks: int, ranks):
    """[(first row, rows, offset)] of the partitions of ``ranks`` in the
    concatenated storage vector (ghost row on either side of each partition;
    mirrors ``sisdc_op2d_create_part``)."""
    out, off = [], 0
    for q in ranks:
        rb, rc = rank_rows(ney, nranks, q)
        out.append((rb, rc, off))
        off += ncomp * (rc + 2) * nex * p1 * p1
    return out


def to_storage(g, parts, out):
    """Owned rows of a global state g (ncomp, ney, nex, p1, p1) into the storage
    vector ``out`` (numpy or torch, 1-D) of ``parts``; ghost rows untouched."""
    nc, _, nex, p1, _ = g.shape
    for rb, rc, off in parts:
        v = out[off:off + nc * (rc + 2) * nex * p1 * p1].reshape(nc, rc + 2, nex, p1, p1)
        blk = g[:, rb:rb + rc]
        if hasattr(v, "copy_"):
            import torch
            v[:, 1:-1].copy_(torch.as_tensor(np.ascontiguousarray(blk)))
        else:
            v[:, 1:-1] = blk
    return out


def from_storage(vec, parts, shape):
    """Owned rows of the storage vector ``vec`` (numpy, 1-D) -> global array of
    ``shape`` (ncomp, ney, nex, p1, p1), rows of other ranks NaN."""
    nc, _, nex, p1, _ = shape
    out = np.full(shape, np.nan)
    for rb, rc, off in parts:
        out[:, rb:rb + rc] = vec[off:off + nc * (rc + 2) * nex * p1 * p1].reshape(nc, rc + 2, nex, p1, p1)[:, 1:-1]
    return out


def halo_schedule(rank: int, nranks: int):
    """Issue order of the NCCL halo exchange of one field (part2d.cu ``halo``):
    ("send", peer, storage row) / ("recv", peer, storage row) with rows counted
    in the partition's storage (0 and rows+1 are the ghost rows).  NCCL pairs
    the k-th send to a peer with that peer's k-th receive from us, so this
    order is correct for 1 (self), 2 (prev == next) and more ranks."""
    prev, next_ = (rank - 1) % nranks, (rank + 1) % nranks
    return [("send", prev, "first"), ("send", next_, "last"), ("recv", next_, "top_ghost"),
            ("recv", prev, "bottom_ghost")]


def bootstrap_id(rank: int, nranks: int, make_id, group=None) -> bytes:
    """Rank 0 makes the 128-byte NCCL unique id, every rank receives it."""
    obj = [make_id() if rank == 0 else None]
    if nranks > 1:
        import torch.distributed as dist
        dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def agree_on_status(bad: int, fails: int, group=None, device=None):
    """Failure flags of a multi-rank partitioned run, agreed over the ranks (the NaN flag
    as an allreduce(min)): the smallest global element index with a non-finite right-hand side (-1:
    none) and the total number of failed implicit solves.  Every rank then raises the same
    ``SolverError`` instead of one rank leaving the others inside a collective.  One rank (or no
    process group): the inputs."""
    try:
        import torch
        import torch.distributed as dist
    except ImportError:   # pragma: no cover
        return bad, fails
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return bad, fails
    big = 2 ** 62
    t = torch.tensor([bad if bad >= 0 else big, -int(fails)], dtype=torch.int64,
                     device=device if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)   # min of -fails = -(max fails); the element index: min
    b, f = int(t[0].item()), -int(t[1].item())
    return (-1 if b >= big else b), f


def raise_on_failure_all(rt, group=None) -> None:
    """``Runtime.raise_on_failure`` with the flags agreed over the ranks of a partitioned run."""
    from ._lib import SolverError
    bad, fails, _ = rt.status()
    bad, fails = agree_on_status(bad, fails, group, rt.device)
    if bad >= 0:
        raise SolverError(f"non-finite right-hand side in element {bad}")
    if fails > 0:
        raise SolverError(f"implicit CG solve did not converge within {rt.maxit} iterations (on some rank)")


@dataclass(frozen=True)
class Partition:
    """Element-row partition of a 2-D mesh.

    ``comm=None``: all ``nranks`` partitions live in this process on one GPU
    (halo exchange and CG allreduce are device copies / fixed-order sums).
    With an :class:`NcclComm` the process owns only partition ``comm.rank``;
    the halo and the CG dot products go through NCCL."""
    nranks: int
    comm: object = None

    @property
    def first_rank(self):
        return 0 if self.comm is None else self.comm.rank

    @property
    def nlocal(self):
        return self.nranks if self.comm is None else 1


class NcclComm:
    """NCCL communicator of the partition layer, bootstrapped through
    torch.distributed (rank 0 makes the unique id, every rank receives it)."""

    def __init__(self, rank: int, nranks: int, device: int = 0, group=None):
        self.rt = get_runtime(device)
        self.lib = self.rt.lib
        self.rank, self.nranks = rank, nranks
        def make_id():
            uid = C.create_string_buffer(128)
            self.rt.check(self.lib.sisdc_nccl_unique_id(uid), "nccl_unique_id")
            return bytes(uid.raw)

        self.group = group   # the torch.distributed group the ranks also agree failures over
        uid = bootstrap_id(rank, nranks, make_id, group)
        h = C.c_void_p()
        self.rt.check(self.lib.sisdc_comm_create(self.rt.h, uid, nranks, rank, C.byref(h)), "comm_create")
        self.h = h

    def __del__(self):
        try:
            self.lib.sisdc_comm_destroy(self.h)
        except Exception:
            pass


class DGOperator2D:
    is2d = True

    def __init__(self, mesh: Mesh2D, problem, penalty_const: float = 2.0, device: int = 0, eager_checks: bool = True,
                 partition: Partition = None, av=None):
        """``av``: ``dgsem.ArtificialViscosityParams(kappa_s, c_s)`` switches on the Persson-Peraire sensor
        (tensor-product generalisation of ``dgsem.py:537-559``; frozen per slab by ``begin_slab``)."""
        self.mesh = mesh
        self.partition = partition
        self.problem = problem
        self.av = av
        self.ncomp = problem.ncomp
        self.p1 = mesh.degree + 1
        self.ndof = self.ncomp * mesh.n_elem * self.p1 * self.p1
        self.rt = get_runtime(device)
        self.lib = self.rt.lib
        self.eager_checks = eager_checks
        d = _lib.Op2DDesc(mesh.nex, mesh.ney, mesh.degree, self.ncomp, _KIND[problem.kind],
                          float(mesh.x_left), float(mesh.x_right), float(mesh.y_bottom), float(mesh.y_top),
                          float(getattr(problem, "gamma", 1.4)), float(problem.nu),
                          float(getattr(problem, "ax", 0.0)), float(getattr(problem, "ay", 0.0)), float(penalty_const),
                          float(getattr(problem, "prandtl", 1.0)))
        self._desc = d
        h = C.c_void_p()
        self.parts = None
        if partition is None:
            self.rt.check(self.lib.sisdc_op2d_create(self.rt.h, C.byref(d), C.byref(h)), "op2d_create")
            self.slab_rows = mesh.ney
        else:
            self._comm = partition.comm   # keeps the communicator alive with the operator
            self.rt.check(self.lib.sisdc_op2d_create_part(
                self.rt.h, C.byref(d), partition.nranks, partition.first_rank, partition.nlocal,
                None if partition.comm is None else partition.comm.h, C.byref(h)), "op2d_create_part")
            k = partition.nlocal
            rb, rc, off, npart = (C.c_int * k)(), (C.c_int * k)(), (C.c_int64 * k)(), C.c_int()
            self.rt.check(self.lib.sisdc_op2d_part_layout(h, k, rb, rc, off, C.byref(npart)), "part_layout")
            self.parts = [(rb[i], rc[i], off[i]) for i in range(npart.value)]
            ranks = range(partition.first_rank, partition.first_rank + partition.nlocal)
            if self.parts != part_layout(mesh.ney, mesh.nex, self.p1, self.ncomp, partition.nranks, ranks):
                raise RuntimeError("library partition layout disagrees with part_layout()")
            self.slab_rows = sum(r + 2 for _, r, _ in self.parts)
            self.ndof = self.ncomp * self.slab_rows * mesh.nex * self.p1 * self.p1
        self.h = h
        self._scratch = None
        self.nu_art = None

    def __del__(self):
        try:
            self.lib.sisdc_op1d_destroy(self.h)
        except Exception:
            pass

    def as_nodes(self, u):
        if self.parts is not None:
            raise ValueError("a partitioned state has ghost rows: use owned_views() / gather()")
        return self.rt.to_device(u).reshape(self.ncomp, self.mesh.ney, self.mesh.nex, self.p1, self.p1)

    # ------------------------------------------------ partitioned layout
    def _part_view(self, vec, i):
        _, rows, off = self.parts[i]
        n = self.ncomp * (rows + 2) * self.mesh.nex * self.p1 * self.p1
        return vec[off:off + n].view(self.ncomp, rows + 2, self.mesh.nex, self.p1, self.p1)

    def owned_views(self, vec):
        """[(first global row, (ncomp, rows, nex, P+1, P+1) view of the owned rows)]"""
        return [(rb, self._part_view(vec, i)[:, 1:-1]) for i, (rb, _, _) in enumerate(self.parts)]

    def scatter(self, u_global):
        """Global state (ncomp, ney, nex, P+1, P+1) -> this process's storage
        vector (ghost rows zero; the operators exchange them before use)."""
        if self.parts is None:
            return self.rt.to_device(u_global).reshape(-1).clone()
        g = np.asarray(u_global.cpu() if hasattr(u_global, "cpu") else u_global, dtype=np.float64)
        g = g.reshape(self.ncomp, self.mesh.ney, self.mesh.nex, self.p1, self.p1)
        return to_storage(g, self.parts, self.rt.zeros(self.ndof))

    def gather(self, vec):
        """Owned rows of this process's partitions -> numpy (ncomp, ney, nex,
        P+1, P+1), rows of other processes' partitions left NaN."""
        if self.parts is None:
            return self.as_nodes(vec).cpu().numpy()
        return from_storage(vec.detach().cpu().numpy(), self.parts,
                            (self.ncomp, self.mesh.ney, self.mesh.nex, self.p1, self.p1))

    def halo_exchange(self, vec, mcount: int = 1, mstride: int = 0, scalar_field: bool = False):
        self.rt.bind_stream()
        self.rt.check(self.lib.sisdc_halo_exchange(self.h, vec.data_ptr(), int(mcount), int(mstride),
                                                   1 if scalar_field else 0), "halo_exchange")

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
            if self.problem.kind == "ns2d":
                raise ValueError("the 'euler' substep scheme needs the (non-SPD) NS viscous operator in the implicit "
                                 "solve; NS2D runs the si1 / si2 schemes")
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

    def apply_viscous(self, u, t: float = 0.0, out=None):
        """NS2D physical viscous term (Stokes stress + heat flux; oracle
        ``Op2D.apply_viscous``): ``sisdc_apply_diffusion`` with the physical
        coefficient kind."""
        if self.problem.kind != "ns2d":
            raise ValueError("apply_viscous is the NS2D viscous operator")
        u = self.rt.to_device(u)
        out = self._out(out)
        self.rt.check(self.lib.sisdc_apply_diffusion(self.h, Coef(_lib.COEF_PHYS, 0.0, None), u.data_ptr(), float(t),
                                                     out.data_ptr()), "apply_viscous")
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
        out = self.rt.empty(self.mesh.nex * self.slab_rows * self.p1 * self.p1)
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

    def _nu_art_buffer(self):
        """One value per element of the storage (ghost rows included on a partition)."""
        return self.rt.zeros(self.slab_rows * self.mesh.nex)

    def persson_viscosity(self, u):
        """Element-wise artificial viscosity of state ``u`` (``dgsem.py:537-559`` on tensor-product
        Legendre modes): (slab_rows * nex,) device tensor, zeros without ``av``."""
        out = self._nu_art_buffer()
        if self.av is None:
            return out
        u = self.rt.to_device(u)
        self.rt.bind_stream()
        self.rt.check(self.lib.sisdc_persson_viscosity(self.h, u.data_ptr(), float(self.av.kappa_s),
                                                       float(self.av.c_s), out.data_ptr()), "persson")
        return out

    def begin_slab(self, u0, t0: float, dt: float) -> None:
        """Freeze per-slab data (``dgsem.py:563-571``): the AV field."""
        if self.av is None:
            return
        if self.nu_art is None:
            self.nu_art = self._nu_art_buffer()
        u0 = self.rt.to_device(u0)
        self.rt.bind_stream()
        self.rt.check(self.lib.sisdc_persson_viscosity(self.h, u0.data_ptr(), float(self.av.kappa_s),
                                                       float(self.av.c_s), self.nu_art.data_ptr()), "persson")
        self.rt.check(self.lib.sisdc_op1d_set_nu_art(self.h, self.nu_art.data_ptr()), "set_nu_art")

    def boundary_at(self, *times):
        """Periodic 2-D meshes carry no trace data."""
