"""Inter-level transfers in time and space (reference ``transfer.py``).

The dense operator matrices are host-side setup (``build_temporal_transfer``
``:61-96``, ``build_spatial_p_transfer`` ``:213-245``); applying them to
device states runs in the library's element-local transfer kernels, with the
composition order of ``SpaceTimeTransfer`` (``:324-352``): fine->coarse
spatial first, coarse->fine temporal first.  Built: embedded projection,
nodes_only convention, p-coarsening on a fixed mesh (every BASELINE config).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .collocation import CollocationRule, gauss_legendre, lagrange_matrix, make_nodes
from .runtime import get_runtime

Direction = str


@dataclass(frozen=True)
class TransferPair:
    """Dense operator triple for one axis (``transfer.py:27-45``)."""
    interp: np.ndarray
    project: np.ndarray
    restrict: np.ndarray
    axis: str
    projection_kind: str
    meta: dict

    def matrix(self, direction: Direction) -> np.ndarray:
        if direction not in ("interp", "project", "restrict"):
            raise ValueError(f"unknown direction {direction!r}")
        return getattr(self, direction)


def _l2_project_matrix(src, dst, domain=(0.0, 1.0)) -> np.ndarray:
    a, b = domain
    gx, gw = gauss_legendre(len(src) + 3)
    pts = 0.5 * (b - a) * gx + 0.5 * (a + b)
    wts = 0.5 * (b - a) * gw
    Ld, Ls = lagrange_matrix(dst, pts), lagrange_matrix(src, pts)
    return np.linalg.solve(Ld.T @ (wts[:, None] * Ld), Ld.T @ (wts[:, None] * Ls))


def build_temporal_transfer(coarse_rule: CollocationRule, fine_rule: CollocationRule,
                            projection_kind: str = "embedded", node_convention: str = "nodes_only") -> TransferPair:
    if coarse_rule.M > fine_rule.M:
        raise ValueError("coarse rule must not have more nodes than the fine one")
    if node_convention != "nodes_only":
        raise NotImplementedError("the GPU path builds the nodes_only convention (the reference default)")
    src, dst = coarse_rule.tau, fine_rule.tau
    interp = lagrange_matrix(src, dst)
    if projection_kind == "embedded":
        project = lagrange_matrix(dst, src)
    elif projection_kind == "l2":
        project = _l2_project_matrix(dst, src)
    else:
        raise ValueError(f"unknown projection kind {projection_kind!r}")
    return TransferPair(interp, project, interp.T.copy(), "temporal", projection_kind,
                        {"node_convention": node_convention, "M": (coarse_rule.M, fine_rule.M)})


def _gll_reference(n: int) -> np.ndarray:
    return 2.0 * make_nodes("lobatto", n).tau - 1.0


@dataclass
class SpatialTransfer:
    """Per-element p-transfer blocks (``transfer.py:129-203``); GPU apply."""
    kind: str
    ncomp: int
    ne_coarse: int
    ne_fine: int
    np_coarse: int
    np_fine: int
    blocks: dict
    projection_kind: str
    jump_policy: Optional[str] = None

    def apply(self, direction: Direction, u_flat):
        """Apply to one device state (``transfer.py:149-163``)."""
        rt = get_runtime()
        u = rt.to_device(u_flat)
        if self.kind == "identity":
            return u.clone()
        h = _xfer_handle(self, None)
        dirn = {"interp": 0, "project": 1, "restrict": 2}[direction]
        npn = self.np_fine if dirn == 0 else self.np_coarse
        if self.kind == "h" and dirn == 0:
            npn = 2 * self.np_fine      # a parent's child pair
        out = rt.empty(self.ncomp * self.ne_coarse * (npn * npn if self.kind == "p2d" else npn))
        rt.bind_stream()
        rt.check(rt.lib.sisdc_xfer_spatial(h.h, dirn, u.data_ptr(), out.data_ptr()), "xfer_spatial")
        return out


def mass_consistent_restriction(p_coarse: int, p_fine: int) -> np.ndarray:
    """R = M_c^-1 I^T M_f with the GLL (lumped) masses: rows sum to exactly 1,
    so a constant nodal residual restricts to itself.  The reference's
    R = I^T (``transfer.py:243``) has row sums 1.2-2.3 on GLL p-hierarchies
    (P 7->3: 1.69/2.31), which over-injects the FAS residual every V-cycle;
    on BASELINE cfg2 it makes the reference diverge with >= 4 cycles and on the
    2-D P 7->3 hierarchy with any cycle count."""
    from .collocation import gauss_lobatto
    xc, wc = gauss_lobatto(p_coarse + 1)
    xf, wf = gauss_lobatto(p_fine + 1)
    I = lagrange_matrix(xc, xf)
    return (1.0 / wc)[:, None] * I.T * wf[None, :]


def build_spatial_p_transfer(p_coarse: int, p_fine: int, n_elem: int, ncomp: int = 1,
                             projection_kind: str = "embedded", restriction: str = "transpose") -> SpatialTransfer:
    if p_coarse > p_fine:
        raise ValueError("coarse degree must not exceed fine degree")
    if p_coarse == p_fine:
        return SpatialTransfer("identity", ncomp, n_elem, n_elem, p_coarse + 1, p_fine + 1, {}, "embedded")
    xc, xf = _gll_reference(p_coarse + 1), _gll_reference(p_fine + 1)
    interp = lagrange_matrix(xc, xf)
    if projection_kind == "embedded":
        project = lagrange_matrix(xf, xc)
    elif projection_kind == "l2":
        project = _l2_project_matrix(xf, xc, domain=(-1.0, 1.0))
    else:
        raise ValueError(f"unknown projection kind {projection_kind!r}")
    if restriction == "transpose":
        restrict = interp.T.copy()          # the reference (transfer.py:243)
    elif restriction == "mass":
        restrict = mass_consistent_restriction(p_coarse, p_fine)
    else:
        raise ValueError(f"unknown restriction {restriction!r}")
    return SpatialTransfer("p", ncomp, n_elem, n_elem, p_coarse + 1, p_fine + 1,
                           {"interp": interp, "project": project, "restrict": restrict}, projection_kind)


def build_spatial_h_transfer(ne_coarse: int, p: int, ncomp: int = 1, projection_kind: str = "embedded",
                             jump_policy: str = "linear_blend") -> SpatialTransfer:
    """2:1 element coarsening (``transfer.py:248-317``): each coarse parent owns
    two children.  Interpolation evaluates the parent on each child half;
    the embedded projection evaluates each child on its half of the parent
    (averaging at the centre node) after a jump preprocessor on the child
    pair (linear_blend: ramps removing the interface jump; average: mean of
    the two interface values); the l2 projection is the Galerkin projection of
    the piecewise child data.  On the GPU the pair of children is one
    contiguous 2(P+1)-node block per parent, so the p-transfer kernels apply
    the stacked blocks unchanged."""
    from .collocation import gauss_legendre
    p1 = p + 1
    xi = _gll_reference(p1)
    IL = lagrange_matrix(xi, 0.5 * (xi - 1.0))
    IR = lagrange_matrix(xi, 0.5 * (xi + 1.0))
    B = np.eye(2 * p1)
    if jump_policy == "linear_blend":
        d = np.zeros(2 * p1)
        d[p1] = 1.0
        d[p1 - 1] = -1.0
        B[:p1] += np.outer(0.25 * (1.0 + xi), d)
        B[p1:] -= np.outer(0.25 * (1.0 - xi), d)
    elif jump_policy == "average":
        B[p1 - 1] = 0.0
        B[p1 - 1, p1 - 1] = B[p1 - 1, p1] = 0.5
        B[p1] = B[p1 - 1]
    else:
        raise ValueError(f"unknown jump policy {jump_policy!r}")
    if projection_kind == "embedded":
        E = np.zeros((p1, 2 * p1))
        for i, x in enumerate(xi):
            if x < 0.0:
                E[i, :p1] = lagrange_matrix(xi, np.array([2.0 * x + 1.0]))[0]
            elif x > 0.0:
                E[i, p1:] = lagrange_matrix(xi, np.array([2.0 * x - 1.0]))[0]
            else:
                E[i, p1 - 1] = E[i, p1] = 0.5
        P = E @ B
    elif projection_kind == "l2":
        gx, gw = gauss_legendre(p1 + 3)
        Lp = lagrange_matrix(xi, gx)
        G = Lp.T @ (gw[:, None] * Lp)
        BL = lagrange_matrix(xi, 0.5 * gx - 0.5).T @ (0.5 * gw[:, None] * lagrange_matrix(xi, gx))
        BR = lagrange_matrix(xi, 0.5 * gx + 0.5).T @ (0.5 * gw[:, None] * lagrange_matrix(xi, gx))
        Gi = np.linalg.inv(G)
        P = np.concatenate((Gi @ BL, Gi @ BR), axis=1)
    else:
        raise ValueError(f"unknown projection kind {projection_kind!r}")
    interp = np.concatenate((IL, IR), axis=0)          # (2 p1, p1): parent -> child pair
    return SpatialTransfer("h", ncomp, ne_coarse, 2 * ne_coarse, p1, p1,
                           {"interp_lr": np.stack((IL, IR)), "project_lr": (P[:, :p1], P[:, p1:]),
                            "interp": interp, "project": P, "restrict": interp.T.copy()},
                           projection_kind, jump_policy)


class _XferHandle:
    def __init__(self, spatial: SpatialTransfer, temporal: Optional[TransferPair]):
        rt = get_runtime()
        self.rt = rt
        if temporal is None:
            It = Pt = np.ones((1, 1))
            Mc = Mf = 1
        else:
            It, Pt = temporal.interp, temporal.project
            Mf, Mc = It.shape
        Isp, Psp, Rsp = spatial.blocks["interp"], spatial.blocks["project"], spatial.blocks["restrict"]
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (It, Pt, Isp, Psp, Rsp)]
        h = C.c_void_p()
        ptrs = [a.ctypes.data_as(_lib.DP) for a in self._keep]
        if spatial.kind == "p2d":   # element slabs of (P+1)^2 nodes, matrices applied in x and y
            rt.check(rt.lib.sisdc_xfer2d_create(rt.h, spatial.ne_fine * spatial.ncomp, spatial.np_coarse,
                                                spatial.np_fine, Mc, Mf, *ptrs, C.byref(h)), "xfer2d_create")
        elif spatial.kind == "h":   # parent element <-> contiguous child pair of 2 (P+1) nodes
            rt.check(rt.lib.sisdc_xfer_create(rt.h, spatial.ne_coarse * spatial.ncomp, spatial.np_coarse,
                                              2 * spatial.np_fine, Mc, Mf,
                                              *ptrs, C.byref(h)), "xfer_create")
        else:
            # (ncomp, n_elem, P+1): the component blocks are element-local transfers too
            rt.check(rt.lib.sisdc_xfer_create(rt.h, spatial.ne_fine * spatial.ncomp, spatial.np_coarse,
                                              spatial.np_fine, Mc, Mf,
                                              *ptrs, C.byref(h)), "xfer_create")
        self.h = h
        self.Mc, self.Mf = Mc, Mf

    def __del__(self):
        try:
            self.rt.lib.sisdc_xfer_destroy(self.h)
        except Exception:
            pass


def _xfer_handle(spatial: SpatialTransfer, temporal: Optional[TransferPair]) -> _XferHandle:
    key = "_xh_t" if temporal is not None else "_xh_s"
    owner = temporal if temporal is not None else spatial
    h = getattr(spatial, key, None)
    if h is None or getattr(h, "_temporal", None) is not temporal:
        h = _XferHandle(spatial, temporal)
        h._temporal = temporal
        setattr(spatial, key, h)
    return h


def build_spatial_p_transfer_2d(p_coarse: int, p_fine: int, nex: int, ney: int, ncomp: int = 1,
                                restriction: str = "mass") -> SpatialTransfer:
    """Tensor-product p-transfer on a fixed 2-D mesh: the 1-D GLL Lagrange
    blocks of ``transfer.py:213-245`` applied along x and along y; the 2-D
    formulation restricts residuals mass-consistently by default."""
    one = build_spatial_p_transfer(p_coarse, p_fine, 1, restriction=restriction)
    if one.kind == "identity":
        return SpatialTransfer("identity", ncomp, nex * ney, nex * ney, p_coarse + 1, p_fine + 1, {}, "embedded")
    return SpatialTransfer("p2d", ncomp, nex * ney, nex * ney, p_coarse + 1, p_fine + 1, one.blocks, "embedded")


def build_identity_spatial(ndof: int) -> SpatialTransfer:
    return SpatialTransfer("identity", 1, 1, 1, ndof, ndof, {}, "embedded")


@dataclass(frozen=True)
class SpaceTimeTransfer:
    """Tensor composition of a temporal and a spatial pair (``transfer.py:324-352``)."""
    temporal: TransferPair
    spatial: SpatialTransfer

    @property
    def handle(self) -> _XferHandle:
        if self.spatial.kind not in ("p", "p2d", "h"):
            raise NotImplementedError("identity spatial transfers have no GPU handle")
        return _xfer_handle(self.spatial, self.temporal)

    def _down(self, sdir, tdir, nodes):
        h = self.handle
        rt = h.rt
        x = rt.to_device(nodes)
        out = rt.empty(h.Mc, self.spatial.ncomp * self.spatial.ne_coarse * self._nodes(self.spatial.np_coarse))
        rt.bind_stream()
        rt.check(rt.lib.sisdc_xfer_down(h.h, sdir, tdir, x.data_ptr(), out.data_ptr()), "xfer_down")
        return out

    def _nodes(self, npe):
        return npe * npe if self.spatial.kind == "p2d" else npe

    def project_solution(self, u_nodes_f, u0_f=None):
        return self._down(1, 1, u_nodes_f)

    def restrict_residual(self, r_nodes_f):
        return self._down(2, 2, r_nodes_f)

    def _up(self, nodes_c, sub=None, out=None, accumulate=False):
        h = self.handle
        rt = h.rt
        uc = rt.to_device(nodes_c)
        if out is None:
            out = rt.empty(h.Mf, self.spatial.ncomp * self.spatial.ne_fine * self._nodes(self.spatial.np_fine))
        rt.bind_stream()
        rt.check(rt.lib.sisdc_xfer_interp(h.h, int(accumulate), uc.data_ptr(),
                                          None if sub is None else sub.data_ptr(), out.data_ptr()), "xfer_interp")
        return out

    def interp_correction(self, d_nodes_c):
        return self._up(d_nodes_c)

    def interp_solution(self, u_nodes_c, u0_c=None):
        return self._up(u_nodes_c)
