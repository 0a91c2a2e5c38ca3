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
    if node_convention == "nodes_only":
        src, dst = coarse_rule.tau, fine_rule.tau
    elif node_convention == "nodes_plus_t0":   # t = 0 is a degree of freedom on both sides (transfer.py:77-79)
        src = np.concatenate(([0.0], coarse_rule.tau))
        dst = np.concatenate(([0.0], fine_rule.tau))
    else:
        raise ValueError(f"unknown node convention {node_convention!r}")
    interp = lagrange_matrix(src, dst)
    if projection_kind == "embedded":
        project = lagrange_matrix(dst, src)
    elif projection_kind == "l2":
        project = _l2_project_matrix(dst, src)
    else:
        raise ValueError(f"unknown projection kind {projection_kind!r}")
    return TransferPair(interp, project, interp.T.copy(), "temporal", projection_kind,
                        {"node_convention": node_convention, "M": (coarse_rule.M, fine_rule.M)})


def _t0(pair: TransferPair) -> bool:
    return pair.meta.get("node_convention") == "nodes_plus_t0"


def temporal_core(pair: TransferPair):
    """(interp, project) node-to-node blocks the GPU transfers apply and the
    columns (a_interp, a_project) that carry the slab-start value
    (``transfer.py:98-121``): with nodes_plus_t0 the output node m is
    A[m+1, 0] u0 + sum_j A[m+1, j+1] nodes[j]; restrictions and corrections pad
    t0 with zero, i.e. use the block alone.  nodes_only: the matrices, no columns."""
    if _t0(pair):
        return (np.ascontiguousarray(pair.interp[1:, 1:]), np.ascontiguousarray(pair.project[1:, 1:]),
                np.ascontiguousarray(pair.interp[1:, 0]), np.ascontiguousarray(pair.project[1:, 0]))
    return pair.interp, pair.project, None, None


def apply_temporal(pair: TransferPair, direction: Direction, nodes, u0=None):
    """Apply a temporal pair along the leading (node) axis (``transfer.py:98-121``)
    to host arrays or device tensors; the output keeps node values only."""
    A = pair.matrix(direction)
    is_t = hasattr(nodes, "device") and not isinstance(nodes, np.ndarray)
    if is_t:
        import torch
        A_ = torch.as_tensor(A, dtype=nodes.dtype, device=nodes.device)
        dot = lambda M, x: torch.tensordot(M, x, dims=([1], [0]))   # noqa: E731
        cat, zeros = (lambda a, b: torch.cat((a, b), dim=0)), torch.zeros_like
    else:
        nodes = np.asarray(nodes)
        A_, dot = A, (lambda M, x: np.tensordot(M, x, axes=(1, 0)))
        cat, zeros = (lambda a, b: np.concatenate((a, b), axis=0)), np.zeros_like
    if _t0(pair):
        if direction == "restrict":
            top = zeros(nodes[:1])
        else:
            if u0 is None:
                raise ValueError("nodes_plus_t0 transfers need the source u0")
            top = (u0 if is_t else np.asarray(u0))[None]
        return dot(A_, cat(top, nodes))[1:]
    return dot(A_, nodes)


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


def _legendre_vandermonde(x, n):
    """V[i, k] = P_k(x_i), k < n (three-term recurrence)."""
    x = np.asarray(x, dtype=float)
    V = np.empty((len(x), n))
    V[:, 0] = 1.0
    if n > 1:
        V[:, 1] = x
    for k in range(1, n - 1):
        V[:, k + 1] = ((2 * k + 1) * x * V[:, k] - k * V[:, k - 1]) / (k + 1)
    return V


def _materialise(fn, n_in):
    """Dense matrix of a linear map given as a function of one input vector."""
    cols = [fn(np.eye(n_in)[j]) for j in range(n_in)]
    return np.stack(cols, axis=1)


def build_spatial_h_transfer(ne_coarse: int, p: int, ncomp: int = 1, projection_kind: str = "embedded",
                             jump_policy: str = "linear_blend") -> SpatialTransfer:
    """2:1 element coarsening (the reference's ``transfer.py:248-317``
    semantics): each coarse parent owns two children of the same degree.

    Derived here in the Legendre modal basis of the parent (not from nodal
    Lagrange products): a nodal vector u on the GLL nodes xi has modal
    coefficients c = V^-1 u, V[i, k] = P_k(xi_i).

    * interp: the parent polynomial evaluated at the child nodes, which sit at
      (xi - 1)/2 and (xi + 1)/2 in parent coordinates;
    * embedded projection: the child pair is first made continuous at its
      shared interface by the jump policy -- linear_blend adds J (1 + xi)/4 to
      the left child and subtracts J (1 - xi)/4 from the right one
      (J = u_R(-1) - u_L(+1): ramps vanishing at the parent's outer ends,
      both interface values become the mean), average replaces both interface
      values by their mean -- then every parent node takes the value of the
      child polynomial that covers it (the centre node, for even P, the mean
      of the two interface values);
    * l2 projection: the modal Galerkin projection of the piecewise child
      polynomial, c_k = (2k + 1)/2 int_{-1}^{1} u P_k, exact by Gauss
      quadrature on each half (no jump handling: conservative by construction);
    * restrict = interp^T.

    The map on one child pair is materialised column by column.  On the GPU
    the pair of children is one contiguous 2(P+1)-node block per parent, so
    the p-transfer kernels apply the stacked blocks unchanged."""
    from .collocation import gauss_legendre
    if jump_policy not in ("linear_blend", "average"):
        raise ValueError(f"unknown jump policy {jump_policy!r}")
    if projection_kind not in ("embedded", "l2"):
        raise ValueError(f"unknown projection kind {projection_kind!r}")
    p1 = p + 1
    xi = _gll_reference(p1)
    Vinv = np.linalg.inv(_legendre_vandermonde(xi, p1))

    def evaluate(u, pts):            # the degree-P polynomial with nodal values u at the points pts
        return _legendre_vandermonde(pts, p1) @ (Vinv @ u)

    IL = _materialise(lambda u: evaluate(u, 0.5 * (xi - 1.0)), p1)
    IR = _materialise(lambda u: evaluate(u, 0.5 * (xi + 1.0)), p1)

    def continuous_pair(pair):
        uL, uR = pair[:p1].copy(), pair[p1:].copy()
        if jump_policy == "linear_blend":
            J = uR[0] - uL[-1]
            uL += 0.25 * (1.0 + xi) * J
            uR -= 0.25 * (1.0 - xi) * J
        else:
            mean = 0.5 * (uL[-1] + uR[0])
            uL[-1] = uR[0] = mean
        return uL, uR

    def embedded(pair):
        uL, uR = continuous_pair(pair)
        out = np.empty(p1)
        for i, x in enumerate(xi):
            if x < 0.0:
                out[i] = evaluate(uL, np.array([2.0 * x + 1.0]))[0]
            elif x > 0.0:
                out[i] = evaluate(uR, np.array([2.0 * x - 1.0]))[0]
            else:
                out[i] = 0.5 * (uL[-1] + uR[0])
        return out

    gx, gw = gauss_legendre(p1 + 3)
    scale = 0.5 * (2.0 * np.arange(p1) + 1.0)

    def l2(pair):
        c = np.zeros(p1)
        for half, shift in ((pair[:p1], -0.5), (pair[p1:], 0.5)):
            x = 0.5 * gx + shift                       # quadrature points of this half, parent coordinates
            vals = evaluate(half, gx)                  # the child polynomial there (its own coordinate is gx)
            c += _legendre_vandermonde(x, p1).T @ (0.5 * gw * vals)
        return _legendre_vandermonde(xi, p1) @ (scale * c)

    P = _materialise(embedded if projection_kind == "embedded" else l2, 2 * p1)
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
            It, Pt, _, _ = temporal_core(temporal)
            Mf, Mc = It.shape
        if spatial.kind == "identity":   # same mesh and degree (time-only coarsening): unit blocks per DOF
            Isp = Psp = Rsp = np.ones((1, 1))
        else:
            Isp, Psp, Rsp = spatial.blocks["interp"], spatial.blocks["project"], spatial.blocks["restrict"]
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (It, Pt, Isp, Psp, Rsp)]
        h = C.c_void_p()
        ptrs = [a.ctypes.data_as(_lib.DP) for a in self._keep]
        if spatial.kind == "p2d":   # element slabs of (P+1)^2 nodes, matrices applied in x and y
            rt.check(rt.lib.sisdc_xfer2d_create(rt.h, spatial.ne_fine * spatial.ncomp, spatial.np_coarse,
                                                spatial.np_fine, Mc, Mf, *ptrs, C.byref(h)), "xfer2d_create")
        elif spatial.kind == "identity":
            rt.check(rt.lib.sisdc_xfer_create(rt.h, spatial.ncomp * spatial.ne_fine * spatial.np_fine, 1, 1, Mc, Mf,
                                              *ptrs, C.byref(h)), "xfer_create")
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

    def _carry_t0(self, out, col, direction, u0):
        """nodes_plus_t0: add the slab-start column, out[m] += col[m] * spatial(u0)."""
        if u0 is None:
            raise ValueError("nodes_plus_t0 transfers need the source u0")
        rt = self.handle.rt
        s0 = self.spatial.apply(direction, u0)
        for m in range(out.shape[0]):
            rt.lincomb(out[m], (1.0, out[m]), (float(col[m]), s0))
        return out

    def project_solution(self, u_nodes_f, u0_f=None):
        out = self._down(1, 1, u_nodes_f)
        if _t0(self.temporal):
            self._carry_t0(out, temporal_core(self.temporal)[3], "project", u0_f)
        return out

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
        out = self._up(u_nodes_c)
        if _t0(self.temporal):
            self._carry_t0(out, temporal_core(self.temporal)[2], "interp", u0_c)
        return out
