"""Multilevel SDC with FAS coupling, on the GPU (reference ``mlsdc.py``).

Level/Hierarchy/begin_slab/start/v_cycle/fas_rhs/run_mlsdc/integrate_mlsdc
with the reference's semantics (``mlsdc.py:31-254``).  The FAS right-hand side
is two fused launches: ``xfer_fas_restrict`` (fine residual with cached f,
projected solution v = P_t P_sp u_f, restricted residual R_t R_sp r) and the
coarse defect of v with fresh rhs evaluations (``eval_rhs_nodes`` +
``collocation_defect``, ``mlsdc.py:68-77``).  The coarse correction is one
``xfer_interp`` launch (u_f += I_sp I_t (u_c - v)).

Each level keeps two NodalSolution buffers that sweeps alternate between, so
a slab allocates nothing after the first one and ``integrate_mlsdc(...,
graph=True)`` can capture one slab in a CUDA graph and replay it per step.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .trace import traced
from . import _lib
from .collocation import CollocationRule, QuadratureWeights, make_nodes, make_weights
from .sdc import NodalSolution, _alloc, from_nodes, predict, refresh_caches, sweep
from .transfer import SpaceTimeTransfer, _t0, build_temporal_transfer, temporal_core


@dataclass
class Level:
    """One rung of the hierarchy plus its per-slab state (``mlsdc.py:31-43``)."""
    ctx: object
    rule: CollocationRule
    weights: QuadratureWeights
    scheme: str
    u0: Optional[object] = None
    t0: float = 0.0
    sol: Optional[NodalSolution] = None
    g: Optional[object] = None
    v: Optional[object] = None
    _bufs: list = field(default_factory=list, repr=False)
    _work: dict = field(default_factory=dict, repr=False)

    def next_buffer(self) -> NodalSolution:
        """A NodalSolution buffer that is not the current iterate."""
        if not self._bufs:
            n = self.ctx.ndof
            self._bufs = [_alloc(self.ctx, self.ctx.rt.zeros(n), self.rule.M, self.scheme, 0.0) for _ in range(2)]
            # the slab start is the same for every iterate of the level: one shared u0 vector, so a sweep
            # into the other buffer does not copy it (one launch fewer per sweep)
            self._bufs[1].u0 = self._bufs[0].u0
        b = self._bufs[0] if self._bufs[0] is not self.sol else self._bufs[1]
        b.t0 = self.t0
        return b

    def work(self, name, *shape):
        t = self._work.get(name)
        if t is None:
            t = self._work[name] = self.ctx.rt.empty(*shape)
        return t


@dataclass
class Hierarchy:
    """Levels (coarsest first), transfers, cycling parameters (``mlsdc.py:46-65``)."""
    levels: list
    transfers: list
    n_coarse: int = 2
    n_sweep: int = 1
    form: str = "incremental"
    post_sweep_on_finest: bool = True
    presmooth: Optional[Callable] = None

    def __post_init__(self):
        if len(self.transfers) != len(self.levels) - 1:
            raise ValueError("need exactly one transfer per adjacent level pair")
        if self.form not in ("incremental", "nonincremental"):
            raise ValueError(f"unknown sweep form {self.form!r}")
        self.fine_sweeps = 0
        self.coarse_passes = 0

    @property
    def fine(self) -> Level:
        return self.levels[-1]


def fas_residual(level: Level, dt: float, form: str = "incremental"):
    """g - F(u) with the iterate's cached rhs (``mlsdc.py:84-87``)."""
    from .sdc import collocation_defect
    return collocation_defect(level.rule, level.weights, dt, level.sol, form, ctx=level.ctx,
                              sign=-1.0, add=level.g)


@traced("sisdc.fas_rhs")
def fas_rhs(hier: Hierarchy, i: int, dt: float):
    """Compose the FAS right-hand side of level i from level i+1 and store the
    restricted solution v on level i (``mlsdc.py:90-101``)."""
    upper, lower, st = hier.levels[i + 1], hier.levels[i], hier.transfers[i]
    rt = lower.ctx.rt
    rt.bind_stream()
    Mc, n_c = lower.rule.M, lower.ctx.ndof
    v = lower.work("v", Mc, n_c)
    rr = lower.work("rr", Mc, n_c)
    fr = lower.work("f_fresh", Mc, n_c)
    g = lower.work("g", Mc, n_c)
    inc = 1 if hier.form == "incremental" else 0
    Wf = upper.weights.w_nn if inc else upper.weights.w_0n
    wa, wp = _lib.darr(Wf)
    rt.check(rt.lib.sisdc_xfer_fas_restrict(
        st.handle.h, wp, float(dt), inc, upper.sol.u0.data_ptr(), upper.sol.u.data_ptr(), upper.sol.f.data_ptr(),
        None if upper.g is None else upper.g.data_ptr(), v.data_ptr(), rr.data_ptr()), "fas_restrict")
    if _t0(st.temporal):   # nodes_plus_t0: v also carries the slab start, whose spatial projection is lower.u0
        a_p = temporal_core(st.temporal)[3]
        for m in range(Mc):
            rt.lincomb(v[m], (1.0, v[m]), (float(a_p[m]), lower.u0))
    lower.v = v
    # coarse defect of v with fresh rhs at the coarse node times (mlsdc.py:68-77)
    times = lower.t0 + dt * lower.rule.tau
    if getattr(lower.ctx, "dirichlet", False):
        lower.ctx.boundary_at(*times)
    ta, tp = _lib.darr(times)
    rt.check(rt.lib.sisdc_eval_rhs_nodes(lower.ctx.h, Mc, v.data_ptr(), tp, fr.data_ptr()), "eval_rhs_nodes")
    if getattr(lower.ctx, "source_fn", None) is not None:
        for m in range(Mc):
            lower.ctx.add_source(fr[m], v[m], times[m])
    Wc = lower.weights.w_nn if inc else lower.weights.w_0n
    wca, wcp = _lib.darr(Wc)
    rt.check(rt.lib.sisdc_collocation_defect(lower.ctx.h, Mc, wcp, float(dt), inc, lower.u0.data_ptr(), v.data_ptr(),
                                             fr.data_ptr(), 1.0, rr.data_ptr(), g.data_ptr()), "fas_compose")
    return g


@traced("sisdc.sweep_level")
def _sweep_level(hier: Hierarchy, i: int, dt: float, n: int) -> None:
    lv = hier.levels[i]
    for _ in range(n):
        lv.sol = sweep(lv.ctx, lv.rule, lv.weights, dt, lv.scheme, lv.sol, g=lv.g, form=hier.form,
                       out=lv.next_buffer())
        if i == len(hier.levels) - 1:
            hier.fine_sweeps += 1
        elif i == 0:
            hier.coarse_passes += 1


@traced("sisdc.v_cycle")
def v_cycle(hier: Hierarchy, dt: float, top: Optional[int] = None, final: bool = False) -> None:
    """One multigrid cycle over levels[0..top] (``mlsdc.py:110-131``)."""
    if top is None:
        top = len(hier.levels) - 1
    hier.levels[top].g = None
    for i in range(top, 0, -1):
        _sweep_level(hier, i, dt, hier.n_sweep)
        hier.levels[i - 1].g = fas_rhs(hier, i - 1, dt)
    _sweep_level(hier, 0, dt, hier.n_coarse)
    for i in range(1, top + 1):
        lv, below = hier.levels[i], hier.levels[i - 1]
        rt = lv.ctx.rt
        rt.bind_stream()
        # u_f += I_sp I_t (u_c - v)   (mlsdc.py:125-126)
        rt.check(rt.lib.sisdc_xfer_interp(hier.transfers[i - 1].handle.h, 1, below.sol.u.data_ptr(),
                                          below.v.data_ptr(), lv.sol.u.data_ptr()), "correction")
        refresh_caches(lv.ctx, lv.rule, dt, lv.scheme, lv.sol)
        if i < top:
            _sweep_level(hier, i, dt, hier.n_sweep)
    if final and hier.post_sweep_on_finest:
        _sweep_level(hier, top, dt, hier.n_sweep)


def _interp_up(hier: Hierarchy, i: int, dt: float) -> None:
    """Initialise level i+1 from the level-i iterate (``mlsdc.py:134-142``)."""
    lv, up = hier.levels[i], hier.levels[i + 1]
    rt = up.ctx.rt
    buf = up.next_buffer()
    rt.copy(buf.u0, up.u0)
    src = lv.sol.u
    if hier.presmooth is not None:   # mlsdc.py:139-140, e.g. lambda u: smooth_start(coarse_op, u)
        src = lv.work("presmooth", *lv.sol.u.shape)
        for m in range(lv.sol.u.shape[0]):
            rt.copy(src[m], hier.presmooth(lv.sol.u[m]))
    rt.check(rt.lib.sisdc_xfer_interp(hier.transfers[i].handle.h, 0, src.data_ptr(), None,
                                      buf.u.data_ptr()), "interp_solution")
    st = hier.transfers[i]
    if _t0(st.temporal):   # nodes_plus_t0: the coarse slab start rides through the interpolation (mlsdc.py:141)
        st._carry_t0(buf.u, temporal_core(st.temporal)[2], "interp", lv.u0)
    up.sol = from_nodes(up.ctx, up.rule, dt, up.scheme, up.u0, up.t0, buf.u, out=buf)


@traced("sisdc.start")
def start(hier: Hierarchy, strategy: str, dt: float, c_fmg: int = 1) -> None:
    """Initial iterates on every level (``mlsdc.py:145-182``)."""
    L = len(hier.levels)
    for lv in hier.levels:
        lv.g = None
        lv.v = None
    if strategy == "constant":
        for lv in hier.levels:
            buf = lv.next_buffer()
            lv.ctx.rt.copy(buf.u0, lv.u0)
            for m in range(lv.rule.M):
                lv.ctx.rt.copy(buf.u[m], lv.u0)
            lv.sol = from_nodes(lv.ctx, lv.rule, dt, lv.scheme, lv.u0, lv.t0, buf.u, out=buf)
        return
    if strategy == "predictor":
        for lv in hier.levels:
            lv.sol = predict(lv.ctx, lv.rule, dt, lv.scheme, lv.u0, lv.t0, out=lv.next_buffer())
        hier.coarse_passes += 1
        return
    lv0 = hier.levels[0]
    lv0.sol = predict(lv0.ctx, lv0.rule, dt, lv0.scheme, lv0.u0, lv0.t0, out=lv0.next_buffer())
    hier.coarse_passes += 1
    if strategy == "cascade":
        for i in range(L - 1):
            _sweep_level(hier, i, dt, hier.n_sweep)
            _interp_up(hier, i, dt)
        return
    if strategy == "fmg":
        _sweep_level(hier, 0, dt, hier.n_sweep)
        _interp_up(hier, 0, dt)
        for t in range(1, L - 1):
            for _ in range(c_fmg):
                v_cycle(hier, dt, top=t, final=False)
            _interp_up(hier, t, dt)
        return
    raise ValueError(f"unknown start strategy {strategy!r}")


@traced("sisdc.begin_slab")
def begin_slab(hier: Hierarchy, u0_fine, t0: float, dt: float) -> None:
    """Slab-start states on all levels, coarse ones by spatial projection
    (``mlsdc.py:185-200``)."""
    L = len(hier.levels)
    fine = hier.levels[-1]
    rt = fine.ctx.rt
    rt.bind_stream()
    u0f = fine.work("u0", fine.ctx.ndof)
    src = rt.to_device(u0_fine)
    if src.data_ptr() != u0f.data_ptr():
        rt.copy(u0f, src)
    fine.u0 = u0f
    for i in range(L - 2, -1, -1):
        lo, hi = hier.levels[i], hier.levels[i + 1]
        u0c = lo.work("u0", lo.ctx.ndof)
        rt.check(rt.lib.sisdc_xfer_spatial(hier.transfers[i].handle.h, 1, hi.u0.data_ptr(), u0c.data_ptr()),
                 "project u0")
        lo.u0 = u0c
    for lv in hier.levels:
        lv.t0 = t0
        lv.sol = None
        lv.g = None
        lv.v = None
        if hasattr(lv.ctx, "begin_slab"):
            lv.ctx.begin_slab(lv.u0, t0, dt)


@traced("sisdc.run_mlsdc")
def run_mlsdc(hier: Hierarchy, u0_fine, t0: float, dt: float, n_cycles: int, strategy: str = "predictor",
              c_fmg: int = 1, observer: Optional[Callable] = None) -> NodalSolution:
    """One slab: start, n_cycles V-cycles, closing fine sweep (``mlsdc.py:203-234``)."""
    begin_slab(hier, u0_fine, t0, dt)
    start(hier, strategy, dt, c_fmg=c_fmg)
    if observer is not None:
        observer(0, hier.fine.sol)
    for c in range(1, n_cycles + 1):
        v_cycle(hier, dt, final=False)
        if observer is not None:
            snap = hier.fine.sol
            if hier.post_sweep_on_finest:
                lv = hier.fine
                snap = sweep(lv.ctx, lv.rule, lv.weights, dt, lv.scheme, snap, form=hier.form)
            observer(c, snap)
    if hier.post_sweep_on_finest and n_cycles > 0:
        _sweep_level(hier, len(hier.levels) - 1, dt, hier.n_sweep)
    return hier.fine.sol


class SlabGraph:
    """One MLSDC slab captured as a CUDA graph over fixed device buffers.

    ``step()`` replays it: input state in ``self.u`` (device), result written
    back into ``self.u``.  Valid for time-independent operators (periodic,
    source-free problems), where t0 only labels the slab.
    """

    def __init__(self, hier: Hierarchy, u0_fine, t0: float, dt: float, n_cycles: int,
                 strategy: str = "fmg", c_fmg: int = 1):
        import torch
        fine = hier.fine
        if any(getattr(lv.ctx, "dirichlet", False) for lv in hier.levels):
            raise ValueError("time-dependent Dirichlet data cannot be captured into a replayed slab graph")
        if any(getattr(lv.ctx, "source_fn", None) is not None for lv in hier.levels):
            raise ValueError("a host-evaluated source term cannot be captured into a replayed slab graph")
        rt = fine.ctx.rt
        self.rt, self.hier = rt, hier
        self.u = rt.to_device(u0_fine).clone()
        args = (t0, dt, n_cycles, strategy, c_fmg)
        # eager warm-up: allocates every level buffer outside the capture
        sol = run_mlsdc(hier, self.u, *args)
        rt.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        n0 = rt.launch_count()
        stream = torch.cuda.Stream(device=rt.device)
        stream.wait_stream(torch.cuda.current_stream(rt.device))
        with torch.cuda.graph(self.graph, stream=stream):
            sol = run_mlsdc(hier, self.u, *args)
            rt.copy(self.u, sol.u[-1])
        self.kernels_per_step = rt.launch_count() - n0
        rt.bind_stream()
        # the warm-up already advanced one step from u0: restore the input
        self.u.copy_(rt.to_device(u0_fine))
        torch.cuda.current_stream(rt.device).synchronize()

    def step(self):
        self.graph.replay()


def integrate_mlsdc(hier: Hierarchy, u0_fine, t0: float, dt: float, n_steps: int, n_cycles: int,
                    strategy: str = "predictor", c_fmg: int = 1, graph: bool = False):
    """March n_steps slabs (``mlsdc.py:237-254``).  ``graph=True`` captures
    one slab and replays it (time-independent operators only)."""
    rt = hier.fine.ctx.rt
    if graph and n_steps > 0:
        g = SlabGraph(hier, u0_fine, t0, dt, n_cycles, strategy, c_fmg)
        rt.reset_status()
        for _ in range(n_steps):
            g.step()
        _raise_on_failure(hier)
        return g.u
    u = rt.to_device(u0_fine)
    t = t0
    for _ in range(n_steps):
        sol = run_mlsdc(hier, u, t, dt, n_cycles, strategy=strategy, c_fmg=c_fmg)
        u = sol.end_value.clone()
        t += dt
    _raise_on_failure(hier)
    return u


def _raise_on_failure(hier) -> None:
    """Latched device failures -> SolverError; a run partitioned over several ranks agrees on the
    flags first (dgsem2d.raise_on_failure_all), so every rank raises instead of one rank leaving
    the others inside a collective."""
    ctx = hier.fine.ctx
    comm = getattr(getattr(ctx, "partition", None), "comm", None)
    if comm is not None and comm.nranks > 1:
        from .dgsem2d import raise_on_failure_all
        raise_on_failure_all(ctx.rt, comm.group)
    else:
        ctx.rt.raise_on_failure()


def build_p_hierarchy(make_op, degrees, node_counts, scheme: str = "si2", nodes: str = "radau_right",
                      n_coarse: int = 2, n_sweep: int = 1, post_sweep_on_finest: bool = True,
                      restriction: str = None, form: str = "incremental", presmooth=None,
                      node_convention: str = "nodes_only") -> Hierarchy:
    """Hierarchy of p-levels on one mesh as the reference CLI builds it
    (``cli.py:776-815``); ``make_op(degree)`` returns a DGOperator."""
    from .transfer import build_spatial_p_transfer, build_spatial_p_transfer_2d
    ops = [make_op(p) for p in degrees]
    rules = [make_nodes(nodes, M) for M in node_counts]
    levels = [Level(o, r, make_weights(r), scheme) for o, r in zip(ops, rules)]
    transfers = []
    for lo, hi in zip(range(len(ops) - 1), range(1, len(ops))):
        pair = build_temporal_transfer(rules[lo], rules[hi], node_convention=node_convention)
        if getattr(ops[lo], "is2d", False):
            # element slabs in storage order (a partitioned operator's ghost rows included)
            spatial = build_spatial_p_transfer_2d(degrees[lo], degrees[hi], ops[lo].mesh.nex,
                                                  getattr(ops[lo], "slab_rows", ops[lo].mesh.ney),
                                                  ops[lo].ncomp, restriction=restriction or "mass")
        else:
            spatial = build_spatial_p_transfer(degrees[lo], degrees[hi], ops[lo].mesh.n_elem, ops[lo].ncomp,
                                               restriction=restriction or "transpose")
        transfers.append(SpaceTimeTransfer(pair, spatial))
    if presmooth == "smooth_start":   # the reference's interface averaging on the lower level
        from .dgsem import smooth_start
        lo_op = ops[0]
        presmooth = lambda u: smooth_start(lo_op, u)   # noqa: E731
    return Hierarchy(levels, transfers, n_coarse=n_coarse, n_sweep=n_sweep, form=form, presmooth=presmooth,
                     post_sweep_on_finest=post_sweep_on_finest)


def build_hierarchy(make_op, levels, scheme: str = "si2", nodes: str = "radau_right", n_coarse: int = 2,
                    n_sweep: int = 1, post_sweep_on_finest: bool = True, form: str = "incremental",
                    projection: str = "embedded", jump_policy: str = "linear_blend",
                    node_convention: str = "nodes_only") -> Hierarchy:
    """Hierarchy from per-level (n_elem, degree, n_nodes), coarsest first, as
    the reference CLI's ``_build_hierarchy`` (``cli.py:789-815``) builds it:
    h-transfer where the element counts differ (2:1), p-transfer where the
    degrees differ, the identity (time-only coarsening) otherwise.
    ``make_op(n_elem, degree)`` returns a 1-D DGOperator."""
    from .transfer import build_identity_spatial, build_spatial_h_transfer, build_spatial_p_transfer
    ops = [make_op(ne, P) for ne, P, _ in levels]
    rules = [make_nodes(nodes, M) for _, _, M in levels]
    lv = [Level(o, r, make_weights(r), scheme) for o, r in zip(ops, rules)]
    transfers = []
    for lo in range(len(ops) - 1):
        hi = lo + 1
        pair = build_temporal_transfer(rules[lo], rules[hi], projection, node_convention)
        (nc, pc, _), (nf, pf, _) = levels[lo], levels[hi]
        if nc != nf:
            if nf != 2 * nc or pc != pf:
                raise ValueError("h-coarsening fuses two elements of the same degree into one")
            spatial = build_spatial_h_transfer(nc, pc, ops[lo].ncomp, projection, jump_policy)
        elif pc != pf:
            spatial = build_spatial_p_transfer(pc, pf, nc, ops[lo].ncomp, projection)
        else:
            spatial = build_identity_spatial(ops[lo].ndof)
        transfers.append(SpaceTimeTransfer(pair, spatial))
    return Hierarchy(lv, transfers, n_coarse=n_coarse, n_sweep=n_sweep, form=form,
                     post_sweep_on_finest=post_sweep_on_finest)
