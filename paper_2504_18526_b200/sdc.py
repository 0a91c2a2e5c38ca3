"""Deferred-correction sweeps on one time slab, on the GPU (reference ``sdc.py``).

Same functions and semantics as the reference sweeper; every per-node
substep is a short fixed sequence of fused kernels on the context's stream:

    stage_rhs  rhs = u_{m-1} + Q_m (+g_m) + dt_m conv(u_{m-1}) - h1_old[m]   (sdc.py:218,228-235)
    cg         stage = S_m(rhs)                                             (dgsem.py:503-533 -> PCG)
    stage_rhs  rhs = u_{m-1} + Q_m (+g_m) + dt_m conv(stage) - h2_old[m]     (sdc.py:237)
    cg         u_m = S_m(rhs)
    caches     f_m, h1_m, h2_m                                              (sdc.py:77-98)

The semi-implicit coefficient (dt_m/2) A_c(u_{m-1})^2 + A_d is never stored:
the kernels evaluate it from u_{m-1} on the fly.  No host synchronisation
happens inside a sweep, so whole slabs can be captured in a CUDA graph.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .trace import traced
from . import _lib
from ._lib import Coef
from .collocation import CollocationRule, QuadratureWeights

Form = str


@dataclass
class NodalSolution:
    """Slab iterate (``sdc.py:24-52``): device tensors u0 (N), u/f/h1/h2 (M, N)."""
    u0: object
    u: object
    f: object
    h1: object
    h2: Optional[object]
    t0: float

    def copy(self) -> "NodalSolution":
        return NodalSolution(self.u0.clone(), self.u.clone(), self.f.clone(), self.h1.clone(),
                             None if self.h2 is None else self.h2.clone(), self.t0)

    @property
    def end_value(self):
        return self.u[-1]


def _rt(ctx):
    return ctx.rt


def _node_times(rule, dt, t0):
    return t0 + dt * rule.tau


def _dts(rule, dt):
    return dt * np.diff(np.concatenate(([0.0], rule.tau)))


def _alloc(ctx, u0, M: int, scheme: str, t0: float) -> NodalSolution:
    rt = _rt(ctx)
    u0 = rt.to_device(u0)
    n = u0.numel()
    h2 = rt.empty(M, n) if scheme == "si2" else None
    return NodalSolution(u0.clone(), rt.empty(M, n), rt.empty(M, n), rt.empty(M, n), h2, t0)


def _scheme_id(scheme):
    try:
        return _lib.SCHEMES[scheme]
    except KeyError:
        raise ValueError(f"unknown scheme {scheme!r}") from None


def _coef(ctx, scheme, u_prev, dt_m) -> Coef:
    """C_m frozen at u_{m-1}: SI for si1/si2, physical for euler (dgsem.py:356-396)."""
    if scheme == "euler":   # the state matters for systems (A_d(u_b)); scalar kernels ignore it
        return Coef(_lib.COEF_PHYS, 0.0, u_prev.data_ptr())
    return Coef(_lib.COEF_SI, float(dt_m), u_prev.data_ptr())


def _register_times(ctx, t0, times):
    """Dirichlet trace data for the slab's times (no-op on periodic meshes)."""
    if getattr(ctx, "dirichlet", False):
        ctx.boundary_at(t0, *times)


def _caches(ctx, scheme, sol, M, m_first, m_count, dts, conv_prev=None, times=None):
    rt = _rt(ctx)
    arr, p = _lib.darr(dts)
    ta, tp = _lib.darr(times if times is not None else np.zeros(M))
    rt.check(rt.lib.sisdc_node_caches(
        ctx.h, _scheme_id(scheme), M, m_first, m_count, sol.u0.data_ptr(), sol.u.data_ptr(),
        None if conv_prev is None else conv_prev.data_ptr(), p, float(sol.t0), tp,
        sol.f.data_ptr(), sol.h1.data_ptr(), None if sol.h2 is None else sol.h2.data_ptr()), "node_caches")
    if getattr(ctx, "source_fn", None) is not None:   # f += src(x, t_m, u_m), host callable (dgsem.py:343-347)
        for m in range(m_first, m_first + m_count):
            ctx.add_source(sol.f[m], sol.u[m], times[m])


@traced("sisdc.refresh_caches")
def refresh_caches(ctx, rule: CollocationRule, dt: float, scheme: str, sol: NodalSolution) -> None:
    """Rebuild all caches after node values changed outside a sweep
    (``sdc.py:101-119``): one kernel over all M nodes."""
    _rt(ctx).bind_stream()
    times = _node_times(rule, dt, sol.t0)
    _register_times(ctx, sol.t0, times)
    _caches(ctx, scheme, sol, rule.M, 0, rule.M, _dts(rule, dt), times=times)


def _stage(ctx, base, conv_in, dt_m, f_old, w_row, dt, g_m, h_old, rhs, conv_out, t=0.0):
    rt = _rt(ctx)
    M = 0 if f_old is None else f_old.shape[0]
    wa, wp = _lib.darr(w_row if w_row is not None else np.zeros(1))
    rt.check(rt.lib.sisdc_stage_rhs(
        ctx.h, base.data_ptr(), conv_in.data_ptr(), float(dt_m),
        None if f_old is None else f_old.data_ptr(), M, wp if f_old is not None else None, float(dt),
        None if g_m is None else g_m.data_ptr(), None if h_old is None else h_old.data_ptr(), float(t),
        rhs.data_ptr(), None if conv_out is None else conv_out.data_ptr()), "stage_rhs")


@traced("sisdc.solve")
def _solve(ctx, coef: Coef, a, rhs, out, t=0.0):
    rt = _rt(ctx)
    rt.check(rt.lib.sisdc_implicit_solve(ctx.h, coef, float(a), rhs.data_ptr(), float(t), out.data_ptr()),
             "implicit_solve")


@traced("sisdc.stage_solve")
def _stage_solve(ctx, coef: Coef, a, base, conv_in, dt_m, f_old, w_row, dt, g_m, h_old, t_conv, t_solve,
                 rhs, conv_out, out):
    """Stage rhs + implicit solve; on 1-D levels the stage runs inside the CG
    launch (``sisdc_stage_solve``), elsewhere as two calls."""
    rt = _rt(ctx)
    M = 0 if f_old is None else f_old.shape[0]
    wa, wp = _lib.darr(w_row if w_row is not None else np.zeros(1))
    rt.check(rt.lib.sisdc_stage_solve(
        ctx.h, coef, float(a), base.data_ptr(), conv_in.data_ptr(), float(dt_m),
        None if f_old is None else f_old.data_ptr(), M, wp if f_old is not None else None, float(dt),
        None if g_m is None else g_m.data_ptr(), None if h_old is None else h_old.data_ptr(),
        float(t_conv), float(t_solve), rhs.data_ptr(), None if conv_out is None else conv_out.data_ptr(),
        out.data_ptr()), "stage_solve")


def _substep(ctx, scheme, up, dtm, f_old, w_row, dt, g_m, h1_old, h2_old, out, t_prev=0.0, t_m=0.0, conv_out=None):
    """One SI substep into ``out`` (predictor when f_old/h are None):
    conv(u_{m-1}) at t_{m-1}, the solves and conv(stage) at t_m (sdc.py:225-237).
    ``conv_out``: where conv(u_{m-1}) is left (default: the operator's scratch)."""
    s = ctx.scratch()
    if conv_out is not None:
        s = dict(s, conv=conv_out)
    c = _coef(ctx, scheme, up, dtm)
    if scheme in ("euler", "si1"):
        _stage_solve(ctx, c, dtm, up, up, dtm, f_old, w_row, dt, g_m, h1_old, t_prev, t_m, s["rhs"], s["conv"], out)
    elif scheme == "si2":
        _stage_solve(ctx, c, dtm, up, up, dtm, f_old, w_row, dt, g_m, h1_old, t_prev, t_m, s["rhs"], s["conv"],
                     s["stage"])
        _stage_solve(ctx, c, dtm, up, s["stage"], dtm, f_old, w_row, dt, g_m, h2_old, t_m, t_m, s["rhs"], None, out)
    else:
        raise ValueError(f"unknown scheme {scheme!r}")
    return s["conv"]


def _batched_caches(ctx, M, dts) -> bool:
    """Node caches of a whole sweep in ONE launch: the new f / h1 / h2 feed the NEXT sweep only (the
    stages of this sweep read the old iterate's caches), so they can be evaluated after the last node
    from the per-node conv(u_{m-1}) vectors the stage kernels leave behind -- the same kernel and the
    same operands as M single-node launches, bitwise.  1-D levels (launch-latency bound: 2 x (M - 1)
    launches fewer per sweep); 2-D levels fill the GPU per node and keep one scratch vector."""
    return (not getattr(ctx, "is2d", False)) and M > 1 and all(d != 0.0 for d in dts) \
        and getattr(ctx, "source_fn", None) is None


def _conv_all(ctx, M):
    buf = getattr(ctx, "_conv_all", None)
    if buf is None or buf.shape[0] != M:
        buf = _rt(ctx).empty(M, ctx.ndof)
        ctx._conv_all = buf
    return buf


@traced("sisdc.predict")
def predict(ctx, rule, dt, scheme, u0, t0, out: Optional[NodalSolution] = None) -> NodalSolution:
    """0-th iterate by marching the substepper (``sdc.py:122-156``)."""
    _rt(ctx).bind_stream()
    sol = out if out is not None else _alloc(ctx, u0, rule.M, scheme, t0)
    if out is not None:
        _rt(ctx).copy(sol.u0, _rt(ctx).to_device(u0))
        sol.t0 = t0
    dts = _dts(rule, dt)
    times = _node_times(rule, dt, t0)
    _register_times(ctx, t0, times)
    batched = _batched_caches(ctx, rule.M, dts)
    convs = _conv_all(ctx, rule.M) if batched else None
    for m in range(rule.M):
        up = sol.u0 if m == 0 else sol.u[m - 1]
        t_prev = t0 if m == 0 else times[m - 1]
        if dts[m] == 0.0:
            _rt(ctx).copy(sol.u[m], up)
            _caches(ctx, scheme, sol, rule.M, m, 1, dts, times=times)
            continue
        conv = _substep(ctx, scheme, up, dts[m], None, None, 0.0, None, None, None, sol.u[m], t_prev, times[m],
                        conv_out=convs[m] if batched else None)
        if not batched:
            _caches(ctx, scheme, sol, rule.M, m, 1, dts, conv, times=times)
    if batched:
        _caches(ctx, scheme, sol, rule.M, 0, rule.M, dts, convs, times=times)
    return sol


def constant_start(ctx, rule, dt, scheme, u0, t0) -> NodalSolution:
    sol = _alloc(ctx, u0, rule.M, scheme, t0)
    sol.u[:] = sol.u0
    refresh_caches(ctx, rule, dt, scheme, sol)
    return sol


def from_nodes(ctx, rule, dt, scheme, u0, t0, u_nodes, out: Optional[NodalSolution] = None) -> NodalSolution:
    sol = out if out is not None else _alloc(ctx, u0, rule.M, scheme, t0)
    if u_nodes is not sol.u:
        sol.u.copy_(_rt(ctx).to_device(u_nodes))
    refresh_caches(ctx, rule, dt, scheme, sol)
    return sol


@traced("sisdc.sweep")
def sweep(ctx, rule: CollocationRule, weights: QuadratureWeights, dt: float, scheme: str,
          sol: NodalSolution, g=None, form: Form = "incremental",
          out: Optional[NodalSolution] = None) -> NodalSolution:
    """One correction sweep (``sdc.py:190-242``); returns the next iterate."""
    if form == "nonincremental":
        return _sweep_nonincremental(ctx, rule, weights, dt, scheme, sol, g, out)
    if form != "incremental":
        raise ValueError(f"unknown sweep form {form!r}")
    rt = _rt(ctx)
    rt.bind_stream()
    new = out if out is not None else _alloc(ctx, sol.u0, rule.M, scheme, sol.t0)
    if out is not None:
        if new.u0.data_ptr() != sol.u0.data_ptr():   # a level's buffers share one u0 (mlsdc.Level.next_buffer)
            rt.copy(new.u0, sol.u0)
        new.t0 = sol.t0
    dts = _dts(rule, dt)
    times = _node_times(rule, dt, new.t0)
    _register_times(ctx, new.t0, times)
    batched = _batched_caches(ctx, rule.M, dts) and new is not sol
    convs = _conv_all(ctx, rule.M) if batched else None
    for m in range(rule.M):
        up = new.u0 if m == 0 else new.u[m - 1]
        t_prev = new.t0 if m == 0 else times[m - 1]
        gm = None if g is None else g[m]
        if dts[m] == 0.0:
            _stage(ctx, up, up, 0.0, sol.f, weights.w_nn[m], dt, gm, None, new.u[m], None, t_prev)
            _caches(ctx, scheme, new, rule.M, m, 1, dts, times=times)
            continue
        conv = _substep(ctx, scheme, up, dts[m], sol.f, weights.w_nn[m], dt, gm, sol.h1[m],
                        None if sol.h2 is None else sol.h2[m], new.u[m], t_prev, times[m],
                        conv_out=convs[m] if batched else None)
        if not batched:
            _caches(ctx, scheme, new, rule.M, m, 1, dts, conv, times=times)
    if batched:   # one launch: f, h1, h2 of all M nodes from the per-node conv(u_{m-1}) vectors
        _caches(ctx, scheme, new, rule.M, 0, rule.M, dts, convs, times=times)
    return new


def _sweep_nonincremental(ctx, rule, weights, dt, scheme, sol, g, out=None):
    """Non-incremental correction sweep (``sdc.py:245-284``): every node is
    built from u0 plus the zero-to-node quadrature Q0[m] = dt w_0n[m] f and
    the running sum S of the substep differences; the si2 internal stage keeps
    the node-to-node quadrature (with g differenced).  B = u0 + S is carried
    as one device vector; the same fused stage / solve / cache kernels as the
    incremental sweep, plus ``lincomb`` for the S updates."""
    rt = _rt(ctx)
    rt.bind_stream()
    new = out if out is not None else _alloc(ctx, sol.u0, rule.M, scheme, sol.t0)
    if out is not None:
        if new.u0.data_ptr() != sol.u0.data_ptr():   # a level's buffers share one u0 (mlsdc.Level.next_buffer)
            rt.copy(new.u0, sol.u0)
        new.t0 = sol.t0
    dts = _dts(rule, dt)
    times = _node_times(rule, dt, new.t0)
    _register_times(ctx, new.t0, times)
    s = ctx.scratch()
    B = rt.empty(sol.u0.numel())
    rt.copy(B, sol.u0)
    conv_up, conv_st, tmp = rt.empty(B.numel()), rt.empty(B.numel()), rt.empty(B.numel())
    for m in range(rule.M):
        gm = None if g is None else g[m]
        dtm = dts[m]
        t_prev = new.t0 if m == 0 else times[m - 1]
        if dtm == 0.0:
            _stage(ctx, B, B, 0.0, sol.f, weights.w_0n[m], dt, gm, None, new.u[m], None, t_prev)
            _caches(ctx, scheme, new, rule.M, m, 1, dts, times=times)
            continue
        up = new.u0 if m == 0 else new.u[m - 1]
        c = _coef(ctx, scheme, up, dtm)
        if scheme in ("euler", "si1"):
            _stage(ctx, B, up, dtm, sol.f, weights.w_0n[m], dt, gm, sol.h1[m], s["rhs"], conv_up, t_prev)
            _solve(ctx, c, dtm, s["rhs"], new.u[m], times[m])
            _caches(ctx, scheme, new, rule.M, m, 1, dts, conv_up, times=times)
            rt.lincomb(B, (1.0, B), (1.0, new.h1[m]), (-1.0, sol.h1[m]))      # S += h1_new - h1_old
        elif scheme == "si2":
            gnn = None
            if g is not None:
                gnn = g[m] if m == 0 else rt.lincomb(tmp, (1.0, g[m]), (-1.0, g[m - 1]))
            _stage(ctx, up, up, dtm, sol.f, weights.w_nn[m], dt, gnn, sol.h1[m], s["rhs"], conv_up, t_prev)
            _solve(ctx, c, dtm, s["rhs"], s["stage"], times[m])
            _stage(ctx, B, s["stage"], dtm, sol.f, weights.w_0n[m], dt, gm, sol.h2[m], s["rhs"], conv_st, times[m])
            _solve(ctx, c, dtm, s["rhs"], new.u[m], times[m])
            _caches(ctx, scheme, new, rule.M, m, 1, dts, conv_up, times=times)
            # S += dt_m (conv(stage) + D[C] u_m) - h2_old  (sdc.py:281)
            rt.check(rt.lib.sisdc_apply_diffusion(ctx.h, c, new.u[m].data_ptr(), float(times[m]), tmp.data_ptr()),
                     "apply_diffusion")
            rt.lincomb(tmp, (1.0, conv_st), (1.0, tmp))
            rt.lincomb(B, (1.0, B), (dtm, tmp), (-1.0, sol.h2[m]))
        else:
            raise ValueError(f"unknown scheme {scheme!r}")
    return new


def collocation_defect(rule, weights, dt, sol: NodalSolution, form: Form = "incremental", ctx=None,
                       sign: float = 1.0, add=None, out=None):
    """F(u) with the cached rhs (``sdc.py:304-319``)."""
    if ctx is None:
        raise ValueError("the GPU defect needs the level's operator context (ctx=)")
    rt = _rt(ctx)
    rt.bind_stream()
    inc = 1 if form == "incremental" else 0
    W = weights.w_nn if inc else weights.w_0n
    wa, wp = _lib.darr(W)
    if out is None:
        out = rt.empty(*sol.u.shape)
    rt.check(rt.lib.sisdc_collocation_defect(ctx.h, rule.M, wp, float(dt), inc, sol.u0.data_ptr(), sol.u.data_ptr(),
                                             sol.f.data_ptr(), float(sign),
                                             None if add is None else add.data_ptr(), out.data_ptr()),
             "collocation_defect")
    return out


def residual(rule, weights, dt, sol, g=None, form: Form = "incremental", ctx=None):
    """g - F(u) (``sdc.py:287-301``)."""
    return collocation_defect(rule, weights, dt, sol, form, ctx=ctx, sign=-1.0, add=g)


@traced("sisdc.run_sdc")
def run_sdc(ctx, rule, weights, dt, scheme, u0, t0, n_sweeps, form: Form = "incremental",
            start: str = "predictor", observer: Optional[Callable] = None) -> NodalSolution:
    """Predictor (or constant start) plus n_sweeps corrections (``sdc.py:322-354``)."""
    if hasattr(ctx, "begin_slab"):
        ctx.begin_slab(u0, t0, dt)
    if start == "predictor":
        sol = predict(ctx, rule, dt, scheme, u0, t0)
    elif start == "constant":
        sol = constant_start(ctx, rule, dt, scheme, u0, t0)
    else:
        raise ValueError(f"unknown start {start!r}")
    if observer is not None:
        observer(0, sol)
    for k in range(1, n_sweeps + 1):
        sol = sweep(ctx, rule, weights, dt, scheme, sol, form=form)
        if observer is not None:
            observer(k, sol)
    return sol


def integrate_sdc(ctx, rule, weights, scheme, u0, t0, dt, n_steps, n_sweeps, form: Form = "incremental"):
    """March n_steps slabs (``sdc.py:357-376``)."""
    u = ctx.rt.to_device(u0)
    t = t0
    for _ in range(n_steps):
        sol = run_sdc(ctx, rule, weights, dt, scheme, u, t, n_sweeps, form=form)
        u = sol.end_value.clone()
        t += dt
    ctx.rt.raise_on_failure()
    return u
