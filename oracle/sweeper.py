"""SDC sweeps, space-time transfers and the FAS multilevel cycle (oracle).

Restates ``sdc.py`` (NodalSolution, predict, incremental/non-incremental
sweeps, caches, collocation defect), ``transfer.py`` (temporal and spatial
p-transfers, SpaceTimeTransfer) and ``mlsdc.py`` (Level/Hierarchy, begin_slab,
start strategies, V-cycle, FAS right-hand side, run/integrate).  Works with any
context exposing the ``OperatorContext`` methods (``integrators.py:29-60``),
here ``oracle.dg1d.Op1D``.  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import quad


# ------------------------------------------------------------------ rules
@dataclass
class Rule:
    """Collocation rule + weights (``collocation.py:83-107,215-217``)."""
    kind: str
    M: int
    tau: np.ndarray = None
    w_nn: np.ndarray = None
    w_0n: np.ndarray = None

    def __post_init__(self):
        if self.tau is None:
            self.tau = quad.make_tau(self.kind, self.M)
        self.w_nn = quad.weights_nn(self.tau)
        self.w_0n = quad.weights_0n(self.w_nn)

    def sub_dts(self, dt):
        """``sdc.py:59-61``."""
        return dt * np.diff(np.concatenate([[0.0], self.tau]))


@dataclass
class Slab:
    """``sdc.NodalSolution`` (``sdc.py:24-52``)."""
    u0: np.ndarray
    u: np.ndarray
    f: np.ndarray
    h1: np.ndarray
    h2: Optional[np.ndarray]
    t0: float

    @staticmethod
    def empty(u0, M, scheme, t0):
        z = lambda: np.zeros((M,) + u0.shape)
        return Slab(u0.copy(), z(), z(), z(), z() if scheme == "si2" else None, t0)


def _caches(ctx, scheme, s, m, dtm, tm, coeff, conv_prev):
    """``sdc.py:77-98``."""
    s.f[m] = ctx.eval_rhs(s.u[m], tm)
    if dtm == 0.0:
        s.h1[m] = 0.0
        if s.h2 is not None:
            s.h2[m] = 0.0
        return
    dm = ctx.apply_diffusion(coeff, s.u[m], tm)
    s.h1[m] = dtm * (conv_prev + dm)
    if s.h2 is not None:
        s.h2[m] = dtm * (ctx.apply_convection(s.u[m], tm) + dm)


def refresh(ctx, rule, dt, scheme, s):
    """``sdc.py:101-119``."""
    times = s.t0 + dt * rule.tau
    dts = rule.sub_dts(dt)
    for m in range(rule.M):
        up = s.u0 if m == 0 else s.u[m - 1]
        tp = s.t0 if m == 0 else times[m - 1]
        if dts[m] == 0.0:
            _caches(ctx, scheme, s, m, 0.0, times[m], None, None)
            continue
        c = ctx.modified_coeff(up, dts[m], scheme)
        _caches(ctx, scheme, s, m, dts[m], times[m], c, ctx.apply_convection(up, tp))


def predict(ctx, rule, dt, scheme, u0, t0):
    """``sdc.py:122-156``."""
    s = Slab.empty(np.asarray(u0), rule.M, scheme, t0)
    times = t0 + dt * rule.tau
    dts = rule.sub_dts(dt)
    for m in range(rule.M):
        up = s.u0 if m == 0 else s.u[m - 1]
        tp = t0 if m == 0 else times[m - 1]
        dtm = dts[m]
        if dtm == 0.0:
            s.u[m] = up
            _caches(ctx, scheme, s, m, 0.0, times[m], None, None)
            continue
        c = ctx.modified_coeff(up, dtm, scheme)
        cp = ctx.apply_convection(up, tp)
        x = ctx.implicit_solve(c, dtm, up + dtm * cp, times[m])
        if scheme == "si2":
            x = ctx.implicit_solve(c, dtm, up + dtm * ctx.apply_convection(x, times[m]), times[m])
        elif scheme not in ("euler", "si1"):
            raise ValueError(scheme)
        s.u[m] = x
        _caches(ctx, scheme, s, m, dtm, times[m], c, cp)
    return s


def from_nodes(ctx, rule, dt, scheme, u0, t0, u_nodes):
    """``sdc.py:159-187`` (constant_start is from_nodes with u0 copies)."""
    s = Slab.empty(np.asarray(u0), rule.M, scheme, t0)
    s.u[:] = u_nodes
    refresh(ctx, rule, dt, scheme, s)
    return s


def sweep(ctx, rule, dt, scheme, old, g=None, form="incremental"):
    """``sdc.py:190-284``."""
    new = Slab.empty(old.u0, rule.M, scheme, old.t0)
    times = old.t0 + dt * rule.tau
    dts = rule.sub_dts(dt)
    if form == "incremental":
        Q = dt * np.tensordot(rule.w_nn, old.f, axes=(1, 0))
        for m in range(rule.M):
            up = new.u0 if m == 0 else new.u[m - 1]
            tp = new.t0 if m == 0 else times[m - 1]
            q = Q[m] if g is None else Q[m] + g[m]
            dtm = dts[m]
            if dtm == 0.0:
                new.u[m] = up + q
                _caches(ctx, scheme, new, m, 0.0, times[m], None, None)
                continue
            c = ctx.modified_coeff(up, dtm, scheme)
            cp = ctx.apply_convection(up, tp)
            if scheme in ("euler", "si1"):
                new.u[m] = ctx.implicit_solve(c, dtm, up + q + dtm * cp - old.h1[m], times[m])
            elif scheme == "si2":
                st = ctx.implicit_solve(c, dtm, up + q + dtm * cp - old.h1[m], times[m])
                new.u[m] = ctx.implicit_solve(
                    c, dtm, up + q + dtm * ctx.apply_convection(st, times[m]) - old.h2[m], times[m])
            else:
                raise ValueError(scheme)
            _caches(ctx, scheme, new, m, dtm, times[m], c, cp)
        return new
    if form != "nonincremental":
        raise ValueError(form)
    Q0 = dt * np.tensordot(rule.w_0n, old.f, axes=(1, 0))
    if scheme == "si2":
        Qnn = dt * np.tensordot(rule.w_nn, old.f, axes=(1, 0))
        gnn = None if g is None else np.diff(g, axis=0, prepend=np.zeros_like(g[:1]))
    S = np.zeros_like(old.u0)
    for m in range(rule.M):
        base = old.u0 + Q0[m] + S if g is None else old.u0 + Q0[m] + g[m] + S
        dtm = dts[m]
        if dtm == 0.0:
            new.u[m] = base
            _caches(ctx, scheme, new, m, 0.0, times[m], None, None)
            continue
        up = new.u0 if m == 0 else new.u[m - 1]
        tp = new.t0 if m == 0 else times[m - 1]
        c = ctx.modified_coeff(up, dtm, scheme)
        cp = ctx.apply_convection(up, tp)
        if scheme in ("euler", "si1"):
            new.u[m] = ctx.implicit_solve(c, dtm, base + dtm * cp - old.h1[m], times[m])
            _caches(ctx, scheme, new, m, dtm, times[m], c, cp)
            S = S + (new.h1[m] - old.h1[m])
        else:
            qs = Qnn[m] if gnn is None else Qnn[m] + gnn[m]
            st = ctx.implicit_solve(c, dtm, up + qs + dtm * cp - old.h1[m], times[m])
            cs = ctx.apply_convection(st, times[m])
            new.u[m] = ctx.implicit_solve(c, dtm, base + dtm * cs - old.h2[m], times[m])
            _caches(ctx, scheme, new, m, dtm, times[m], c, cp)
            S = S + (dtm * (cs + ctx.apply_diffusion(c, new.u[m], times[m])) - old.h2[m])
    return new


def defect(rule, dt, s, form="incremental"):
    """``sdc.py:304-319``."""
    if form == "incremental":
        Q = dt * np.tensordot(rule.w_nn, s.f, axes=(1, 0))
        prev = np.concatenate([s.u0[None], s.u[:-1]], axis=0)
        return s.u - prev - Q
    return s.u - s.u0[None] - dt * np.tensordot(rule.w_0n, s.f, axes=(1, 0))


def run_sdc(ctx, rule, dt, scheme, u0, t0, n_sweeps, form="incremental"):
    """``sdc.py:322-354`` (predictor start)."""
    ctx.begin_slab(np.asarray(u0), t0, dt)
    s = predict(ctx, rule, dt, scheme, u0, t0)
    for _ in range(n_sweeps):
        s = sweep(ctx, rule, dt, scheme, s, form=form)
    return s


# --------------------------------------------------------------- transfers
class PTransfer:
    """Spatial p-transfer per element on GLL nodes (``transfer.py:213-245``)
    composed with the temporal Lagrange transfer (``transfer.py:61-121``) as
    in ``SpaceTimeTransfer`` (``transfer.py:324-352``); embedded projection,
    nodes_only convention."""

    def __init__(self, ctx_c, ctx_f, rule_c, rule_f, t0=False):
        self.nc, self.ne = ctx_f.nc, ctx_f.ne
        self.pc, self.pf = ctx_c.p1, ctx_f.p1
        xc, xf = quad.gll(self.pc)[0], quad.gll(self.pf)[0]
        self.Isp = quad.lagrange(xc, xf)
        self.Psp = quad.lagrange(xf, xc)
        # nodes_plus_t0 (transfer.py:77-79, 98-121): t = 0 joins both node sets; interp / project carry
        # the source level's slab start through column 0, restrictions and corrections pad it with zero
        self.t0 = bool(t0)
        tc = np.concatenate(([0.0], rule_c.tau)) if t0 else rule_c.tau
        tf = np.concatenate(([0.0], rule_f.tau)) if t0 else rule_f.tau
        self.It = quad.lagrange(tc, tf)
        self.Pt = quad.lagrange(tf, tc)

    def sp(self, A, u, n_in):
        return np.einsum("ij,cej->cei", A, u.reshape(self.nc, self.ne, n_in)).reshape(-1)

    def project_u0(self, u0f):
        return self.sp(self.Psp, u0f, self.pf)

    def _tm(self, A, nodes, top):
        if not self.t0:
            return np.tensordot(A, nodes, axes=(1, 0))
        top = np.zeros_like(nodes[0]) if top is None else top
        return np.tensordot(A, np.concatenate((top[None], nodes), axis=0), axes=(1, 0))[1:]

    def project_solution(self, uf, u0f=None):
        s = np.stack([self.sp(self.Psp, x, self.pf) for x in uf])
        return self._tm(self.Pt, s, None if u0f is None else self.sp(self.Psp, u0f, self.pf))

    def restrict_residual(self, rf):
        s = np.stack([self.sp(self.Isp.T, x, self.pf) for x in rf])
        return self._tm(self.It.T, s, None)

    def interp(self, dc, u0c=None):
        """Corrections: t0 carries zero (u0c None); solutions: the coarse slab start."""
        t = self._tm(self.It, dc, u0c)
        return np.stack([self.sp(self.Isp, x, self.pc) for x in t])


# -------------------------------------------------------------- multilevel
@dataclass
class Lev:
    """``mlsdc.Level`` (``mlsdc.py:31-43``)."""
    ctx: object
    rule: Rule
    scheme: str = "si2"
    u0: Optional[np.ndarray] = None
    t0: float = 0.0
    sol: Optional[Slab] = None
    g: Optional[np.ndarray] = None
    v: Optional[np.ndarray] = None


@dataclass
class Hier:
    """``mlsdc.Hierarchy`` (``mlsdc.py:46-65``), levels coarsest first."""
    levels: list
    transfers: list
    n_coarse: int = 2
    n_sweep: int = 1
    form: str = "incremental"
    post_sweep: bool = True
    fine_sweeps: int = 0
    coarse_passes: int = 0


def _defect_state(lv, un, dt, form):
    """``mlsdc.py:68-77``: fresh rhs evaluations at the level's node times."""
    times = lv.t0 + dt * lv.rule.tau
    f = np.stack([lv.ctx.eval_rhs(un[m], times[m]) for m in range(lv.rule.M)])
    if form == "incremental":
        prev = np.concatenate([lv.u0[None], un[:-1]], axis=0)
        return un - prev - dt * np.tensordot(lv.rule.w_nn, f, axes=(1, 0))
    return un - lv.u0[None] - dt * np.tensordot(lv.rule.w_0n, f, axes=(1, 0))


def fas_rhs(h, i, dt):
    """``mlsdc.py:84-101``."""
    up, lo, st = h.levels[i + 1], h.levels[i], h.transfers[i]
    F = defect(up.rule, dt, up.sol, h.form)
    r = -F if up.g is None else up.g - F
    v = st.project_solution(up.sol.u, up.u0) if getattr(st, "t0", False) else st.project_solution(up.sol.u)
    lo.v = v
    return _defect_state(lo, v, dt, h.form) + st.restrict_residual(r)


def _sweep_level(h, i, dt, n):
    lv = h.levels[i]
    for _ in range(n):
        lv.sol = sweep(lv.ctx, lv.rule, dt, lv.scheme, lv.sol, g=lv.g, form=h.form)
        if i == len(h.levels) - 1:
            h.fine_sweeps += 1
        elif i == 0:
            h.coarse_passes += 1


def v_cycle(h, dt, top=None, final=False):
    """``mlsdc.py:110-131``."""
    if top is None:
        top = len(h.levels) - 1
    h.levels[top].g = None
    for i in range(top, 0, -1):
        _sweep_level(h, i, dt, h.n_sweep)
        h.levels[i - 1].g = fas_rhs(h, i - 1, dt)
    _sweep_level(h, 0, dt, h.n_coarse)
    for i in range(1, top + 1):
        lv, lo = h.levels[i], h.levels[i - 1]
        lv.sol.u = lv.sol.u + h.transfers[i - 1].interp(lo.sol.u - lo.v)
        refresh(lv.ctx, lv.rule, dt, lv.scheme, lv.sol)
        if i < top:
            _sweep_level(h, i, dt, h.n_sweep)
    if final and h.post_sweep:
        _sweep_level(h, top, dt, h.n_sweep)


def _interp_up(h, i, dt):
    """``mlsdc.py:134-142`` (no presmoother)."""
    lv, up = h.levels[i], h.levels[i + 1]
    st = h.transfers[i]
    fine = st.interp(lv.sol.u, lv.u0) if getattr(st, "t0", False) else st.interp(lv.sol.u)
    up.sol = from_nodes(up.ctx, up.rule, dt, up.scheme, up.u0, up.t0, fine)


def start(h, strategy, dt, c_fmg=1):
    """``mlsdc.py:145-182``."""
    for lv in h.levels:
        lv.g = lv.v = None
    L = len(h.levels)
    if strategy == "predictor":
        for lv in h.levels:
            lv.sol = predict(lv.ctx, lv.rule, dt, lv.scheme, lv.u0, lv.t0)
        h.coarse_passes += 1
        return
    if strategy == "constant":
        for lv in h.levels:
            lv.sol = from_nodes(lv.ctx, lv.rule, dt, lv.scheme, lv.u0, lv.t0,
                                np.broadcast_to(lv.u0, (lv.rule.M,) + lv.u0.shape))
        return
    lv0 = h.levels[0]
    lv0.sol = predict(lv0.ctx, lv0.rule, dt, lv0.scheme, lv0.u0, lv0.t0)
    h.coarse_passes += 1
    if strategy == "cascade":
        for i in range(L - 1):
            _sweep_level(h, i, dt, h.n_sweep)
            _interp_up(h, i, dt)
        return
    if strategy == "fmg":
        _sweep_level(h, 0, dt, h.n_sweep)
        _interp_up(h, 0, dt)
        for t in range(1, L - 1):
            for _ in range(c_fmg):
                v_cycle(h, dt, top=t, final=False)
            _interp_up(h, t, dt)
        return
    raise ValueError(strategy)


def begin_slab(h, u0f, t0, dt):
    """``mlsdc.py:185-200``."""
    L = len(h.levels)
    h.levels[-1].u0 = np.asarray(u0f).copy()
    for i in range(L - 2, -1, -1):
        h.levels[i].u0 = h.transfers[i].project_u0(h.levels[i + 1].u0)
    for lv in h.levels:
        lv.t0, lv.sol, lv.g, lv.v = t0, None, None, None
        lv.ctx.begin_slab(lv.u0, t0, dt)


def run_mlsdc(h, u0f, t0, dt, n_cycles, strategy="fmg", c_fmg=1):
    """``mlsdc.py:203-234`` (no observer)."""
    begin_slab(h, u0f, t0, dt)
    start(h, strategy, dt, c_fmg)
    for _ in range(n_cycles):
        v_cycle(h, dt, final=False)
    if h.post_sweep and n_cycles > 0:
        _sweep_level(h, len(h.levels) - 1, dt, h.n_sweep)
    return h.levels[-1].sol


def integrate_mlsdc(h, u0f, t0, dt, n_steps, n_cycles, strategy="fmg", c_fmg=1):
    """``mlsdc.py:237-254``."""
    u, t = np.asarray(u0f), t0
    for _ in range(n_steps):
        u = run_mlsdc(h, u, t, dt, n_cycles, strategy, c_fmg).u[-1].copy()
        t += dt
    return u


def build_two_level(make_ctx, rule_c, rule_f, n_coarse=2, n_sweep=1, form="incremental",
                    post_sweep=True, scheme="si2", t0=False):
    """Two-level p-hierarchy as the reference CLI builds it (``cli.py:789-815``)."""
    cc, cf = make_ctx("coarse"), make_ctx("fine")
    levels = [Lev(cc, rule_c, scheme), Lev(cf, rule_f, scheme)]
    return Hier(levels, [PTransfer(cc, cf, rule_c, rule_f, t0=t0)], n_coarse, n_sweep, form, post_sweep)
