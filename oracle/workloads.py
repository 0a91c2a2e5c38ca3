"""Oracle builders for the BASELINE workloads (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

from . import dg1d, quad, sweeper


def make_problem(w):
    return dg1d.ConvDiff(**w.params) if w.problem == "convdiff" else dg1d.Burgers(**w.params)


def build_hierarchy(w, solver="pcg", rtol=1e-14, log=None, form="incremental", t0=False):
    """Two-level p-hierarchy of workload ``w`` (configs.Workload1D); every
    level appends its CG iterations to the shared ``log`` in call order."""
    log = [] if log is None else log

    def mk(lvl):
        P = w.p_coarse if lvl == "coarse" else w.p_fine
        return dg1d.Op1D(w.x_left, w.x_right, w.n_elem, P, make_problem(w), solver=solver, rtol=rtol, cg_log=log)

    h = sweeper.build_two_level(mk, sweeper.Rule("radau_right", w.m_coarse), sweeper.Rule("radau_right", w.m_fine),
                                form=form, t0=t0)
    return h, log


def fine_nodes(w):
    return quad.gll(w.p_fine + 1)[0]


def build_hierarchy_2d(make_problem2d, x0, x1, y0, y1, nex, ney, p_coarse, p_fine, m_coarse, m_fine,
                       rtol=1e-14, log=None, n_coarse=2, av=None):
    """Two-level 2-D p-hierarchy (oracle) sharing one CG log in call order."""
    from . import dg2d
    log = [] if log is None else log

    def mk(lvl):
        P = p_coarse if lvl == "coarse" else p_fine
        return dg2d.Op2D(x0, x1, y0, y1, nex, ney, P, make_problem2d(), rtol=rtol, cg_log=log, av=av)

    cc, cf = mk("coarse"), mk("fine")
    rc, rf = sweeper.Rule("radau_right", m_coarse), sweeper.Rule("radau_right", m_fine)
    levels = [sweeper.Lev(cc, rc), sweeper.Lev(cf, rf)]
    return sweeper.Hier(levels, [dg2d.PTransfer2D(cc, cf, rc, rf)], n_coarse, 1, "incremental", True), log


def problem2d(w):
    """Oracle physics of a configs.Workload2D: NS2D (eta, Pr) when viscous, else Euler2D."""
    from . import dg2d
    if w.eta > 0:
        return dg2d.NS2D(w.gamma, w.eta, w.prandtl)
    return dg2d.Euler2D(w.gamma, 0.0)
