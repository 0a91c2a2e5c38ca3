"""Oracle builders for the BASELINE workloads (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

from . import dg1d, quad, sweeper


def make_problem(w):
    return dg1d.ConvDiff(**w.params) if w.problem == "convdiff" else dg1d.Burgers(**w.params)


def build_hierarchy(w, solver="pcg", rtol=1e-14, log=None):
    """Two-level p-hierarchy of workload ``w`` (configs.Workload1D); every
    level appends its CG iterations to the shared ``log`` in call order."""
    log = [] if log is None else log

    def mk(lvl):
        P = w.p_coarse if lvl == "coarse" else w.p_fine
        return dg1d.Op1D(w.x_left, w.x_right, w.n_elem, P, make_problem(w), solver=solver, rtol=rtol, cg_log=log)

    h = sweeper.build_two_level(mk, sweeper.Rule("radau_right", w.m_coarse), sweeper.Rule("radau_right", w.m_fine))
    return h, log


def fine_nodes(w):
    return quad.gll(w.p_fine + 1)[0]
