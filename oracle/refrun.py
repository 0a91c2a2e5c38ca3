"""Run the installed reference (``oracle/_ref``, see ``build_ref.py``) on a
BASELINE 1-D workload through its own public API (TEST / BENCH
INFRASTRUCTURE ONLY).

The hierarchy is built exactly as a reference user would
(``Mesh1D``/``DGOperator``/``make_nodes``/``build_temporal_transfer``/
``build_spatial_p_transfer``/``Hierarchy``, ``cli.py:776-815``) and
marched with ``sisdc.mlsdc.run_mlsdc`` (``mlsdc.py:203-234``), whose implicit
substeps use the reference's SuperLU path (``dgsem.py:503-533``).
"""
from __future__ import annotations

import time

import numpy as np

from .build_ref import import_reference


def build_hierarchy(w, form: str = "incremental"):
    """Two-level p-hierarchy of workload ``w`` (configs.Workload1D) built
    with the reference's own classes."""
    import_reference()
    from sisdc import collocation as rc, dgsem as rd, mlsdc as rm, problems as rp, transfer as rt
    prob = (rp.ConvectionDiffusion(w.params["speed"], w.params["nu"]) if w.problem == "convdiff"
            else rp.Burgers(w.params["nu"]))
    ops = [rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, w.n_elem, P), prob) for P in (w.p_coarse, w.p_fine)]
    rules = [rc.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
    levels = [rm.Level(o, r, rc.make_weights(r), "si2") for o, r in zip(ops, rules)]
    pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_only")
    spat = rt.build_spatial_p_transfer(w.p_coarse, w.p_fine, w.n_elem, 1, "embedded")
    return rm.Hierarchy(levels, [rt.SpaceTimeTransfer(pair, spat)], n_coarse=2, n_sweep=1, form=form,
                        post_sweep_on_finest=True)


def initial(w):
    import_reference()
    from sisdc import collocation as rc, dgsem as rd
    mesh = rd.Mesh1D(w.x_left, w.x_right, w.n_elem, w.p_fine)
    u0 = w.initial_state(rc.gauss_lobatto(w.p_fine + 1)[0])
    dt, n = w.time_step(u0, rd.compute_delta(w.p_fine))
    return mesh, u0, dt, n


def time_steps(w, n_steps: int, warmup: int = 1, budget_s: float | None = None):
    """March ``warmup`` then ``n_steps`` SI-MLSDC slabs with the reference;
    returns (seconds per step, steps timed, final state).  ``budget_s`` stops
    early (at >= 3 timed steps) so a bounded sample stays bounded."""
    import_reference()
    from sisdc import mlsdc as rm
    _, u, dt, _ = initial(w)
    hier = build_hierarchy(w)
    s = 0
    for _ in range(warmup):   # factorisations (per-shift SuperLU cache) happen here
        u = rm.run_mlsdc(hier, u, s * dt, dt, w.n_cycles, strategy="fmg").end_value.copy()
        s += 1
    t0 = time.perf_counter()
    done = 0
    for _ in range(n_steps):
        u = rm.run_mlsdc(hier, u, s * dt, dt, w.n_cycles, strategy="fmg").end_value.copy()
        s += 1
        done += 1
        if budget_s is not None and done >= 3 and time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return el / done, done, np.asarray(u)
