"""Generate golden vectors by running the REFERENCE itself in-process.

Usage (in the build container, where /root/reference exists):
    python oracle/make_golden.py
Writes tests/golden/*.npz.  The reference package is imported read-only from
/root/reference/pkg/src; nothing from it is copied into the repo -- only its
numerical outputs on seeded inputs.  The CG-trajectory goldens run the
reference's own sdc/mlsdc code with ``DGOperator.implicit_solve`` replaced by
the pinned PCG of ``oracle/cg.py`` (the north star's CG formulation); the
two-reduction Hestenes-Stiefel form is recorded too (``*_hs_iters*``).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from sisdc import collocation as rc, dgsem as rd, mlsdc as rm, problems as rp, sdc as rs, transfer as rt  # noqa: E402

from oracle.cg import bicgstab, element_block_preconditioner, pcg, pcg_hs  # noqa: E402
from paper_2504_18526_b200.configs import CFG1, CFG2, CNS_CASES, MANUFACTURED, SOD_CASES  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def ref_problem(w):
    if w.problem == "convdiff":
        return rp.ConvectionDiffusion(w.params["speed"], w.params["nu"])
    return rp.Burgers(w.params["nu"])


def build_ref_hier(w, form="incremental", node_convention="nodes_only"):
    ops = [rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, w.n_elem, P), ref_problem(w))
           for P in (w.p_coarse, w.p_fine)]
    rules = [rc.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
    wts = [rc.make_weights(r) for r in rules]
    levels = [rm.Level(o, r, ww, "si2") for o, r, ww in zip(ops, rules, wts)]
    pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", node_convention)
    spat = rt.build_spatial_p_transfer(w.p_coarse, w.p_fine, w.n_elem, 1, "embedded")
    return rm.Hierarchy(levels, [rt.SpaceTimeTransfer(pair, spat)], n_coarse=2, n_sweep=1,
                        form=form, post_sweep_on_finest=True), ops


class PcgPatch:
    """Swap DGOperator.implicit_solve for the pinned PCG; log iterations."""

    def __init__(self, rtol=1e-14, solver=pcg):
        self.rtol = rtol
        self.solver = solver
        self.log = []
        self._orig = rd.DGOperator.implicit_solve

    def __enter__(self):
        patch = self

        def solve(op, coeff, a, rhs, t=0.0):
            if a == 0.0:
                return rhs
            rhs = np.asarray(rhs)
            m = op._mass_flat
            b = m * rhs.reshape(-1)
            if not b.any():
                return np.zeros_like(rhs)
            Amat = op.assemble_implicit(coeff, a)
            diag = np.asarray(Amat.diagonal())
            if op.mesh.bc == "dirichlet":   # affine SIP: linear part + boundary data on the rhs
                dbc = op.apply_diffusion(coeff, np.zeros(op.ndof), t)
                b = b + a * m * dbc
                A = lambda x: m * x - a * m * (op.apply_diffusion(coeff, x, t) - dbc)
            else:
                A = lambda x: m * x - a * m * op.apply_diffusion(coeff, x, t)
            if op.ncomp > 1:   # systems: element-block Jacobi of the assembled matrix
                diag = element_block_preconditioner(Amat, op.ncomp, op.mesh.n_elem, op.p1)
            x, it, margin = patch.solver(A, diag, b, rhs.reshape(-1).copy(), patch.rtol, 1000)
            assert it >= 0
            patch.log.append((it, margin))
            return x.reshape(rhs.shape)

        rd.DGOperator.implicit_solve = solve
        return self

    def __exit__(self, *exc):
        rd.DGOperator.implicit_solve = self._orig


def gen_tables():
    out = {}
    for M in (1, 2, 3, 4, 5, 7):
        r = rc.make_nodes("radau_right", M)
        ww = rc.make_weights(r)
        out[f"radau_tau_{M}"] = r.tau
        out[f"radau_wnn_{M}"] = ww.w_nn
        out[f"radau_w0n_{M}"] = ww.w_0n
    for M in (2, 3, 5):
        out[f"lobatto_tau_{M}"] = rc.make_nodes("lobatto", M).tau
    for P in (3, 4, 7, 8):
        x, wt = rc.gauss_lobatto(P + 1)
        out[f"gll_x_{P}"], out[f"gll_w_{P}"] = x, wt
        out[f"D_{P}"] = rd._diff_matrix(x)
        out[f"delta_{P}"] = np.array(rd.compute_delta(P))
    for pc, pf in ((4, 8), (3, 7)):
        s = rt.build_spatial_p_transfer(pc, pf, 1)
        out[f"psp_interp_{pc}_{pf}"] = s.blocks["interp"]
        out[f"psp_project_{pc}_{pf}"] = s.blocks["project"]
    for mc, mf in ((2, 4), (3, 5), (2, 5)):
        pr_ = rt.build_temporal_transfer(rc.make_nodes("radau_right", mc), rc.make_nodes("radau_right", mf))
        out[f"t_interp_{mc}_{mf}"], out[f"t_project_{mc}_{mf}"] = pr_.interp, pr_.project
    np.savez_compressed(os.path.join(OUT, "tables.npz"), **out)


def gen_operators():
    """Operator outputs on seeded fields at the cfg-1/cfg-2 meshes and a
    small 1-D CNS mesh (matrix coefficients)."""
    rng = np.random.default_rng(1234)
    out = {}
    for tag, w, ne in (("cfg1", CFG1, CFG1.n_elem), ("cfg2", CFG2, 64)):
        for P in (w.p_fine, w.p_coarse):
            op = rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, ne, P), ref_problem(w))
            k = f"{tag}_P{P}"
            u = 1.0 + 0.3 * rng.standard_normal(op.ndof)
            fld = 0.01 + 0.02 * rng.random((ne, P + 1))
            out[k + "_u"] = u
            out[k + "_fld"] = fld
            out[k + "_conv"] = op.apply_convection(u)
            out[k + "_diff_const"] = op.apply_diffusion(0.0137, u)
            out[k + "_diff_field"] = op.apply_diffusion(fld, u)
            out[k + "_rhs"] = op.eval_rhs(u, 0.0)
            c = op.modified_diffusion_matrix(u, 0.0123, "si2")
            out[k + "_modc"] = np.asarray(c)
            out[k + "_diagA_field"] = op.assemble_implicit(fld, 0.0123).diagonal()
            out[k + "_diagA_const"] = op.assemble_implicit(0.0137, 0.0123).diagonal()
            rhs = u * 0.5 + 0.1 * np.sin(np.arange(op.ndof))
            out[k + "_solve_rhs"] = rhs
            out[k + "_solve_const"] = op.implicit_solve(0.0137, 0.0123, rhs)
            op2 = rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, ne, P), ref_problem(w))
            out[k + "_solve_field"] = op2.implicit_solve(fld, 0.0123, rhs)
    cf = rp.CompressibleFlow(eta=1e-3)
    op = rd.DGOperator(rd.Mesh1D(0.0, 1.0, 8, 5), cf)
    u3 = np.stack([1.0 + 0.1 * rng.random((8, 6)), 0.3 * rng.random((8, 6)), 3.0 + 0.3 * rng.random((8, 6))])
    u = u3.reshape(-1)
    out["cns_u"] = u
    out["cns_conv"] = op.apply_convection(u)
    out["cns_rhs"] = op.eval_rhs(u, 0.0)
    out["cns_coeff"] = cf.diffusion_coeff(u3)
    out["cns_diff"] = op.apply_diffusion(cf.diffusion_coeff(u3), u)
    out["cns_modc"] = op.modified_diffusion_matrix(u, 0.01, "si2")
    np.savez_compressed(os.path.join(OUT, "operators.npz"), **out)


def gen_trajectories():
    """Reference MLSDC steps for cfg1/cfg2: LU (the reference as shipped) and
    with the pinned PCG swapped in (iteration counts logged)."""
    out = {}
    import dataclasses
    cfg2c5 = dataclasses.replace(CFG2, n_cycles=5)   # the CLI-default schedule, one step (diverges later)
    for tag, w, nsteps in (("cfg1", CFG1, 3), ("cfg2", CFG2, 2), ("cfg2c5", cfg2c5, 1)):
        hier, ops = build_ref_hier(w)
        fine = ops[1]
        u0 = w.initial_state(fine.mesh.ref_nodes)
        dt, n = w.time_step(u0, rd.compute_delta(w.p_fine))
        out[f"{tag}_u0"] = u0
        out[f"{tag}_dt"] = np.array(dt)
        out[f"{tag}_nsteps_total"] = np.array(n)
        # LU trajectory (reference unmodified)
        u = u0
        for s in range(nsteps):
            sol = rm.run_mlsdc(hier, u, s * dt, dt, w.n_cycles, strategy="fmg")
            if s == 0:
                out[f"{tag}_lu_step1_nodes"] = sol.u.copy()
            u = sol.end_value.copy()
            out[f"{tag}_lu_u{s + 1}"] = u
        # PCG trajectory (reference sweeps/cycles, pinned PCG solve)
        for rtol, rk, solver in ((1e-14, "pcg", pcg), (1e-13, "pcg13", pcg), (1e-14, "hs", pcg_hs)):
            hier, ops = build_ref_hier(w)
            with PcgPatch(rtol, solver) as pp:
                u = u0
                for s in range(nsteps):
                    n0 = len(pp.log)
                    sol = rm.run_mlsdc(hier, u, s * dt, dt, w.n_cycles, strategy="fmg")
                    u = sol.end_value.copy()
                    out[f"{tag}_{rk}_u{s + 1}"] = u
                    out[f"{tag}_{rk}_iters{s + 1}"] = np.array([it for it, _ in pp.log[n0:]])
                    out[f"{tag}_{rk}_margin{s + 1}"] = np.array([mg for _, mg in pp.log[n0:]])
        if tag == "cfg2c5":
            continue
        # single-level SDC: predictor + 2 sweeps on the fine level (LU)
        opf = rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, w.n_elem, w.p_fine), ref_problem(w))
        rule = rc.make_nodes("radau_right", w.m_fine)
        wts = rc.make_weights(rule)
        sol = rs.run_sdc(opf, rule, wts, dt, "si2", u0, 0.0, 2)
        out[f"{tag}_sdc2_u"], out[f"{tag}_sdc2_f"] = sol.u, sol.f
        out[f"{tag}_sdc2_h1"], out[f"{tag}_sdc2_h2"] = sol.h1, sol.h2
    np.savez_compressed(os.path.join(OUT, "trajectories.npz"), **out)


def gen_t0conv():
    """node_convention = "nodes_plus_t0" (transfer.py:61-121, cli.py:289): the augmented
    temporal matrices, apply_temporal on seeded data in every direction, and two
    reference SI-MLSDC steps of cfg1 (LU as shipped, and with the pinned PCG)."""
    out = {}
    w = CFG1
    rules = [rc.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
    for kind in ("embedded", "l2"):
        pair = rt.build_temporal_transfer(rules[0], rules[1], kind, "nodes_plus_t0")
        out[f"{kind}_interp"], out[f"{kind}_project"], out[f"{kind}_restrict"] = pair.interp, pair.project, pair.restrict
    pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_plus_t0")
    rng = np.random.default_rng(11)
    nc, nf, u0 = rng.standard_normal((w.m_coarse, 7)), rng.standard_normal((w.m_fine, 7)), rng.standard_normal(7)
    out["in_c"], out["in_f"], out["in_u0"] = nc, nf, u0
    out["ap_interp"] = rt.apply_temporal(pair, "interp", nc, u0)
    out["ap_project"] = rt.apply_temporal(pair, "project", nf, u0)
    out["ap_restrict"] = rt.apply_temporal(pair, "restrict", nf)
    hier, ops = build_ref_hier(w, node_convention="nodes_plus_t0")
    u_init = w.initial_state(ops[1].mesh.ref_nodes)
    dt, _ = w.time_step(u_init, rd.compute_delta(w.p_fine))
    out["u0"], out["dt"] = u_init, np.array(dt)
    u = u_init
    for s in range(2):
        sol = rm.run_mlsdc(hier, u, s * dt, dt, w.n_cycles, strategy="fmg")
        u = sol.end_value.copy()
        out[f"lu_u{s + 1}"] = u
    hier, ops = build_ref_hier(w, node_convention="nodes_plus_t0")
    with PcgPatch(1e-14, pcg) as pp:
        u = u_init
        for s in range(2):
            n0 = len(pp.log)
            sol = rm.run_mlsdc(hier, u, s * dt, dt, w.n_cycles, strategy="fmg")
            u = sol.end_value.copy()
            out[f"pcg_u{s + 1}"] = u
            out[f"pcg_iters{s + 1}"] = np.array([it for it, _ in pp.log[n0:]])
    np.savez_compressed(os.path.join(OUT, "t0conv.npz"), **out)


def gen_nonincremental():
    """The reference's non-incremental sweep form (sdc.py:245-284): single-level
    run_sdc (predictor + 2 sweeps, si2 and si1) and one MLSDC step with the
    non-incremental hierarchy (mlsdc.py:68-101 form branches), SuperLU as
    shipped and with the pinned PCG (iteration counts)."""
    out = {}
    for tag, w in (("cfg1", CFG1), ("cfg2", CFG2)):
        opf = rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, w.n_elem, w.p_fine), ref_problem(w))
        u0 = w.initial_state(opf.mesh.ref_nodes)
        dt, _ = w.time_step(u0, rd.compute_delta(w.p_fine))
        rule = rc.make_nodes("radau_right", w.m_fine)
        wts = rc.make_weights(rule)
        for scheme in ("si2", "si1"):
            sol = rs.run_sdc(opf, rule, wts, dt, scheme, u0, 0.0, 2, form="nonincremental")
            out[f"{tag}_ni_{scheme}_u"], out[f"{tag}_ni_{scheme}_f"] = sol.u, sol.f
            out[f"{tag}_ni_{scheme}_h1"] = sol.h1
        hier, _ = build_ref_hier(w, "nonincremental")
        out[f"{tag}_ni_mlsdc_lu_u1"] = rm.run_mlsdc(hier, u0, 0.0, dt, w.n_cycles, strategy="fmg").end_value.copy()
        hier, _ = build_ref_hier(w, "nonincremental")
        with PcgPatch(1e-14, pcg) as pp:
            out[f"{tag}_ni_mlsdc_pcg_u1"] = rm.run_mlsdc(hier, u0, 0.0, dt, w.n_cycles, strategy="fmg").end_value.copy()
            out[f"{tag}_ni_mlsdc_pcg_iters1"] = np.array([it for it, _ in pp.log])
    np.savez_compressed(os.path.join(OUT, "nonincremental.npz"), **out)


# Dirichlet workload: the paper's Burgers moving front (problems.py:284-291,
# PAPER.md "Burgers moving front"): nu = 1e-2 on [-1, 1], exact-front trace data
DIRICHLET = dict(nu=1e-2, n_elem=20, p_fine=8, p_coarse=4, m_fine=5, m_coarse=3, cfl=1.0, t0=0.0)
AV_CASE = dict(n_elem=16, p_fine=4, p_coarse=2)


def dirichlet_ref(av=None, form="incremental", **over):
    d = {**DIRICHLET, **over}
    prob, exact = rp.burgers_front_problem(d["nu"])
    ops = [rd.DGOperator(rd.Mesh1D(-1.0, 1.0, d["n_elem"], p, bc="dirichlet"), prob, av=av)
           for p in (d["p_coarse"], d["p_fine"])]
    rules = [rc.make_nodes("radau_right", M) for M in (d["m_coarse"], d["m_fine"])]
    wts = [rc.make_weights(r) for r in rules]
    levels = [rm.Level(o, r, ww, "si2") for o, r, ww in zip(ops, rules, wts)]
    pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_only")
    spat = rt.build_spatial_p_transfer(d["p_coarse"], d["p_fine"], d["n_elem"], 1, "embedded")
    hier = rm.Hierarchy(levels, [rt.SpaceTimeTransfer(pair, spat)], n_coarse=2, n_sweep=1, form=form,
                        post_sweep_on_finest=True)
    return hier, ops, exact


def gen_dirichlet():
    """Dirichlet faces with time-dependent trace data (dgsem.py:179-201,212-216,
    282-289, assembly :460-481): operators at two times, implicit solves, a
    single-level SDC slab and two SI-MLSDC steps (SuperLU as shipped; with the
    pinned PCG: iteration counts), plus one step with Persson-Peraire AV."""
    d = DIRICHLET
    out = {}
    hier, ops, exact = dirichlet_ref()
    fine = ops[1]
    x = fine.mesh.nodes_x
    u0 = fine.flat(exact(x, d["t0"])[None])
    lam = float(np.abs(u0).max())
    dt = rd.dt_from_cfl(d["cfl"], fine.mesh.dx, lam, d["p_fine"])
    out["u0"], out["dt"] = u0, np.array(dt)
    rng = np.random.default_rng(11)
    us = u0 + 1e-3 * rng.standard_normal(u0.shape)
    out["us"] = us
    for j, t in enumerate((0.013, 0.071)):
        out[f"t{j}"] = np.array(t)
        out[f"conv{j}"] = fine.apply_convection(us, t)
        C = fine.modified_diffusion_matrix(us, 0.4 * dt, "si2")
        out[f"coef{j}"] = np.asarray(C)
        out[f"diff{j}"] = fine.apply_diffusion(C, us, t)
        out[f"rhs{j}"] = fine.eval_rhs(us, t)
        out[f"solve{j}"] = fine.implicit_solve(C, 0.4 * dt, us, t)
    rule = rc.make_nodes("radau_right", d["m_fine"])
    sol = rs.run_sdc(fine, rule, rc.make_weights(rule), dt, "si2", u0, d["t0"], 2)
    out["sdc2_u"], out["sdc2_h1"] = sol.u, sol.h1
    u = u0
    for step in range(2):
        u = rm.run_mlsdc(hier, u, d["t0"] + step * dt, dt, 3, strategy="fmg").end_value.copy()
        out[f"mlsdc_lu_u{step + 1}"] = u
    hier, ops, _ = dirichlet_ref()
    with PcgPatch(1e-14, pcg) as pp:
        u = u0
        for step in range(2):
            n0 = len(pp.log)
            u = rm.run_mlsdc(hier, u, d["t0"] + step * dt, dt, 3, strategy="fmg").end_value.copy()
            out[f"mlsdc_pcg_u{step + 1}"] = u
            out[f"mlsdc_pcg_iters{step + 1}"] = np.array([it for it, _ in pp.log[n0:]])
    # under-resolved front (16 elements, P 4/2) with the Persson-Peraire viscosity
    # (PAPER.md: kappa_s = c_s = 0.5), frozen per slab by begin_slab
    hier, ops, _ = dirichlet_ref(av=rd.ArtificialViscosityParams(0.5, 0.5), **AV_CASE)
    ua = ops[1].flat(exact(ops[1].mesh.nodes_x, d["t0"])[None])
    dta = rd.dt_from_cfl(d["cfl"], ops[1].mesh.dx, float(np.abs(ua).max()), AV_CASE["p_fine"])
    out["av_u0"], out["av_dt"] = ua, np.array(dta)
    out["av_nu_art"] = ops[1].persson_viscosity(ua)
    with PcgPatch(1e-14, pcg) as pp:
        out["av_mlsdc_pcg_u1"] = rm.run_mlsdc(hier, ua, d["t0"], dta, 3, strategy="fmg").end_value.copy()
        out["av_mlsdc_pcg_iters1"] = np.array([it for it, _ in pp.log])
    np.savez_compressed(os.path.join(OUT, "dirichlet.npz"), **out)


def gen_htransfer():
    """Spatial h-transfer (transfer.py:248-317): the block operators applied to
    seeded vectors for both jump policies and the l2 projection, the p-transfer
    l2 projection, and one SI-MLSDC step of cfg1's conv-diff with 2:1 element
    coarsening (64 -> 32 elements at P = 8; pinned PCG: iteration counts)."""
    out = {}
    rng = np.random.default_rng(21)
    for pol, kind in (("linear_blend", "embedded"), ("average", "embedded"), ("linear_blend", "l2")):
        st = rt.build_spatial_h_transfer(6, 5, 1, kind, pol)
        uc, uf = rng.standard_normal(6 * 6), rng.standard_normal(12 * 6)
        tag = f"h_{pol}_{kind}"
        out[f"{tag}_uc"], out[f"{tag}_uf"] = uc, uf
        for d in ("interp", "project", "restrict"):
            out[f"{tag}_{d}"] = st.apply(d, uc if d == "interp" else uf)
    sp = rt.build_spatial_p_transfer(3, 7, 5, 1, "l2")
    ufp = rng.standard_normal(5 * 8)
    out["p_l2_uf"], out["p_l2_project"] = ufp, sp.apply("project", ufp)
    w = CFG1
    ops = [rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, ne, w.p_fine), ref_problem(w))
           for ne in (w.n_elem // 2, w.n_elem)]
    rules = [rc.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
    wts = [rc.make_weights(r) for r in rules]
    levels = [rm.Level(o, r, ww, "si2") for o, r, ww in zip(ops, rules, wts)]
    pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_only")
    spat = rt.build_spatial_h_transfer(w.n_elem // 2, w.p_fine, 1, "embedded", "linear_blend")
    hier = rm.Hierarchy(levels, [rt.SpaceTimeTransfer(pair, spat)], n_coarse=2, n_sweep=1,
                        form="incremental", post_sweep_on_finest=True)
    u0 = w.initial_state(ops[1].mesh.ref_nodes)
    dt, _ = w.time_step(u0, rd.compute_delta(w.p_fine))
    with PcgPatch(1e-14, pcg) as pp:
        out["hml_pcg_u1"] = rm.run_mlsdc(hier, u0, 0.0, dt, w.n_cycles, strategy="fmg").end_value.copy()
        out["hml_pcg_iters1"] = np.array([it for it, _ in pp.log])
    np.savez_compressed(os.path.join(OUT, "htransfer.npz"), **out)


def gen_presmooth():
    """smooth_start (dgsem.py:574-589) on a state, and one cfg1/cfg2 SI-MLSDC step
    with the presmoothing hook (mlsdc.py:139-140) on the coarse level, pinned PCG."""
    out = {}
    for tag, w in (("cfg1", CFG1), ("cfg2", CFG2)):
        hier, ops = build_ref_hier(w)
        hier.presmooth = lambda u, op=ops[0]: rd.smooth_start(op, u)
        u0 = w.initial_state(ops[1].mesh.ref_nodes)
        dt, _ = w.time_step(u0, rd.compute_delta(w.p_fine))
        out[f"{tag}_smooth_fine_u0"] = rd.smooth_start(ops[1], u0)
        with PcgPatch(1e-14, pcg) as pp:
            out[f"{tag}_ps_pcg_u1"] = rm.run_mlsdc(hier, u0, 0.0, dt, w.n_cycles, strategy="fmg").end_value.copy()
            out[f"{tag}_ps_pcg_iters1"] = np.array([it for it, _ in pp.log])
    np.savez_compressed(os.path.join(OUT, "presmooth.npz"), **out)


def gen_cns():
    """1-D compressible flow (CompressibleFlow, matrix SI coefficients) on the
    reference's acoustic wave (problems.py:294-316): the reference's own
    test_dgsem.py:553-600 set-ups (single-level SDC at CFL 0.8 si1 and CFL 256
    si2) and a two-level MLSDC step, each with SuperLU (as shipped) and with
    the pinned Jacobi-BiCGStab swapped into DGOperator.implicit_solve."""
    out = {}
    for w in CNS_CASES:
        def build():
            prob = rp.CompressibleFlow(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl)
            ops = [rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, w.n_elem, P), prob)
                   for P in (w.p_coarse, w.p_fine)]
            rules = [rc.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
            return ops, rules
        ops, rules = build()
        u0 = w.initial_state(ops[1].mesh.ref_nodes)
        dt = w.time_step(u0, rd.compute_delta(w.p_fine))
        out[f"{w.name}_u0"] = u0
        out[f"{w.name}_dt"] = np.array(dt)

        def run(ops, rules):
            if w.mlsdc:
                wts = [rc.make_weights(r) for r in rules]
                levels = [rm.Level(o, r, ww, w.scheme) for o, r, ww in zip(ops, rules, wts)]
                pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_only")
                spat = rt.build_spatial_p_transfer(w.p_coarse, w.p_fine, w.n_elem, 3, "embedded")
                hier = rm.Hierarchy(levels, [rt.SpaceTimeTransfer(pair, spat)], n_coarse=2, n_sweep=1,
                                    form="incremental", post_sweep_on_finest=True)
                u, res = u0, []
                for s_ in range(w.n_steps):
                    u = rm.run_mlsdc(hier, u, s_ * dt, dt, w.n_cycles, strategy="fmg").end_value.copy()
                    res.append(u)
                return res
            rule = rules[1]
            wts = rc.make_weights(rule)
            u, res = u0, []
            for s_ in range(w.n_steps):
                u = rs.run_sdc(ops[1], rule, wts, dt, w.scheme, u, s_ * dt, w.n_sweeps).end_value.copy()
                res.append(u)
            return res
        for s_, u in enumerate(run(ops, rules)):
            out[f"{w.name}_lu_u{s_ + 1}"] = u
        ops, rules = build()
        with PcgPatch(1e-14, bicgstab) as pp:
            res = run(ops, rules)
        for s_, u in enumerate(res):
            out[f"{w.name}_bicg_u{s_ + 1}"] = u
        out[f"{w.name}_bicg_iters"] = np.array([it for it, _ in pp.log])
        out[f"{w.name}_bicg_margin"] = np.array([mg for _, mg in pp.log])
        print(w.name, "solves", len(pp.log), "iters", out[f"{w.name}_bicg_iters"].tolist()[:40],
              "rel(lu, bicg)", np.linalg.norm(res[-1] - out[f"{w.name}_lu_u{len(res)}"]) / np.linalg.norm(res[-1]))
    # operator goldens on the acoustic state: SI coefficient and a solve
    w = CNS_CASES[0]
    prob = rp.CompressibleFlow(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl)
    op = rd.DGOperator(rd.Mesh1D(w.x_left, w.x_right, w.n_elem, w.p_fine), prob)
    u0 = w.initial_state(op.mesh.ref_nodes)
    dt = w.time_step(u0, rd.compute_delta(w.p_fine))
    c = op.modified_diffusion_matrix(u0, 0.5 * dt, "si2")
    out["op_u"] = u0
    out["op_conv"] = op.apply_convection(u0)
    out["op_rhs"] = op.eval_rhs(u0, 0.0)
    out["op_modc"] = c
    out["op_diff_modc"] = op.apply_diffusion(c, u0)
    out["op_diagA"] = op.assemble_implicit(c, 0.5 * dt).diagonal()
    rhs = u0 * (1.0 + 1e-3 * np.sin(np.arange(op.ndof)))
    out["op_solve_rhs"] = rhs
    out["op_solve"] = op.implicit_solve(c, 0.5 * dt, rhs)
    np.savez_compressed(os.path.join(OUT, "cns.npz"), **out)


def gen_sources():
    """Burgers with a source term (problems.py:55-92, dgsem.py:328-347): the
    reference's manufactured steady state (test_dgsem.py:365-380), eval_rhs and
    apply_source on a manufactured unsteady solution, a single-level SDC slab
    and two SI-MLSDC steps (SuperLU and the pinned PCG) on a Dirichlet mesh."""
    out = {}
    w = MANUFACTURED
    nu0, ww = 0.05, 2 * np.pi

    def src_ss(x, t, u=None):
        return (2.0 + np.sin(ww * x)) * ww * np.cos(ww * x) + nu0 * ww * ww * np.sin(ww * x)
    prob = rp.Burgers(nu0, source=src_ss, boundary=lambda t: (np.array([2.0 + np.sin(-ww)]),
                                                               np.array([2.0 + np.sin(ww)])))
    op = rd.DGOperator(rd.Mesh1D(-1.0, 1.0, 20, 12, bc="dirichlet"), prob)
    u = op.flat((2.0 + np.sin(ww * op.mesh.nodes_x))[None])
    out["ss_u"] = u
    out["ss_rhs"] = op.eval_rhs(u, 0.0)

    def mk(P):
        return rd.DGOperator(rd.Mesh1D(-1.0, 1.0, w.n_elem, P, bc="dirichlet"),
                             rp.Burgers(w.nu, source=w.source, boundary=w.boundary))
    fine = mk(w.p_fine)
    u0 = fine.flat(w.exact(fine.mesh.nodes_x, 0.0)[None])
    lam = float(np.max(np.abs(u0)))
    dt = rd.dt_from_cfl(w.cfl, fine.mesh.dx, lam, w.p_fine)
    out["u0"], out["dt"] = u0, np.array(dt)
    out["rhs_t03"] = fine.eval_rhs(u0, 0.3)
    out["src_t03"] = fine.apply_source(u0, 0.3)
    rule = rc.make_nodes("radau_right", w.m_fine)
    sol = rs.run_sdc(fine, rule, rc.make_weights(rule), dt, "si2", u0, 0.0, 2)
    out["sdc2_u"], out["sdc2_f"] = sol.u, sol.f

    def hier():
        ops = [mk(P) for P in (w.p_coarse, w.p_fine)]
        rules = [rc.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
        levels = [rm.Level(o, r, rc.make_weights(r), "si2") for o, r in zip(ops, rules)]
        pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_only")
        spat = rt.build_spatial_p_transfer(w.p_coarse, w.p_fine, w.n_elem, 1, "embedded")
        return rm.Hierarchy(levels, [rt.SpaceTimeTransfer(pair, spat)], n_coarse=2, n_sweep=1,
                            form="incremental", post_sweep_on_finest=True)
    h = hier()
    u = u0
    for s_ in (1, 2):
        u = rm.run_mlsdc(h, u, (s_ - 1) * dt, dt, w.n_cycles, strategy="fmg").end_value.copy()
        out[f"mlsdc_lu_u{s_}"] = u
    h = hier()
    with PcgPatch(1e-14, pcg) as pp:
        u = u0
        for s_ in (1, 2):
            n0 = len(pp.log)
            u = rm.run_mlsdc(h, u, (s_ - 1) * dt, dt, w.n_cycles, strategy="fmg").end_value.copy()
            out[f"mlsdc_pcg_u{s_}"] = u
            out[f"mlsdc_pcg_iters{s_}"] = np.array([it for it, _ in pp.log[n0:]])
    out["exact_t2"] = fine.flat(w.exact(fine.mesh.nodes_x, 2 * dt)[None])
    print("sources: steady |rhs| max", np.abs(out["ss_rhs"]).max(), "mlsdc vs exact",
          np.linalg.norm(out["mlsdc_lu_u2"] - out["exact_t2"]) / np.linalg.norm(out["exact_t2"]))
    np.savez_compressed(os.path.join(OUT, "sources.npz"), **out)


def gen_sod():
    """1-D CompressibleFlow with Dirichlet faces: the reference CLI's Sod shock
    tube (cli.py:766-772) with Persson-Peraire viscosity, two SI-MLSDC steps
    with SuperLU (as shipped) and with the pinned BiCGStab, plus operators
    (convection with the boundary states, eval_rhs, the modal sensor, the
    affine matrix SIP and one implicit solve) at the initial state."""
    out = {}
    for w in SOD_CASES:
        left, right = w.states()

        def build():
            prob = rp.CompressibleFlow(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl,
                                       boundary=lambda t: (left, right))
            av = rd.ArtificialViscosityParams(*w.av) if w.av else None
            ops = [rd.DGOperator(rd.Mesh1D(0.0, 1.0, w.n_elem, P, bc="dirichlet"), prob, av=av)
                   for P in (w.p_coarse, w.p_fine)]
            rules = [rc.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
            levels = [rm.Level(o, r, rc.make_weights(r), "si2") for o, r in zip(ops, rules)]
            pair = rt.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_only")
            spat = rt.build_spatial_p_transfer(w.p_coarse, w.p_fine, w.n_elem, 3, "embedded")
            return rm.Hierarchy(levels, [rt.SpaceTimeTransfer(pair, spat)], n_coarse=2, n_sweep=1,
                                form="incremental", post_sweep_on_finest=True), ops
        h, ops = build()
        fine = ops[1]
        u0 = fine.nodal_field(w.initial)
        lam = rd.max_wave_speed(fine, u0)
        dt = rd.dt_from_cfl(w.cfl, fine.mesh.dx, lam, w.p_fine)
        k = w.name
        out[k + "_u0"], out[k + "_dt"] = u0, np.array(dt)
        op = rd.DGOperator(rd.Mesh1D(0.0, 1.0, w.n_elem, w.p_fine, bc="dirichlet"), fine.problem,
                           av=rd.ArtificialViscosityParams(*w.av) if w.av else None)
        out[k + "_conv"] = op.apply_convection(u0, 0.0)
        op.begin_slab(u0, 0.0, dt)
        out[k + "_nu_art"] = op.persson_viscosity(u0)
        out[k + "_rhs"] = op.eval_rhs(u0, 0.0)
        c = op.modified_diffusion_matrix(u0, 0.5 * dt, "si2")
        out[k + "_modc"] = c
        out[k + "_diff"] = op.apply_diffusion(c, u0, 0.0)
        out[k + "_solve"] = op.implicit_solve(c, 0.5 * dt, u0, 0.0)
        u = u0
        for s_ in range(w.n_steps):
            u = rm.run_mlsdc(h, u, s_ * dt, dt, w.n_cycles, strategy="fmg").end_value.copy()
            out[f"{k}_lu_u{s_ + 1}"] = u
        h, ops = build()
        with PcgPatch(1e-14, bicgstab) as pp:
            u = u0
            for s_ in range(w.n_steps):
                u = rm.run_mlsdc(h, u, s_ * dt, dt, w.n_cycles, strategy="fmg").end_value.copy()
                out[f"{k}_bicg_u{s_ + 1}"] = u
        out[k + "_bicg_iters"] = np.array([it for it, _ in pp.log])
        print(k, "solves", len(pp.log), "max it", max(it for it, _ in pp.log), "lu vs bicg",
              np.linalg.norm(out[f"{k}_lu_u{w.n_steps}"] - u) / np.linalg.norm(u))
    np.savez_compressed(os.path.join(OUT, "sod.npz"), **out)


STUDY_CONFIG = {
    "study": "cfl-sweep",
    "problem": {"kind": "convection_diffusion", "speed": 1.0, "nu": 0.002},
    "levels": [{"n_elem": 12, "degree": 3, "n_nodes": 2}, {"n_elem": 12, "degree": 6, "n_nodes": 4}],
    "time": {"t_end": 0.05},
    "sweep": {"cfl_values": [0.5, 1.0, 2.0, 4.0], "max_iterations": 6},
    "reference": {"kind": "exact"},
}


CONV_CONFIG = {
    "study": "convergence",
    "problem": {"kind": "convection_diffusion", "speed": 1.0, "nu": 0.002},
    "levels": [{"degree": 3, "n_nodes": 2}, {"degree": 6, "n_nodes": 4}],
    "time": {"t_end": 0.02},
    "method": {"iterations": 3},
    "convergence": {"element_counts": [[8, 8], [16, 16], [32, 32]], "cfl_values": [0.5, 1.0]},
}


def gen_study():
    """The reference CLI's own cfl-sweep study (cli.py:1110-1194) on its
    wave-packet convection-diffusion problem, run in-process: its
    errors.csv / iterations.csv contents are the goldens of the GPU ensemble
    dispatch (paper_2504_18526_b200/study.py)."""
    import json
    import tempfile
    from sisdc import cli as rcli
    cfg = rcli.parse_config(json.dumps(STUDY_CONFIG))
    with tempfile.TemporaryDirectory() as d:
        outputs, failures = rcli.run_study(cfg, d)
        err = open(os.path.join(d, "errors.csv")).read()
        its = open(os.path.join(d, "iterations.csv")).read()
    out = {"config": np.array(json.dumps(STUDY_CONFIG)), "errors_csv": np.array(err), "iterations_csv": np.array(its)}
    cfg = rcli.parse_config(json.dumps(CONV_CONFIG))
    with tempfile.TemporaryDirectory() as d:
        rcli.run_study(cfg, d)
        out["conv_config"] = np.array(json.dumps(CONV_CONFIG))
        out["conv_errors_csv"] = np.array(open(os.path.join(d, "errors.csv")).read())
        out["conv_orders_csv"] = np.array(open(os.path.join(d, "orders.csv")).read())
    print(str(out["conv_errors_csv"]), str(out["conv_orders_csv"]))
    print(its)
    np.savez_compressed(os.path.join(OUT, "study.npz"), **out)


# ------------------------------------------------ multilevel (L = 3) hierarchies
# The paper's Burgers moving front (cli.py:751-755 front on
# [-1, 1], nu = 1e-2, exact solution as reference), high-resolution hierarchies
# of tab:burgers_iterations_cfl_hires: MLSDC-SI(2,2)_{3,5,7} with p-coarsening
# {5,10,15} on 200 elements and h-coarsening {50,100,200} at P = 15.
ML_LEVELS = {
    "p3": [(200, 5, 3), (200, 10, 5), (200, 15, 7)],
    "h3": [(50, 15, 3), (100, 15, 5), (200, 15, 7)],
    "i3": [(200, 15, 3), (200, 15, 5), (200, 15, 7)],   # time-only coarsening (identity spatial)
    "sdc": [(200, 15, 7)],
}
ML_STEP_CASES = {   # one SI-MLSDC step at CFL 4, 3 V-cycles, from the exact state at t = 0
    "p3_fmg1": ("p3", "fmg", 1), "p3_fmg2": ("p3", "fmg", 2), "p3_cascade": ("p3", "cascade", 1),
    "p3_predictor": ("p3", "predictor", 1), "p3_constant": ("p3", "constant", 1),
    "h3_fmg1": ("h3", "fmg", 1), "h3_fmg2": ("h3", "fmg", 2), "h3_cascade": ("h3", "cascade", 1),
    "i3_fmg1": ("i3", "fmg", 1),
}
ML_STUDY_CASES = {   # rows of tab:burgers_iterations_cfl_hires
    "sdc": ("sdc", "predictor", 1), "i3_fmg1": ("i3", "fmg", 1), "h3_fmg2": ("h3", "fmg", 2),
    "h3_fmg1": ("h3", "fmg", 1), "h3_cascade": ("h3", "cascade", 1), "p3_fmg1": ("p3", "fmg", 1),
}
ML_STUDY_CFL = (8.0, 16.0, 32.0, 64.0)


def ml_config(levels, start, c_fmg, cfl_values=(4.0,), max_iterations=16):
    lv = [{"n_elem": ne, "degree": P, "n_nodes": M} for ne, P, M in ML_LEVELS[levels]]
    method = {"start": start, "c_fmg": c_fmg} if len(lv) > 1 else {"start": start}
    return {"study": "cfl-sweep", "problem": {"kind": "burgers", "nu": 0.01}, "levels": lv,
            "time": {"t_end": 0.1}, "method": method,
            "sweep": {"cfl_values": list(cfl_values), "max_iterations": max_iterations},
            "reference": {"kind": "exact"}}


def gen_multilevel_steps():
    """One SI-MLSDC step per 3-level case, built by the reference CLI's own
    _build_operators/_build_hierarchy (cli.py:776-815): the reference as
    shipped (SuperLU) and with the pinned PCG (iteration sequence)."""
    import json
    from sisdc import cli as rcli
    out = {}
    for name, (levels, start, c_fmg) in ML_STEP_CASES.items():
        cfg = rcli.parse_config(json.dumps(ml_config(levels, start, c_fmg)))
        bundle = rcli.build_problem(cfg.problem)
        res = {}
        for solver in ("lu", "pcg"):
            ops, rules, weights = rcli._build_operators(cfg, bundle)
            hier = rcli._build_hierarchy(cfg, ops, rules, weights)
            op = ops[-1]
            u0 = rcli._initial_state(op, bundle)
            lam = rd.max_wave_speed(op, u0)
            dt = rd.dt_from_cfl(4.0, op.mesh.dx, lam, op.mesh.degree)
            if solver == "lu":
                res["lu"] = rm.run_mlsdc(hier, u0, 0.0, dt, 3, strategy=start, c_fmg=c_fmg).end_value.copy()
            else:
                with PcgPatch(1e-14, pcg) as pp:
                    res["pcg"] = rm.run_mlsdc(hier, u0, 0.0, dt, 3, strategy=start, c_fmg=c_fmg).end_value.copy()
                res["iters"] = np.array([it for it, _ in pp.log])
                res["margins"] = np.array([mg for _, mg in pp.log])
        out[f"{name}_pcg_margins1"] = res["margins"]
        out[f"{name}_u0"], out[f"{name}_dt"] = u0, np.array(dt)
        out[f"{name}_lu_u1"], out[f"{name}_pcg_u1"], out[f"{name}_pcg_iters1"] = res["lu"], res["pcg"], res["iters"]
        print(name, len(res["iters"]), int(res["iters"].sum()),
              np.linalg.norm(res["lu"] - res["pcg"]) / np.linalg.norm(res["lu"]), flush=True)
    out["config"] = np.array(json.dumps({k: list(v) for k, v in ML_STEP_CASES.items()}))
    out["levels"] = np.array(json.dumps(ML_LEVELS))
    np.savez_compressed(os.path.join(OUT, "multilevel.npz"), **out)


def _ml_study_job(args):
    import json
    import tempfile
    name, cfl, solver = args
    from sisdc import cli as rcli
    levels, start, c_fmg = ML_STUDY_CASES[name]
    cfg = rcli.parse_config(json.dumps(ml_config(levels, start, c_fmg, (cfl,))))
    with tempfile.TemporaryDirectory() as d:
        if solver == "pcg":
            with PcgPatch(1e-14, pcg):
                rcli.run_study(cfg, d)
        else:
            rcli.run_study(cfg, d)
        return name, cfl, open(os.path.join(d, "errors.csv")).read(), open(os.path.join(d, "iterations.csv")).read()


def gen_multilevel_study(procs=8, solver="lu"):
    """The reference CLI's cfl-sweep study (cli.py:1110-1194) on the paper's
    high-resolution Burgers front hierarchies, one process per (case, CFL):
    the iterations.csv / errors.csv rows the GPU study must reproduce, and
    the paper's own table values next to them."""
    import json
    from multiprocessing import Pool
    jobs = [(n, c, solver) for n in ML_STUDY_CASES for c in sorted(ML_STUDY_CFL, reverse=True)]
    with Pool(procs) as pool:
        res = pool.map(_ml_study_job, jobs, chunksize=1)
    out = {"config": np.array(json.dumps({"cases": {k: list(v) for k, v in ML_STUDY_CASES.items()},
                                          "levels": ML_LEVELS, "cfl": list(ML_STUDY_CFL),
                                          "max_iterations": 16, "t_end": 0.1, "nu": 0.01}))}
    for name in ML_STUDY_CASES:
        errs = [r for r in res if r[0] == name]
        errs.sort(key=lambda r: r[1])
        head_e, head_i = errs[0][2].split("\n")[0], errs[0][3].split("\n")[0]
        out[f"{name}_errors_csv"] = np.array("\n".join([head_e] + [ln for r in errs
                                                                    for ln in r[2].strip().split("\n")[1:]]) + "\n")
        out[f"{name}_iterations_csv"] = np.array("\n".join([head_i] + [ln for r in errs
                                                                        for ln in r[3].strip().split("\n")[1:]]) + "\n")
        print(name, str(out[f"{name}_iterations_csv"]), flush=True)
    np.savez_compressed(os.path.join(OUT, "multilevel_study.npz" if solver == "lu" else
                                     "multilevel_study_pcg.npz"), **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1 and sys.argv[1] == "sod":
        gen_sod()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "study":
        gen_study()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "multilevel":
        gen_multilevel_steps()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "multilevel_study":
        gen_multilevel_study()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "multilevel_study_pcg":
        gen_multilevel_study(solver="pcg")
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "sources":
        gen_sources()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "cns":
        gen_cns()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "t0conv":
        gen_t0conv()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "nonincremental":
        gen_nonincremental()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "dirichlet":
        gen_dirichlet()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "presmooth":
        gen_presmooth()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "htransfer":
        gen_htransfer()
        sys.exit(0)
    gen_tables()
    gen_operators()
    gen_trajectories()
    gen_nonincremental()
    gen_t0conv()
    gen_dirichlet()
    gen_presmooth()
    gen_htransfer()
    gen_cns()
    gen_sources()
    gen_study()
    gen_sod()
    gen_multilevel_steps()
    gen_multilevel_study()
    gen_multilevel_study(solver="pcg")
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
