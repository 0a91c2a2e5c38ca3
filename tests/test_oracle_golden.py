"""Pin the CPU oracle against golden vectors produced by the reference itself
(oracle/make_golden.py runs /root/reference in-process)."""
import numpy as np
import pytest

from oracle import dg1d, quad, sweeper, workloads
from paper_2504_18526_b200.configs import CFG1, CFG2


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(1.0, np.abs(np.asarray(b)).max()))


def test_tables(golden):
    G = golden["tables"]
    for M in (1, 2, 3, 4, 5, 7):
        tau = quad.radau_right(M)
        assert np.abs(tau - G[f"radau_tau_{M}"]).max() < 1e-15
        assert np.abs(quad.weights_nn(tau) - G[f"radau_wnn_{M}"]).max() < 1e-14
        assert np.abs(quad.weights_0n(quad.weights_nn(tau)) - G[f"radau_w0n_{M}"]).max() < 1e-14
    for M in (2, 3, 5):
        assert np.abs(quad.lobatto(M) - G[f"lobatto_tau_{M}"]).max() < 1e-15
    for P in (3, 4, 7, 8):
        x, w = quad.gll(P + 1)
        assert np.abs(x - G[f"gll_x_{P}"]).max() < 1e-15
        assert np.abs(w - G[f"gll_w_{P}"]).max() < 1e-15
        assert rel(quad.diff_matrix(x), G[f"D_{P}"]) < 1e-14
        assert abs(quad.delta_of_degree(P) - float(G[f"delta_{P}"])) < 1e-12
    for pc, pf in ((4, 8), (3, 7)):
        assert rel(quad.lagrange(quad.gll(pc + 1)[0], quad.gll(pf + 1)[0]), G[f"psp_interp_{pc}_{pf}"]) < 1e-14
        assert rel(quad.lagrange(quad.gll(pf + 1)[0], quad.gll(pc + 1)[0]), G[f"psp_project_{pc}_{pf}"]) < 1e-14


@pytest.mark.parametrize("tag,w,ne", [("cfg1", CFG1, CFG1.n_elem), ("cfg2", CFG2, 64)])
def test_operators(golden, tag, w, ne):
    G = golden["operators"]
    for P in (w.p_fine, w.p_coarse):
        k = f"{tag}_P{P}"
        op = dg1d.Op1D(w.x_left, w.x_right, ne, P, workloads.make_problem(w), solver="lu")
        u, fld = G[k + "_u"], G[k + "_fld"]
        assert rel(op.apply_convection(u), G[k + "_conv"]) < 1e-13
        assert rel(op.apply_diffusion(0.0137, u), G[k + "_diff_const"]) < 1e-13
        assert rel(op.apply_diffusion(fld, u), G[k + "_diff_field"]) < 1e-13
        assert rel(op.eval_rhs(u), G[k + "_rhs"]) < 1e-13
        assert rel(np.asarray(op.modified_coeff(u, 0.0123, "si2")), G[k + "_modc"]) < 1e-14
        assert rel(op.mflat + 0.0123 * op.stiffness_diag(fld), G[k + "_diagA_field"]) < 1e-14
        assert rel(op.mflat + 0.0123 * op.stiffness_diag(0.0137), G[k + "_diagA_const"]) < 1e-14
        rhs = G[k + "_solve_rhs"]
        assert rel(op.implicit_solve(0.0137, 0.0123, rhs), G[k + "_solve_const"]) < 1e-12
        op2 = dg1d.Op1D(w.x_left, w.x_right, ne, P, workloads.make_problem(w), solver="lu")
        assert rel(op2.implicit_solve(fld, 0.0123, rhs), G[k + "_solve_field"]) < 1e-11
        op3 = dg1d.Op1D(w.x_left, w.x_right, ne, P, workloads.make_problem(w), solver="pcg")
        assert rel(op3.implicit_solve(fld, 0.0123, rhs), G[k + "_solve_field"]) < 1e-11


def test_cns_matrix_coefficient(golden):
    G = golden["operators"]
    op = dg1d.Op1D(0.0, 1.0, 8, 5, dg1d.CNS1D(eta=1e-3))
    u = G["cns_u"]
    assert rel(op.apply_convection(u), G["cns_conv"]) < 1e-13
    assert rel(op.eval_rhs(u), G["cns_rhs"]) < 1e-13
    assert rel(op.apply_diffusion(G["cns_coeff"], u), G["cns_diff"]) < 1e-13
    assert rel(op.modified_coeff(u, 0.01, "si2"), G["cns_modc"]) < 1e-13


CFG2C5 = __import__("dataclasses").replace(CFG2, n_cycles=5)


@pytest.mark.parametrize("tag,w", [("cfg1", CFG1), ("cfg2", CFG2), ("cfg2c5", CFG2C5)])
def test_mlsdc_step_lu_and_pcg(golden, tag, w):
    """One SI-MLSDC step from the shared golden input: LU restatement vs the
    reference as shipped; PCG vs the reference with the pinned PCG swapped in
    (identical CG iteration sequence)."""
    G = golden["trajectories"]
    dt = float(G[f"{tag}_dt"])
    u0 = G[f"{tag}_u0"]
    assert np.abs(u0 - w.initial_state(workloads.fine_nodes(w))).max() < 1e-14
    for solver, key, tol in (("lu", "lu", 1e-12), ("pcg", "pcg", 1e-12)):
        h, log = workloads.build_hierarchy(w, solver=solver)
        sol = sweeper.run_mlsdc(h, u0, 0.0, dt, w.n_cycles, "fmg")
        ref = G[f"{tag}_{key}_u1"]
        assert np.linalg.norm(sol.u[-1] - ref) / np.linalg.norm(ref) < tol
        assert h.fine_sweeps == w.n_cycles + 1 and h.coarse_passes == 2 + 2 * w.n_cycles
        if solver == "pcg":
            assert [it for it, _ in log] == G[f"{tag}_pcg_iters1"].tolist()
            # the two-reduction textbook form takes the same iterations
            assert G[f"{tag}_pcg_iters1"].tolist() == G[f"{tag}_hs_iters1"].tolist()
    if tag == "cfg1":
        assert np.abs(sol.u - G["cfg1_lu_step1_nodes"]).max() < 1e-12


def test_single_level_sdc(golden):
    G = golden["trajectories"]
    w = CFG1
    op = dg1d.Op1D(w.x_left, w.x_right, w.n_elem, w.p_fine, workloads.make_problem(w), solver="lu")
    rule = sweeper.Rule("radau_right", w.m_fine)
    s = sweeper.run_sdc(op, rule, float(G["cfg1_dt"]), "si2", G["cfg1_u0"], 0.0, 2)
    # f = eval_rhs(u) amplifies state roundoff by ||D[nu]|| ~ 1e4: looser bound
    for k, tol in (("u", 1e-13), ("f", 1e-10), ("h1", 1e-12), ("h2", 1e-12)):
        assert rel(getattr(s, k), G[f"cfg1_sdc2_{k}"]) < tol


@pytest.mark.parametrize("tag,w", [("cfg1", CFG1), ("cfg2", CFG2)])
def test_nonincremental_form(golden, tag, w):
    """The reference's non-incremental sweep (sdc.py:245-284) and
    non-incremental MLSDC (mlsdc.py:68-101): single-level predictor + 2 sweeps
    (si2, si1) and one MLSDC step, LU vs the reference as shipped, PCG vs the
    reference with the pinned PCG (identical iterations)."""
    G, T = golden["nonincremental"], golden["trajectories"]
    dt, u0 = float(T[f"{tag}_dt"]), T[f"{tag}_u0"]
    op = dg1d.Op1D(w.x_left, w.x_right, w.n_elem, w.p_fine, workloads.make_problem(w), solver="lu")
    rule = sweeper.Rule("radau_right", w.m_fine)
    for scheme in ("si2", "si1"):
        s = sweeper.run_sdc(op, rule, dt, scheme, u0, 0.0, 2, form="nonincremental")
        assert rel(s.u, G[f"{tag}_ni_{scheme}_u"]) < 1e-12
        assert rel(s.h1, G[f"{tag}_ni_{scheme}_h1"]) < 1e-12
    for solver, key in (("lu", "lu"), ("pcg", "pcg")):
        h, log = workloads.build_hierarchy(w, solver=solver, form="nonincremental")
        sol = sweeper.run_mlsdc(h, u0, 0.0, dt, w.n_cycles, "fmg")
        ref = G[f"{tag}_ni_mlsdc_{key}_u1"]
        assert np.linalg.norm(sol.u[-1] - ref) / np.linalg.norm(ref) < 1e-12
        if solver == "pcg":
            assert [it for it, _ in log] == G[f"{tag}_ni_mlsdc_pcg_iters1"].tolist()


# ------------------------------------------------ Dirichlet faces (moving front)
def _front_oracle(w, solver, log=None):
    from paper_2504_18526_b200.configs import burgers_front_boundary
    bnd = burgers_front_boundary(w.nu)

    def mk(lvl):
        P = w.p_coarse if lvl == "coarse" else w.p_fine
        return dg1d.Op1D(-1.0, 1.0, w.n_elem, P, dg1d.Burgers(w.nu, boundary=bnd), solver=solver,
                         bc="dirichlet", av=w.av, cg_log=log)
    return mk


def test_dirichlet_front(golden):
    """Dirichlet faces with time-dependent trace data vs the reference
    (burgers_front_problem): operators at two times, implicit solves (LU and
    the pinned PCG on the affine system), single-level SDC, two SI-MLSDC
    steps (PCG: identical iteration sequence), and the AV case."""
    from paper_2504_18526_b200.configs import FRONT, FRONT_AV
    G = golden["dirichlet"]
    w = FRONT
    op = _front_oracle(w, "lu")("fine")
    dt, us = float(G["dt"]), G["us"]
    for j in (0, 1):
        t = float(G[f"t{j}"])
        assert rel(op.apply_convection(us, t), G[f"conv{j}"]) < 1e-13
        C = op.modified_coeff(us, 0.4 * dt)
        assert rel(C, G[f"coef{j}"]) < 1e-15
        assert rel(op.apply_diffusion(C, us, t), G[f"diff{j}"]) < 1e-13
        assert rel(op.eval_rhs(us, t), G[f"rhs{j}"]) < 1e-13
        assert rel(op.implicit_solve(C, 0.4 * dt, us, t), G[f"solve{j}"]) < 1e-12
        opc = _front_oracle(w, "pcg")("fine")
        assert rel(opc.implicit_solve(C, 0.4 * dt, us, t), G[f"solve{j}"]) < 1e-11
    rule = sweeper.Rule("radau_right", w.m_fine)
    s = sweeper.run_sdc(op, rule, dt, "si2", G["u0"], 0.0, 2)
    assert rel(s.u, G["sdc2_u"]) < 1e-12 and rel(s.h1, G["sdc2_h1"]) < 1e-11
    log = []
    mk = _front_oracle(w, "pcg", log)
    h = sweeper.build_two_level(mk, sweeper.Rule("radau_right", w.m_coarse), rule)
    u = G["u0"]
    for step in (1, 2):
        n0 = len(log)
        u = sweeper.run_mlsdc(h, u, (step - 1) * dt, dt, w.n_cycles, "fmg").u[-1]
        assert [it for it, _ in log[n0:]] == G[f"mlsdc_pcg_iters{step}"].tolist()
        assert np.linalg.norm(u - G[f"mlsdc_pcg_u{step}"]) / np.linalg.norm(G[f"mlsdc_pcg_u{step}"]) < 1e-12
    wa = FRONT_AV
    log = []
    mk = _front_oracle(wa, "pcg", log)
    h = sweeper.build_two_level(mk, sweeper.Rule("radau_right", wa.m_coarse), sweeper.Rule("radau_right", wa.m_fine))
    assert rel(h.levels[1].ctx.persson_viscosity(G["av_u0"]), G["av_nu_art"]) < 1e-13
    u = sweeper.run_mlsdc(h, G["av_u0"], 0.0, float(G["av_dt"]), wa.n_cycles, "fmg").u[-1]
    assert [it for it, _ in log] == G["av_mlsdc_pcg_iters1"].tolist()
    assert np.linalg.norm(u - G["av_mlsdc_pcg_u1"]) / np.linalg.norm(G["av_mlsdc_pcg_u1"]) < 1e-12


def _cns_oracle_run(w, log, solver="pcg", u0=None, dt=None):
    """The oracle's restatement of the reference's SDC / MLSDC on the 1-D CNS
    acoustic workloads (oracle/make_golden.py gen_cns)."""
    prob = dg1d.CNS1D(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl)

    def mk(P):
        return dg1d.Op1D(w.x_left, w.x_right, w.n_elem, P, prob, solver=solver, cg_log=log)
    fine = mk(w.p_fine)
    if u0 is None:
        u0 = w.initial_state(fine.xi)
        dt = w.time_step(u0, quad.delta_of_degree(w.p_fine))
    res = []
    u = u0
    if w.mlsdc:
        h = sweeper.build_two_level(lambda lvl: mk(w.p_coarse if lvl == "coarse" else w.p_fine),
                                    sweeper.Rule("radau_right", w.m_coarse), sweeper.Rule("radau_right", w.m_fine))
        for s in range(w.n_steps):
            u = sweeper.run_mlsdc(h, u, s * dt, dt, w.n_cycles).u[-1].copy()
            res.append(u)
    else:
        rule = sweeper.Rule("radau_right", w.m_fine)
        for s in range(w.n_steps):
            u = sweeper.run_sdc(fine, rule, dt, w.scheme, u, s * dt, w.n_sweeps).u[-1].copy()
            res.append(u)
    return u0, dt, res


@pytest.mark.parametrize("case", ["cns_resolved", "cns_mlsdc", "cns_mlsdc_visc"])
def test_cns_oracle_pinned_to_reference(golden, case):
    """1-D CompressibleFlow (matrix coefficients): the
    oracle's block-Jacobi BiCGStab path reproduces the reference run with the
    same solver swapped in (identical iteration sequence), and the reference
    as shipped (SuperLU) to the conditioning of the acoustic system."""
    from paper_2504_18526_b200.configs import CNS_CASES
    G = golden["cns"]
    w = {c.name: c for c in CNS_CASES}[case]
    log = []
    fine_xi = quad.gll(w.p_fine + 1)[0]
    u0 = w.initial_state(fine_xi)   # the seeded IC on the oracle's own GLL nodes
    assert np.abs(u0 - G[f"{case}_u0"]).max() <= 1e-13 * np.abs(u0).max()
    assert abs(w.time_step(u0, quad.delta_of_degree(w.p_fine)) / float(G[f"{case}_dt"]) - 1.0) < 1e-13
    u0, dt, res = _cns_oracle_run(w, log, u0=G[f"{case}_u0"], dt=float(G[f"{case}_dt"]))
    assert [it for it, _ in log] == G[f"{case}_bicg_iters"].tolist()
    for s, u in enumerate(res):
        assert np.linalg.norm(u - G[f"{case}_bicg_u{s + 1}"]) / np.linalg.norm(u) < 1e-12
        assert np.linalg.norm(u - G[f"{case}_lu_u{s + 1}"]) / np.linalg.norm(u) < 5e-11


def test_source_terms_pinned_to_reference(golden):
    """Burgers with a source term (dgsem.py:328-347):
    the oracle restatement reproduces the reference's manufactured steady
    state, eval_rhs with the unsteady manufactured source, and two SI-MLSDC
    steps with the pinned PCG (identical iteration sequence)."""
    from paper_2504_18526_b200.configs import MANUFACTURED as w
    G = golden["sources"]
    nu0, ww = 0.05, 2 * np.pi

    def src_ss(x, t, u=None):
        return (2.0 + np.sin(ww * x)) * ww * np.cos(ww * x) + nu0 * ww * ww * np.sin(ww * x)
    op = dg1d.Op1D(-1.0, 1.0, 20, 12, dg1d.Burgers(nu0, source=src_ss, boundary=lambda t: (
        np.array([2.0 + np.sin(-ww)]), np.array([2.0 + np.sin(ww)]))), bc="dirichlet")
    assert np.abs(op.eval_rhs(G["ss_u"], 0.0) - G["ss_rhs"]).max() < 1e-9
    log = []

    def mk(P):
        return dg1d.Op1D(-1.0, 1.0, w.n_elem, P, dg1d.Burgers(w.nu, boundary=w.boundary, source=w.source),
                         bc="dirichlet", cg_log=log)
    fine = mk(w.p_fine)
    u0, dt = G["u0"], float(G["dt"])
    assert rel(fine.eval_rhs(u0, 0.3), G["rhs_t03"]) < 1e-12
    h = sweeper.build_two_level(lambda lvl: mk(w.p_coarse if lvl == "coarse" else w.p_fine),
                                sweeper.Rule("radau_right", w.m_coarse), sweeper.Rule("radau_right", w.m_fine))
    u = u0
    for s in (1, 2):
        n0 = len(log)
        u = sweeper.run_mlsdc(h, u, (s - 1) * dt, dt, w.n_cycles).u[-1].copy()
        assert [it for it, _ in log[n0:]] == G[f"mlsdc_pcg_iters{s}"].tolist()
        assert np.linalg.norm(u - G[f"mlsdc_pcg_u{s}"]) / np.linalg.norm(u) < 1e-12
        assert np.linalg.norm(u - G[f"mlsdc_lu_u{s}"]) / np.linalg.norm(u) < 1e-11


@pytest.mark.parametrize("case", ["sod_euler_av", "sod_ns_av"])
def test_cns_dirichlet_sod_pinned_to_reference(golden, case):
    """CompressibleFlow with Dirichlet faces (the oracle's matrix-coefficient
    Dirichlet SIP, dgsem.py:282-308) on the reference CLI's Sod tube with AV:
    operators and two SI-MLSDC steps with the identical BiCGStab sequence."""
    from paper_2504_18526_b200.configs import SOD_CASES
    G = golden["sod"]
    w = {c.name: c for c in SOD_CASES}[case]

    class Sod(dg1d.CNS1D):
        def __init__(self):
            super().__init__(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl)
            self.boundary = w.boundary
    log = []

    def mk(P):
        return dg1d.Op1D(0.0, 1.0, w.n_elem, P, Sod(), bc="dirichlet", av=w.av, cg_log=log)
    u0, dt = G[case + "_u0"], float(G[case + "_dt"])
    op = mk(w.p_fine)
    assert rel(op.apply_convection(u0, 0.0), G[case + "_conv"]) < 1e-13
    op.begin_slab(u0, 0.0, dt)
    assert rel(op.persson_viscosity(u0), G[case + "_nu_art"]) < 1e-13
    assert rel(op.eval_rhs(u0, 0.0), G[case + "_rhs"]) < 1e-12
    h = sweeper.build_two_level(lambda lvl: mk(w.p_coarse if lvl == "coarse" else w.p_fine),
                                sweeper.Rule("radau_right", w.m_coarse), sweeper.Rule("radau_right", w.m_fine))
    log.clear()
    u = u0
    for s in range(w.n_steps):
        u = sweeper.run_mlsdc(h, u, s * dt, dt, w.n_cycles).u[-1].copy()
        assert np.linalg.norm(u - G[f"{case}_bicg_u{s + 1}"]) / np.linalg.norm(u) < 1e-12
    assert [it for it, _ in log] == G[case + "_bicg_iters"].tolist()


def test_nodes_plus_t0_convention_against_reference():
    """node_convention = "nodes_plus_t0" (transfer.py:61-121): the product's temporal
    matrices and apply_temporal, and the oracle's two-level MLSDC steps, against
    the reference's own outputs (tests/golden/t0conv.npz)."""
    import os
    from oracle import sweeper as osw, workloads
    from paper_2504_18526_b200 import collocation, transfer
    from paper_2504_18526_b200.configs import CFG1 as w
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "t0conv.npz"))
    rules = [collocation.make_nodes("radau_right", M) for M in (w.m_coarse, w.m_fine)]
    for kind in ("embedded", "l2"):
        pair = transfer.build_temporal_transfer(rules[0], rules[1], kind, "nodes_plus_t0")
        for d in ("interp", "project", "restrict"):
            assert np.abs(pair.matrix(d) - G[f"{kind}_{d}"]).max() < 1e-12
    pair = transfer.build_temporal_transfer(rules[0], rules[1], "embedded", "nodes_plus_t0")
    assert np.abs(transfer.apply_temporal(pair, "interp", G["in_c"], G["in_u0"]) - G["ap_interp"]).max() < 1e-12
    assert np.abs(transfer.apply_temporal(pair, "project", G["in_f"], G["in_u0"]) - G["ap_project"]).max() < 1e-12
    assert np.abs(transfer.apply_temporal(pair, "restrict", G["in_f"]) - G["ap_restrict"]).max() < 1e-12
    with pytest.raises(ValueError):
        transfer.apply_temporal(pair, "interp", G["in_c"])            # needs the source u0
    with pytest.raises(ValueError):
        transfer.build_temporal_transfer(rules[0], rules[1], "embedded", "bogus")
    # nodes_only: plain matrix product
    p0 = transfer.build_temporal_transfer(rules[0], rules[1])
    assert np.abs(transfer.apply_temporal(p0, "interp", G["in_c"]) - p0.interp @ G["in_c"]).max() < 1e-14
    # the oracle sweeper in both solver modes
    dt = float(G["dt"])
    for solver, key, tol in (("lu", "lu_u", 1e-12), ("pcg", "pcg_u", 1e-12)):
        h, log = workloads.build_hierarchy(w, solver=solver, t0=True)
        for s in (1, 2):
            # every step from the reference's own input: with this convention a cfg1 step amplifies
            # an input perturbation ~100x (2e-14 after step 1 becomes 2e-12 after step 2 otherwise)
            u = G["u0"] if s == 1 else G[f"{key}1"]
            n0 = len(log)
            u = osw.run_mlsdc(h, u, (s - 1) * dt, dt, w.n_cycles, "fmg").u[-1].copy()
            assert np.linalg.norm(u - G[f"{key}{s}"]) / np.linalg.norm(G[f"{key}{s}"]) < tol
            if solver == "pcg":
                assert [it for it, _ in log[n0:]] == G[f"pcg_iters{s}"].tolist()
