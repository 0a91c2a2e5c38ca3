"""Dirichlet faces with time-dependent trace data on the GPU (SURVEY 8a rows
a1/a3/a4 bc branches, 8f.1): the paper's Burgers moving front against the
reference's own outputs (tests/golden/dirichlet.npz, oracle/make_golden.py):
operators at two times, implicit solves of the affine SIP system (identical
CG iterations to the oracle's pinned PCG), a single-level SDC slab, two
SI-MLSDC steps with the reference-with-PCG iteration sequence, and the
under-resolved front with Persson-Peraire viscosity."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from oracle import dg1d  # noqa: E402
from paper_2504_18526_b200.configs import FRONT, FRONT_AV, burgers_front_boundary  # noqa: E402


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def l2rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def rt():
    from paper_2504_18526_b200.runtime import get_runtime
    r = get_runtime()
    r.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
    return r


def gpu_op(w, P, ne=None):
    from paper_2504_18526_b200 import dgsem, problems
    prob, _ = problems.burgers_front_problem(w.nu)
    av = dgsem.ArtificialViscosityParams(*w.av) if w.av else None
    return dgsem.DGOperator(dgsem.Mesh1D(-1.0, 1.0, ne or w.n_elem, P, bc="dirichlet"), prob, av=av)


def test_dirichlet_operators_and_solves(rt, golden):
    G = golden["dirichlet"]
    w = FRONT
    op = gpu_op(w, w.p_fine)
    dt, us = float(G["dt"]), G["us"]
    log = []
    orc = dg1d.Op1D(-1.0, 1.0, w.n_elem, w.p_fine, dg1d.Burgers(w.nu, boundary=burgers_front_boundary(w.nu)),
                    bc="dirichlet", solver="pcg", cg_log=log)
    for j in (0, 1):
        t = float(G[f"t{j}"])
        assert rel(op.apply_convection(us, t), G[f"conv{j}"]) < 1e-12
        c = op.modified_diffusion_matrix(us, 0.4 * dt, "si2")
        assert rel(op.coefficient_field(c).reshape(-1), np.asarray(G[f"coef{j}"]).reshape(-1)) < 1e-14
        assert rel(op.apply_diffusion(c, us, t), G[f"diff{j}"]) < 1e-12
        assert rel(op.eval_rhs(us, t), G[f"rhs{j}"]) < 1e-10
        n0 = rt.status()[2]
        x = op.implicit_solve(c, 0.4 * dt, us, t)
        orc.implicit_solve(orc.modified_coeff(us, 0.4 * dt), 0.4 * dt, us, t)
        assert rt.cg_log()[0][n0:].tolist() == [log[-1][0]]
        assert l2rel(x, G[f"solve{j}"]) < 1e-11
    # a time without registered trace data is an error, never a silent periodic fallback
    out = op.rt.empty(op.ndof)
    rc = op.lib.sisdc_apply_convection(op.h, op.rt.to_device(us).data_ptr(), 12345.678, out.data_ptr())
    with pytest.raises(ValueError):
        op.rt.check(rc, "apply_convection")


def test_dirichlet_sdc_and_mlsdc(rt, golden):
    from paper_2504_18526_b200 import collocation, mlsdc, sdc
    G = golden["dirichlet"]
    w = FRONT
    dt = float(G["dt"])
    op = gpu_op(w, w.p_fine)
    rule = collocation.make_nodes("radau_right", w.m_fine)
    s = sdc.run_sdc(op, rule, collocation.make_weights(rule), dt, "si2", G["u0"], 0.0, 2)
    assert l2rel(s.u, G["sdc2_u"]) < 1e-11
    h = mlsdc.build_p_hierarchy(lambda P: gpu_op(w, P), [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
    u = G["u0"]
    for step in (1, 2):
        n0 = rt.status()[2]
        sol = mlsdc.run_mlsdc(h, u, (step - 1) * dt, dt, w.n_cycles, strategy="fmg")
        assert rt.cg_log()[0][n0:].tolist() == G[f"mlsdc_pcg_iters{step}"].tolist()
        assert l2rel(sol.u[-1], G[f"mlsdc_pcg_u{step}"]) < 1e-11
        # the reference as shipped (SuperLU + defect iteration to 1e-12 ||b||)
        assert l2rel(sol.u[-1], G[f"mlsdc_lu_u{step}"]) < 1e-9
        u = sol.u[-1].clone()
    rt.raise_on_failure()
    with pytest.raises(ValueError):
        mlsdc.SlabGraph(h, G["u0"], 0.0, dt, w.n_cycles, "fmg")


def test_dirichlet_front_with_av(rt, golden):
    from paper_2504_18526_b200 import mlsdc
    G = golden["dirichlet"]
    w = FRONT_AV
    h = mlsdc.build_p_hierarchy(lambda P: gpu_op(w, P), [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
    assert rel(h.fine.ctx.persson_viscosity(G["av_u0"]), G["av_nu_art"]) < 1e-12
    n0 = rt.status()[2]
    sol = mlsdc.run_mlsdc(h, G["av_u0"], 0.0, float(G["av_dt"]), w.n_cycles, strategy="fmg")
    assert rt.cg_log()[0][n0:].tolist() == G["av_mlsdc_pcg_iters1"].tolist()
    assert l2rel(sol.u[-1], G["av_mlsdc_pcg_u1"]) < 1e-11
    rt.raise_on_failure()
