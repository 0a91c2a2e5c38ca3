"""Burgers with a source term on the GPU path (SURVEY 8a rows a2 ``Burgers``
``source`` and a5 ``apply_source``, ``dgsem.py:328-347``): the source is the
reference's host callable src(x, t, u3), evaluated on the host at the node
coordinates and added to f on the device wherever the reference's eval_rhs
includes it (node caches, fresh FAS evaluations).  Parity against the
reference's outputs (tests/golden/sources.npz): its manufactured steady state
(test_dgsem.py:365-380), eval_rhs / apply_source of an unsteady manufactured
solution, a single-level SDC slab and two SI-MLSDC steps with the
reference-with-PCG iteration sequence."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_2504_18526_b200.configs import MANUFACTURED as W  # noqa: E402


def host(a):
    return a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)


def rel(a, b):
    a, b = host(a), host(b)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def l2rel(a, b):
    a, b = host(a).reshape(-1), host(b).reshape(-1)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture
def rt():
    from paper_2504_18526_b200.runtime import get_runtime
    r = get_runtime()
    r.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
    r.reset_status()
    return r


def gpu_op(P, tabulated=False):
    from paper_2504_18526_b200 import dgsem, problems
    return dgsem.DGOperator(dgsem.Mesh1D(-1.0, 1.0, W.n_elem, P, bc="dirichlet"),
                            problems.Burgers(W.nu, source=W.source, boundary=W.boundary,
                                             source_depends_on_state=not tabulated))


def test_source_steady_state_and_rhs(rt, golden):
    from paper_2504_18526_b200 import dgsem, problems
    G = golden["sources"]
    nu0, ww = 0.05, 2 * np.pi

    def src_ss(x, t, u=None):
        return (2.0 + np.sin(ww * x)) * ww * np.cos(ww * x) + nu0 * ww * ww * np.sin(ww * x)
    op = dgsem.DGOperator(dgsem.Mesh1D(-1.0, 1.0, 20, 12, bc="dirichlet"), problems.Burgers(
        nu0, source=src_ss, boundary=lambda t: (np.array([2.0 + np.sin(-ww)]), np.array([2.0 + np.sin(ww)]))))
    r = op.eval_rhs(G["ss_u"], 0.0)
    assert float(host(r).__abs__().max()) < 1e-8          # the reference test's own bound
    assert rel(r, G["ss_rhs"]) < 1e-9
    fine = gpu_op(W.p_fine)
    assert rel(fine.eval_rhs(G["u0"], 0.3), G["rhs_t03"]) < 1e-12
    assert rel(fine.apply_source(G["u0"], 0.3), G["src_t03"]) < 1e-15
    # a non-finite source value is reported like a non-finite rhs (dgsem.py:348-351)
    from paper_2504_18526_b200._lib import SolverError
    bad = dgsem.DGOperator(dgsem.Mesh1D(-1.0, 1.0, 4, 3, bc="dirichlet"), problems.Burgers(
        0.01, source=lambda x, t, u=None: np.where(x > 0.6, np.nan, 0.0), boundary=W.boundary))
    with pytest.raises(SolverError, match="element 3"):
        bad.eval_rhs(np.ones(bad.ndof), 0.0)


def test_source_sdc_and_mlsdc(rt, golden):
    from paper_2504_18526_b200 import collocation, mlsdc, sdc
    G = golden["sources"]
    dt = float(G["dt"])
    op = gpu_op(W.p_fine)
    rule = collocation.make_nodes("radau_right", W.m_fine)
    s = sdc.run_sdc(op, rule, collocation.make_weights(rule), dt, "si2", G["u0"], 0.0, 2)
    assert l2rel(s.u, G["sdc2_u"]) < 1e-11
    assert rel(s.f, G["sdc2_f"]) < 1e-8   # f amplifies state roundoff by ||D[nu]|| (as in test_gpu_parity)
    h = mlsdc.build_p_hierarchy(gpu_op, [W.p_coarse, W.p_fine], [W.m_coarse, W.m_fine])
    u = G["u0"]
    for step in (1, 2):
        n0 = rt.status()[2]
        sol = mlsdc.run_mlsdc(h, u, (step - 1) * dt, dt, W.n_cycles, strategy="fmg")
        assert rt.cg_log()[0][n0:].tolist() == G[f"mlsdc_pcg_iters{step}"].tolist()
        assert l2rel(sol.u[-1], G[f"mlsdc_pcg_u{step}"]) < 1e-11
        assert l2rel(sol.u[-1], G[f"mlsdc_lu_u{step}"]) < 1e-10
        u = sol.u[-1].clone()
    rt.raise_on_failure()
    assert l2rel(u, G["exact_t2"]) < 1e-4   # the manufactured solution itself
    with pytest.raises(ValueError, match="cannot be captured"):
        mlsdc.SlabGraph(h, G["u0"], 0.0, dt, W.n_cycles, "fmg")


def test_tabulated_source_keeps_the_state_on_the_device(rt, golden):
    """A known forcing src(x, t) (``source_depends_on_state=False``) is tabulated per node time on the
    device: the callable never sees the state (it receives None), and the SI-MLSDC steps reproduce
    the same reference goldens with the identical CG iteration sequence."""
    from paper_2504_18526_b200 import mlsdc
    G = golden["sources"]
    dt = float(G["dt"])
    seen = []

    def src(x, t, u=None):
        seen.append(u)
        return W.source(x, t, None)
    from paper_2504_18526_b200 import dgsem, problems
    mk = lambda P: dgsem.DGOperator(dgsem.Mesh1D(-1.0, 1.0, W.n_elem, P, bc="dirichlet"), problems.Burgers(
        W.nu, source=src, boundary=W.boundary, source_depends_on_state=False))
    h = mlsdc.build_p_hierarchy(mk, [W.p_coarse, W.p_fine], [W.m_coarse, W.m_fine])
    assert h.fine.ctx.source_tabulated
    u = G["u0"]
    for step in (1, 2):
        n0 = rt.status()[2]
        sol = mlsdc.run_mlsdc(h, u, (step - 1) * dt, dt, W.n_cycles, strategy="fmg")
        assert rt.cg_log()[0][n0:].tolist() == G[f"mlsdc_pcg_iters{step}"].tolist()
        assert l2rel(sol.u[-1], G[f"mlsdc_pcg_u{step}"]) < 1e-11
        u = sol.u[-1].clone()
    rt.raise_on_failure()
    assert seen and all(s is None for s in seen)
    # one table per distinct node time of the slab and level, not one host evaluation per use
    assert len(seen) <= 2 * (W.m_fine + W.m_coarse + 2)
    assert rel(gpu_op(W.p_fine, tabulated=True).apply_source(G["u0"], 0.3), G["src_t03"]) < 1e-15
