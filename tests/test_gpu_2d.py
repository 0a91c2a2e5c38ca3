"""2-D CUDA path vs the 2-D CPU restatement (oracle/dg2d.py) on small meshes.

The reference is 1-D only, so 2-D parity is against the builder's own
restatement ("parity unpinned by the reference"); the restatement
itself is pinned to the reference's 1-D goldens on y-invariant data
(tests/test_oracle2d.py).
"""
import dataclasses

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from oracle import dg2d, sweeper as osw, workloads  # noqa: E402
from paper_2504_18526_b200.configs import CFG3, CFG4  # noqa: E402


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def small(w, nex, ney=None):
    return dataclasses.replace(w, nex=nex, ney=ney or nex)


def pair(w, P):
    from paper_2504_18526_b200 import dgsem2d
    L = w.length
    mesh = dgsem2d.Mesh2D(0.0, L, 0.0, L, w.nex, w.ney, P)
    op = dgsem2d.DGOperator2D(mesh, dgsem2d.CompressibleEuler2D(w.gamma, w.nu))
    orc = dg2d.Op2D(0.0, L, 0.0, L, w.nex, w.ney, P, dg2d.Euler2D(w.gamma, w.nu))
    X, Y = mesh.nodes_xy
    return op, orc, w.initial_state(X, Y)


@pytest.fixture(scope="module")
def rt():
    from paper_2504_18526_b200.runtime import get_runtime
    r = get_runtime()
    r.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
    return r


@pytest.mark.parametrize("w,P", [(small(CFG3, 4), 7), (small(CFG4, 3, 5), 7), (small(CFG3, 6), 3)])
def test_operators_2d(rt, w, P):
    op, orc, u = pair(w, P)
    assert rel(op.apply_convection(u), orc.apply_convection(u)) < 1e-12
    fld = 0.01 + 0.01 * np.random.default_rng(1).random(w.nex * w.ney * (P + 1) ** 2)
    assert rel(op.apply_diffusion(fld, u), orc.apply_diffusion(fld, u)) < 1e-12
    assert rel(op.apply_diffusion(0.0123, u), orc.apply_diffusion(0.0123, u)) < 1e-12
    if w.nu > 0:
        assert rel(op.eval_rhs(u), orc.eval_rhs(u)) < 1e-12
    c = op.modified_diffusion_matrix(u, 3e-3, "si2")
    assert rel(op.coefficient_field(c), np.asarray(orc.modified_coeff(u, 3e-3)).reshape(-1)) < 1e-14


@pytest.mark.parametrize("w,P", [(small(CFG3, 4), 7), (small(CFG4, 6), 3)])
def test_implicit_solve_2d(rt, w, P):
    op, orc, u = pair(w, P)
    c = op.modified_diffusion_matrix(u, 2e-3, "si2")
    co = orc.modified_coeff(u, 2e-3)
    n0 = rt.status()[2]
    x = op.implicit_solve(c, 2e-3, u)
    xo = orc.implicit_solve(co, 2e-3, u)
    its = rt.cg_log()[0][n0:].tolist()
    assert its == [orc.cg_log[-1][0]]
    assert rel(x, xo) < 1e-13


def test_mlsdc_step_2d(rt):
    """One SI-MLSDC step of a small vortex (4x4 elements, P 7/3, M 4/2):
    GPU vs the 2-D restatement, identical CG iteration sequence."""
    from paper_2504_18526_b200 import dgsem, dgsem2d, mlsdc
    w = small(CFG3, 4)
    L = w.length
    mk = lambda P: dgsem2d.DGOperator2D(dgsem2d.Mesh2D(0.0, L, 0.0, L, w.nex, w.ney, P),
                                        dgsem2d.CompressibleEuler2D(w.gamma, w.nu))
    h = mlsdc.build_p_hierarchy(mk, [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
    X, Y = h.fine.ctx.mesh.nodes_xy
    u0 = w.initial_state(X, Y)
    dt = w.time_step(u0, dgsem.compute_delta(w.p_fine))
    n0 = rt.status()[2]
    sol = mlsdc.run_mlsdc(h, u0, 0.0, dt, w.n_cycles, strategy="fmg")
    its = rt.cg_log()[0][n0:].tolist()
    oh, log = workloads.build_hierarchy_2d(lambda: dg2d.Euler2D(w.gamma, w.nu), 0.0, L, 0.0, L, w.nex, w.ney,
                                           w.p_coarse, w.p_fine, w.m_coarse, w.m_fine)
    so = osw.run_mlsdc(oh, u0, 0.0, dt, w.n_cycles, "fmg")
    ref = so.u[-1]
    assert np.linalg.norm(sol.u[-1].cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-11
    assert its == [i for i, _ in log]
    rt.raise_on_failure()
