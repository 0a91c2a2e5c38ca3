"""Size-independent properties at BASELINE.json's FULL 2-D sizes (configs[3]: 256^2 elements, P = 7,
16.8M DOF; configs[4]: 1024^2, 268M DOF), where the CPU restatement cannot follow: conservation of the
convective and viscous operators, symmetry / definiteness of the SIP operator in the mass inner
product, the implicit solve checked by applying the operator to its solution, the tensor-core viscous
kernel against the line kernel, and the element-row partition against the single domain (bitwise
operators, identical CG iteration sequence of one SI-MLSDC step)."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_2504_18526_b200.configs import CFG3, CFG4, CFG5  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2504_18526_b200.runtime import get_runtime
    r = get_runtime()
    r.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
    return r


def _op(w, P, partition=None):
    from paper_2504_18526_b200 import dgsem2d
    mesh = dgsem2d.Mesh2D(0.0, w.length, 0.0, w.length, w.nex, w.ney, P)
    return dgsem2d.DGOperator2D(mesh, w.gpu_problem(), partition=partition)


def _mass(op, torch):
    """Lumped mass (dy/2 w_j)(dx/2 w_i) per node of an element, device (P+1, P+1)."""
    w1 = torch.as_tensor(op.mesh_weights if hasattr(op, "mesh_weights") else _gll_w(op), device=op.rt.device)
    return (0.5 * op.mesh.dy * w1)[:, None] * (0.5 * op.mesh.dx * w1)[None, :]


def _gll_w(op):
    from paper_2504_18526_b200.collocation import gauss_lobatto
    return gauss_lobatto(op.p1)[1]


def test_cfg4_full_size_operator_properties(rt, monkeypatch):
    import torch
    w = CFG4
    op = _op(w, w.p_fine)
    X, Y = op.mesh.nodes_xy
    u = rt.to_device(w.initial_state(X, Y))
    m = _mass(op, torch)
    scale = float((op.as_nodes(u).abs() * m).sum())

    def integral(v):   # per-field integrals over the periodic domain
        return (op.as_nodes(v) * m).sum(dim=(1, 2, 3, 4))
    # conservation: the weak convective and viscous operators integrate to zero on a periodic mesh
    assert float(integral(op.apply_convection(u)).abs().max()) < 1e-11 * scale
    visc = op.apply_viscous(u).clone()
    assert float(integral(visc).abs().max()) < 1e-11 * scale
    # the tensor-core viscous kernel against the line kernel at full size: bitwise
    monkeypatch.setenv("SISDC_VISC_LINE", "1")
    assert bool((op.apply_viscous(u) == visc).all())
    monkeypatch.delenv("SISDC_VISC_LINE")
    # SIP with the SI coefficient: symmetric and negative semi-definite in the mass inner product
    a = 1e-4   # ~ dt_m / 2 of the workload's step (dt ~ 2e-4)
    c = op.modified_diffusion_matrix(u, a, "si2")
    g = torch.Generator(device=rt.device).manual_seed(5)
    x = torch.randn(op.ndof, dtype=torch.float64, device=rt.device, generator=g)
    y = torch.randn(op.ndof, dtype=torch.float64, device=rt.device, generator=g)
    dx, dy = op.apply_diffusion(c, x).clone(), op.apply_diffusion(c, y).clone()
    ydx = float((op.as_nodes(y) * op.as_nodes(dx) * m).sum())
    xdy = float((op.as_nodes(x) * op.as_nodes(dy) * m).sum())
    assert abs(ydx - xdy) < 1e-10 * abs(ydx)
    assert float((op.as_nodes(x) * op.as_nodes(dx) * m).sum()) < 0.0
    # the implicit solve, checked through the operator: (I - a D[c]) x = rhs
    n0 = rt.status()[2]
    sol = op.implicit_solve(c, a, u).clone()
    its = rt.cg_log()[0][n0:].tolist()
    assert len(its) == 1 and 0 < its[0] < 1000
    res = sol - a * op.apply_diffusion(c, sol) - u
    assert float(res.norm() / u.norm()) < 1e-11
    rt.raise_on_failure()


def test_cfg4_full_size_partition_vs_single_domain(rt):
    """Element-row partition at the full cfg4 size: eval_rhs bitwise, and one SI-MLSDC step with the
    identical CG iteration sequence (fused fine and coarse passes, fused setup) and <= 1e-11."""
    from paper_2504_18526_b200 import dgsem, dgsem2d, mlsdc
    w = CFG4

    def step(partition):
        h = mlsdc.build_p_hierarchy(lambda P: _op(w, P, partition), [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
        fine = h.fine.ctx
        X, Y = fine.mesh.nodes_xy
        u0 = w.initial_state(X, Y)
        dt = w.time_step(u0, dgsem.compute_delta(w.p_fine))
        us = fine.scatter(u0)
        rhs = fine.gather(fine.eval_rhs(us)).reshape(-1)
        n0 = rt.status()[2]
        sol = mlsdc.run_mlsdc(h, us, 0.0, dt, w.n_cycles, strategy="fmg")
        rt.raise_on_failure()
        return rhs, fine.gather(sol.u[-1]).reshape(-1), rt.cg_log()[0][n0:].tolist()

    rhs1, u1, its1 = step(None)
    rhs4, u4, its4 = step(dgsem2d.Partition(4))
    assert np.array_equal(rhs1, rhs4)
    assert its4 == its1
    assert np.linalg.norm(u4 - u1) / np.linalg.norm(u1) < 1e-11


def test_cfg5_full_size_conservation_and_partition(rt):
    """BASELINE configs[4] (268M fine DOF): conservation of the full right-hand side and the 8-way
    element-row partition (the 8-GPU layout) against the single domain, bitwise."""
    import torch
    from paper_2504_18526_b200 import dgsem2d
    w = CFG5
    op = _op(w, w.p_fine)
    X, Y = op.mesh.nodes_xy
    u0 = w.initial_state(X, Y)
    del X, Y
    u = rt.to_device(u0)
    m = _mass(op, torch)
    r1 = op.eval_rhs(u)
    scale = float((op.as_nodes(u).abs() * m).sum())
    assert float((op.as_nodes(r1) * m).sum(dim=(1, 2, 3, 4)).abs().max()) < 1e-11 * scale
    ref = r1.cpu().numpy().reshape(-1)
    del r1, u, op
    torch.cuda.empty_cache()
    part = _op(w, w.p_fine, dgsem2d.Partition(8))
    got = part.gather(part.eval_rhs(part.scatter(u0))).reshape(-1)
    assert np.array_equal(got, ref)
    rt.raise_on_failure()


@pytest.mark.parametrize("w", [CFG3, CFG4], ids=["cfg3", "cfg4"])
def test_full_size_step_conserves_the_field_integrals(rt, w):
    """One SI-MLSDC step at the full size of BASELINE configs[2] (Euler vortex, 128^2) and configs[3]
    (NS shear layer, 256^2): every operator of the sweep is conservative on the periodic mesh
    (convection, viscous / SI diffusion inside the implicit solve, FAS-corrected transfers), so the
    integrals of rho, rho u, rho v, rho E are those of the initial state."""
    import torch
    from paper_2504_18526_b200 import dgsem, mlsdc
    h = mlsdc.build_p_hierarchy(lambda P: _op(w, P), [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
    fine = h.fine.ctx
    X, Y = fine.mesh.nodes_xy
    u0 = rt.to_device(w.initial_state(X, Y))
    dt = w.time_step(u0.cpu().numpy(), dgsem.compute_delta(w.p_fine))
    m = _mass(fine, torch)
    i0 = (fine.as_nodes(u0) * m).sum(dim=(1, 2, 3, 4))
    sol = mlsdc.run_mlsdc(h, u0, 0.0, dt, w.n_cycles, strategy="fmg")
    rt.raise_on_failure()
    u1 = sol.u[-1]
    assert float((u1 - u0).abs().max()) > 0.0
    i1 = (fine.as_nodes(u1) * m).sum(dim=(1, 2, 3, 4))
    scale = (fine.as_nodes(u0).abs() * m).sum(dim=(1, 2, 3, 4)).max()
    assert float((i1 - i0).abs().max() / scale) < 1e-12
