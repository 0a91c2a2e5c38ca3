"""1-D compressible flow on the GPU (SURVEY 8a rows a2 ``CompressibleFlow``
and a6's matrix-valued SI coefficient): three conservative fields, 3x3
coefficients per node, the non-symmetric implicit system solved by the
pinned element-block-Jacobi BiCGStab (``oracle/cg.py``, ``csrc/cns1d.cu``).

Parity against the reference's own outputs (``tests/golden/cns.npz``,
``oracle/make_golden.py gen_cns``; the acoustic wave of ``problems.py:294-316``):
operators, a solve, the reference's test_dgsem.py:553-600 single-level SDC
set-ups and two SI-MLSDC workloads, each with the reference-with-BiCGStab
iteration sequence reproduced solve by solve."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from oracle import dg1d  # noqa: E402
from paper_2504_18526_b200.configs import CNS_CASES  # noqa: E402

CASES = {w.name: w for w in CNS_CASES}


def host(a):
    return a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)


def rel(a, b):
    a, b = host(a), host(b)
    return float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))


def l2rel(a, b):
    a = host(a).reshape(-1)
    b = host(b).reshape(-1)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def field_rel(a, b, nc=3):
    """max over the three fields of the per-field relative L2 error (rho is
    ~1e-2 and rho E ~2.5e3 on the acoustic wave)."""
    a = host(a).reshape(nc, -1)
    b = host(b).reshape(nc, -1)
    assert np.all(np.isfinite(a)), "non-finite GPU output"
    errs = []
    for c in range(nc):
        d, nb = np.linalg.norm(a[c] - b[c]), np.linalg.norm(b[c])
        errs.append(d / nb if nb > 0 else d)   # an all-zero reference field (Sod momentum): absolute norm
    return float(np.max(np.array(errs)))       # np.max propagates NaN


@pytest.fixture
def rt():
    from paper_2504_18526_b200.runtime import get_runtime
    r = get_runtime()
    r.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
    r.reset_status()   # latched flags of an earlier test must not leak into this one
    return r


def gpu_op(w, P, ne=None, eta=None):
    from paper_2504_18526_b200 import dgsem, problems
    prob = problems.CompressibleFlow(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta if eta is None else eta, Pr=w.prandtl)
    return dgsem.DGOperator(dgsem.Mesh1D(w.x_left, w.x_right, ne or w.n_elem, P), prob)


def test_cns_operators_vs_reference(rt, golden):
    """Convection (Rusanov on the system), eval_rhs with A_d(u), SIP with a
    given matrix field, the SI coefficient (dt/2) A_c^2 + A_d (golden
    operators.npz: 8 elements, P = 5, eta = 1e-3)."""
    from paper_2504_18526_b200 import dgsem, problems
    G = golden["operators"]
    op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, 8, 5), problems.CompressibleFlow(eta=1e-3))
    u = G["cns_u"]
    assert rel(op.apply_convection(u), G["cns_conv"]) < 1e-12
    assert rel(op.eval_rhs(u), G["cns_rhs"]) < 1e-12
    assert rel(op.apply_diffusion(G["cns_coeff"], u), G["cns_diff"]) < 1e-12
    c = op.modified_diffusion_matrix(u, 0.01, "si2")
    assert rel(op.coefficient_field(c), G["cns_modc"]) < 1e-13
    assert rel(op.apply_diffusion(c, u), op.apply_diffusion(G["cns_modc"], u)) < 1e-13


def test_cns_acoustic_operators_and_solve(rt, golden):
    G = golden["cns"]
    w = CASES["cns_resolved"]
    op = gpu_op(w, w.p_fine)
    u, dt = G["op_u"], float(G["cns_resolved_dt"])
    assert rel(op.apply_convection(u), G["op_conv"]) < 1e-11   # rho v^3 ~ 1e5 cancels to ~1e-1 in rho
    assert rel(op.eval_rhs(u), G["op_rhs"]) < 1e-11
    c = op.modified_diffusion_matrix(u, 0.5 * dt, "si2")
    assert rel(op.coefficient_field(c), G["op_modc"]) < 1e-13
    # C = (dt/2) A_c^2 has entries ~ H^2 dt ~ 1e5 acting on derivatives of fields
    # of very different scale (rho ~ 1e-2, rho E ~ 2.5e3): the SIP result
    # carries ~1e-10 relative roundoff in the reference itself
    assert rel(op.apply_diffusion(c, u), G["op_diff_modc"]) < 5e-10
    # the solve: same BiCGStab iteration count as the oracle, reference solution to conditioning
    log = []
    orc = dg1d.Op1D(w.x_left, w.x_right, w.n_elem, w.p_fine,
                    dg1d.CNS1D(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl), cg_log=log)
    xo = orc.implicit_solve(orc.modified_coeff(u, 0.5 * dt), 0.5 * dt, G["op_solve_rhs"])
    n0 = rt.status()[2]
    x = op.implicit_solve(c, 0.5 * dt, G["op_solve_rhs"])
    its = rt.cg_log()[0][n0:].tolist()
    assert its == [log[-1][0]], (its, log)
    assert field_rel(x, xo) < 1e-12
    assert field_rel(x, G["op_solve"]) < 1e-10   # vs SuperLU: conditioning-limited (rho field)
    # (M + a B[C]) x = M rhs checked matrix-free on the device
    m = np.tile(op.mass_node, 3 * w.n_elem)
    r = m * host(x) - 0.5 * dt * m * host(op.apply_diffusion(c, x)) - m * G["op_solve_rhs"]
    assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(m * G["op_solve_rhs"])
    # error behaviour: a = 0 returns rhs, b = 0 returns zeros
    assert rel(op.implicit_solve(c, 0.0, u), u) == 0.0
    z = op.implicit_solve(c, 0.5 * dt, np.zeros_like(u))
    assert float(host(z).__abs__().max()) == 0.0
    rt.raise_on_failure()


@pytest.mark.parametrize("case", ["cns_resolved", "cns_large"])
def test_cns_single_level_sdc(rt, golden, case):
    """The reference's own acoustic-wave tests (test_dgsem.py:553-600) as
    parity cases: run_sdc on 12 elements P = 7, si1 at CFL 0.8 and si2 at
    CFL 256 (cond ~1e10: the solve is conditioning-limited there)."""
    from paper_2504_18526_b200 import collocation, sdc
    G = golden["cns"]
    w = CASES[case]
    op = gpu_op(w, w.p_fine)
    rule = collocation.make_nodes("radau_right", w.m_fine)
    wts = collocation.make_weights(rule)
    dt = float(G[f"{case}_dt"])
    u = G[f"{case}_u0"]
    n0 = rt.status()[2]
    for s in range(w.n_steps):
        u = sdc.run_sdc(op, rule, wts, dt, w.scheme, u, s * dt, w.n_sweeps).u[-1].clone()
        tol = 1e-11 if case == "cns_resolved" else 1e-9   # cond ~1e10 at CFL 256
        assert field_rel(u, G[f"{case}_bicg_u{s + 1}"]) < tol
        # SuperLU vs BiCGStab differ by the conditioning of the acoustic system
        # (the reference with the two solvers differs by 1.1e-11 globally after 2 steps)
        assert field_rel(u, G[f"{case}_lu_u{s + 1}"]) < (2e-9 if case == "cns_resolved" else 5e-8)
    its = rt.cg_log()[0][n0:]
    ref = G[f"{case}_bicg_iters"]
    if case == "cns_resolved":
        assert its.tolist() == ref.tolist()
    else:   # cond ~1e10: roundoff moves the Krylov iterates (restarts), not the converged solution
        assert len(its) == len(ref) and (its > 0).all() and its.max() <= 1000
    rt.raise_on_failure()
    u3 = host(u).reshape(3, w.n_elem, -1)
    rho, vel = u3[0], u3[1] / u3[0]
    p = (w.gamma - 1.0) * (u3[2] - 0.5 * u3[1] * vel)
    assert (rho > 0).all() and (p > 0).all()


@pytest.mark.parametrize("case", ["cns_mlsdc", "cns_mlsdc_visc"])
def test_cns_mlsdc_steps(rt, golden, case):
    """Two-level SI-MLSDC (P 7/3, M 5/3 Euler-like; P 6/3, M 4/2 viscous):
    identical BiCGStab iteration sequence to the reference-with-BiCGStab,
    <= 1e-11 per field against it, and the SuperLU reference to the
    system's conditioning; CUDA-graph replay bitwise equal to eager."""
    from paper_2504_18526_b200 import mlsdc
    G = golden["cns"]
    w = CASES[case]
    h = mlsdc.build_p_hierarchy(lambda P: gpu_op(w, P), [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
    dt = float(G[f"{case}_dt"])
    u = G[f"{case}_u0"]
    n0 = rt.status()[2]
    for s in range(w.n_steps):
        u = mlsdc.run_mlsdc(h, u, s * dt, dt, w.n_cycles, strategy="fmg").u[-1].clone()
        assert field_rel(u, G[f"{case}_bicg_u{s + 1}"]) < 1e-11
        assert field_rel(u, G[f"{case}_lu_u{s + 1}"]) < 2e-9
    assert rt.cg_log()[0][n0:].tolist() == G[f"{case}_bicg_iters"].tolist()
    rt.raise_on_failure()
    g = mlsdc.SlabGraph(h, G[f"{case}_u0"], 0.0, dt, w.n_cycles, "fmg")
    g.step()
    eager = mlsdc.run_mlsdc(h, G[f"{case}_u0"], 0.0, dt, w.n_cycles, strategy="fmg").u[-1]
    assert np.array_equal(host(g.u), host(eager))


def test_cns_smooth_start_all_fields(rt):
    """smooth_start works for any ncomp (dgsem.py:574-589): interface averaging per field,
    periodic wrap included, against the reference's formula restated on the host."""
    from paper_2504_18526_b200 import dgsem
    w = CASES["cns_resolved"]
    op = gpu_op(w, w.p_fine)
    rng = np.random.default_rng(3)
    u = w.initial_state(op.ref_nodes) + 0.01 * rng.standard_normal(op.ndof)
    u3 = u.reshape(3, op.mesh.n_elem, op.p1).copy()
    mean = 0.5 * (u3[:, :-1, -1] + u3[:, 1:, 0])
    u3[:, :-1, -1] = mean
    u3[:, 1:, 0] = mean
    wrap = 0.5 * (u3[:, -1, -1] + u3[:, 0, 0])
    u3[:, -1, -1] = wrap
    u3[:, 0, 0] = wrap
    got = dgsem.smooth_start(op, u).cpu().numpy()
    assert np.abs(got - u3.reshape(-1)).max() == 0.0


SOD = None


def sod_op(w, P):
    from paper_2504_18526_b200 import dgsem, problems
    prob = problems.CompressibleFlow(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl, boundary=w.boundary)
    av = dgsem.ArtificialViscosityParams(*w.av) if w.av else None
    return dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, w.n_elem, P, bc="dirichlet"), prob, av=av)


@pytest.mark.parametrize("case", ["sod_euler_av", "sod_ns_av"])
def test_cns_sod_dirichlet(rt, golden, case):
    """CompressibleFlow with Dirichlet faces: the reference CLI's Sod shock
    tube (cli.py:766-772) with Persson-Peraire viscosity -- operators with the
    boundary states, the affine matrix SIP and its implicit solve, and two
    SI-MLSDC steps with the reference-with-BiCGStab iteration sequence."""
    from paper_2504_18526_b200 import mlsdc
    from paper_2504_18526_b200.configs import SOD_CASES
    G = golden["sod"]
    w = {c.name: c for c in SOD_CASES}[case]
    u0, dt = G[case + "_u0"], float(G[case + "_dt"])
    op = sod_op(w, w.p_fine)
    assert rel(op.apply_convection(u0, 0.0), G[case + "_conv"]) < 1e-12
    op.begin_slab(u0, 0.0, dt)
    assert rel(op.persson_viscosity(u0), G[case + "_nu_art"]) < 1e-12
    assert rel(op.eval_rhs(u0, 0.0), G[case + "_rhs"]) < 1e-11
    c = op.modified_diffusion_matrix(u0, 0.5 * dt, "si2")
    assert rel(op.coefficient_field(c), G[case + "_modc"]) < 1e-13
    assert rel(op.apply_diffusion(c, u0, 0.0), G[case + "_diff"]) < 1e-11
    assert field_rel(op.implicit_solve(c, 0.5 * dt, u0, 0.0), G[case + "_solve"]) < 1e-12
    h = mlsdc.build_p_hierarchy(lambda P: sod_op(w, P), [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
    n0 = rt.status()[2]
    u = u0
    for s in range(w.n_steps):
        u = mlsdc.run_mlsdc(h, u, s * dt, dt, w.n_cycles, strategy="fmg").u[-1].clone()
        assert field_rel(u, G[f"{case}_bicg_u{s + 1}"]) < 1e-11
        assert field_rel(u, G[f"{case}_lu_u{s + 1}"]) < 1e-10
    assert rt.cg_log()[0][n0:].tolist() == G[case + "_bicg_iters"].tolist()
    rt.raise_on_failure()


@pytest.mark.parametrize("bc", ["periodic", "dirichlet"])
def test_cns_multi_cta_cluster_solve(rt, bc):
    """The BiCGStab cluster path with K > 1 CTAs (face halo through DSMEM,
    rank-ordered cluster reductions): 100 elements at P = 7 span 4 CTAs.
    Same iteration count as the oracle and <= 1e-12 per field; periodic and
    Dirichlet (Sod states) faces."""
    from paper_2504_18526_b200 import dgsem, problems
    from paper_2504_18526_b200.configs import SOD_CASES
    w = CASES["cns_mlsdc"]
    ne, P = 100, 7
    if bc == "periodic":
        prob_g = problems.CompressibleFlow(eta=2e-4)
        prob_o = dg1d.CNS1D(eta=2e-4)
        op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, ne, P), prob_g)
        u = AcousticState(w, ne, P, op.ref_nodes)
    else:
        sod = SOD_CASES[0]

        class Sod(dg1d.CNS1D):
            def __init__(self):
                super().__init__(eta=2e-4)
                self.boundary = sod.boundary
        prob_g = problems.CompressibleFlow(eta=2e-4, boundary=sod.boundary)
        prob_o = Sod()
        op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, ne, P, bc="dirichlet"), prob_g)
        u = host(op.nodal_field(lambda x: 0.5 * (sod.initial(x - 0.01) + sod.initial(x + 0.01)))).copy()
    log = []
    orc = dg1d.Op1D(0.0, 1.0, ne, P, prob_o, bc=bc, cg_log=log)
    lam = dgsem.max_wave_speed(op, u)
    a = 0.4 * dgsem.dt_from_cfl(2.0, 1.0 / ne, lam, P)
    c = op.modified_diffusion_matrix(u, a, "si2")
    rhs = u * (1.0 + 1e-3 * np.sin(np.arange(u.size)))
    n0 = rt.status()[2]
    x = op.implicit_solve(c, a, rhs, 0.0)
    xo = orc.implicit_solve(orc.modified_coeff(u, a), a, rhs, 0.0)
    assert rt.cg_log()[0][n0:].tolist() == [log[-1][0]]
    assert field_rel(x, xo) < 1e-12
    rt.raise_on_failure()


def AcousticState(w, ne, P, nodes):
    import dataclasses
    return dataclasses.replace(w, n_elem=ne, p_fine=P).initial_state(nodes)


@pytest.mark.parametrize("ne,P", [(700, 7), (1100, 3)])
def test_cns_grid_mode_beyond_one_cluster(rt, ne, P):
    """Levels above 16 CTAs x 256 nodes (dgsem.py:503-533 solves any size): the cluster BiCGStab
    as a cooperative launch (face-node halo and reduction slots through global memory, grid
    barriers).  Same iteration count as the oracle's pinned BiCGStab, <= 1e-11 per field."""
    from paper_2504_18526_b200 import dgsem, problems
    w = CASES["cns_resolved"]
    op = dgsem.DGOperator(dgsem.Mesh1D(w.x_left, w.x_right, ne, P),
                          problems.CompressibleFlow(gamma=w.gamma, R_gas=w.R_gas, eta=1e-3, Pr=w.prandtl))
    assert ne * (P + 1) > 16 * 256
    log = []
    orc = dg1d.Op1D(w.x_left, w.x_right, ne, P, dg1d.CNS1D(gamma=w.gamma, R_gas=w.R_gas, eta=1e-3, Pr=w.prandtl),
                    cg_log=log)
    x = np.asarray(op.mesh.nodes_x)
    L = w.x_right - w.x_left
    s = np.sin(2 * np.pi * (x - w.x_left) / L)
    rho, v, p = 1.2 * (1.0 + 0.05 * s), 30.0 * s, 1.0e5 * (1.0 + 0.05 * s)
    u = np.stack([rho, rho * v, p / (w.gamma - 1.0) + 0.5 * rho * v * v]).reshape(-1)
    dt = 0.2 * (L / ne) / (P + 1) ** 2 / 350.0
    rhs = u * (1.0 + 0.01 * np.cos(3 * 2 * np.pi * np.tile(x.reshape(-1), 3) / L))
    n0 = rt.status()[2]
    xg = op.implicit_solve(op.modified_diffusion_matrix(u, dt, "si2"), dt, rhs)
    xo = orc.implicit_solve(orc.modified_coeff(u, dt), dt, rhs)
    its = rt.cg_log()[0][n0:].tolist()
    assert its == [log[-1][0]], (its, log[-1])
    assert field_rel(xg, xo) < 1e-11
    rt.raise_on_failure()
