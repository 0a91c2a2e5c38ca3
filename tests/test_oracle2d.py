"""The 2-D restatement against the reference's own 1-D goldens (y-invariant
data) and basic 2-D identities (no GPU)."""
import numpy as np

from oracle import dg2d


def rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def test_y_invariant_reduces_to_reference_1d(golden):
    G = golden["operators"]
    ne, P, ney = 64, 8, 3
    op = dg2d.Op2D(0.0, 2 * np.pi, 0.0, 1.0, ne, ney, P, dg2d.Burgers2D(5e-3))
    u1, fld1 = G["cfg2_P8_u"], G["cfg2_P8_fld"]
    u2 = np.broadcast_to(u1.reshape(1, 1, ne, 1, P + 1), (1, ney, ne, P + 1, P + 1)).reshape(-1)
    C2 = np.broadcast_to(fld1.reshape(1, ne, 1, P + 1), (ney, ne, P + 1, P + 1))
    c2 = op.apply_convection(u2).reshape(1, ney, ne, P + 1, P + 1)
    d2 = op.apply_diffusion(C2, u2).reshape(1, ney, ne, P + 1, P + 1)
    for j in range(ney):
        for k in range(P + 1):
            assert rel(c2[0, j, :, k, :].reshape(-1), G["cfg2_P8_conv"]) < 1e-13
            assert rel(d2[0, j, :, k, :].reshape(-1), G["cfg2_P8_diff_field"]) < 1e-13
    # the implicit solve of a y-invariant rhs is y-invariant and equals the 1-D LU solve
    op2 = dg2d.Op2D(0.0, 2 * np.pi, 0.0, 1.0, ne, 2, P, dg2d.Burgers2D(5e-3))
    rhs1 = G["cfg2_P8_solve_rhs"]
    rhs2 = np.broadcast_to(rhs1.reshape(1, 1, ne, 1, P + 1), (1, 2, ne, P + 1, P + 1)).reshape(-1)
    C2b = np.broadcast_to(fld1.reshape(1, ne, 1, P + 1), (2, ne, P + 1, P + 1))
    x2 = op2.implicit_solve(C2b, 0.0123, rhs2).reshape(1, 2, ne, P + 1, P + 1)
    assert rel(x2[0, 1, :, 4, :].reshape(-1), G["cfg2_P8_solve_field"]) < 1e-12


def test_sip_symmetric_and_dense_solve():
    op = dg2d.Op2D(0, 1, 0, 1, 3, 2, 3, dg2d.Advection2D(1.0, 0.5, 0.01))
    n = op.n
    rng = np.random.default_rng(0)
    C = 0.01 + 0.02 * rng.random((2, 3, 4, 4))
    L = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1
        L[:, j] = op.apply_diffusion(C, e)
    m = np.tile(op.m2.reshape(1, 1, 4, 4), (2, 3, 1, 1)).reshape(-1)
    MA = m[:, None] * (np.eye(n) - 0.05 * L)
    assert np.abs(MA - MA.T).max() < 1e-15
    assert np.abs(np.diag(MA) - (m + 0.05 * op.stiffness_diag(C))).max() < 1e-15
    rhs = rng.standard_normal(n)
    assert rel(op.implicit_solve(C, 0.05, rhs), np.linalg.solve(np.eye(n) - 0.05 * L, rhs)) < 1e-12


def test_euler_conservation_and_free_stream():
    op = dg2d.Op2D(0, 10, 0, 10, 4, 4, 7, dg2d.Euler2D())
    X, Y = op.nodes()
    rho = 1 + 0.1 * np.sin(2 * np.pi * X / 10) * np.cos(2 * np.pi * Y / 10)
    u = np.stack([rho, rho * 1.0, rho * 0.5, 2.5 + 0.5 * rho]).reshape(-1)
    cv = op.apply_convection(u).reshape(4, 4, 4, 8, 8)
    for c in range(4):
        assert abs(float((cv[c] * op.m2).sum())) < 1e-12
    const = np.stack([np.full(X.shape, 1.2), np.full(X.shape, 0.6), np.full(X.shape, -0.3),
                      np.full(X.shape, 3.0)]).reshape(-1)
    assert np.abs(op.apply_convection(const)).max() < 1e-12


def _lift3(u1, ne, p1, ney):
    """1-D (rho, rho u, E) on (ne, p1) -> y-invariant 2-D (rho, rho u, 0, E)."""
    u3 = u1.reshape(3, ne, p1)
    z = np.zeros_like(u3[0])
    u4 = np.stack([u3[0], u3[1], z, u3[2]])
    return np.broadcast_to(u4[:, None, :, None, :], (4, ney, ne, p1, p1)).reshape(-1)


def _check_reduces(v2, ref1, ne, p1, ney, tol):
    v = v2.reshape(4, ney, ne, p1, p1)
    r3 = ref1.reshape(3, ne, p1)
    for j in range(ney):
        for k in range(p1):
            for c2, c1 in ((0, 0), (1, 1), (3, 2)):
                a, b = v[c2, j, :, k, :], r3[c1]
                assert np.abs(a - b).max() <= tol * max(1e-300, np.abs(b).max()), (c2, j, k)
            assert np.abs(v[2, j, :, k, :]).max() <= tol * np.abs(r3[1]).max() + 1e-300


def test_ns2d_y_invariant_reduces_to_reference_cns(golden):
    """NS2D / Euler2D on y-invariant data with v = 0 reproduce the reference's
    1-D CompressibleFlow (problems.py:160-240): convection (Rusanov with
    lambda = |v| + c), the physical viscous operator (matrix SIP with A_d,
    dgsem.py:251-309) and eval_rhs, per field (rho v stays ~0)."""
    G = golden["operators"]          # CompressibleFlow(eta=1e-3), 8 elements, P = 5 on [0, 1]
    ne, P, ney = 8, 5, 2
    p1 = P + 1
    op = dg2d.Op2D(0.0, 1.0, 0.0, 0.7, ne, ney, P, dg2d.NS2D(1.4, 1e-3, 0.75))
    u2 = _lift3(G["cns_u"], ne, p1, ney)
    _check_reduces(op.apply_convection(u2), G["cns_conv"], ne, p1, ney, 1e-13)
    _check_reduces(op.apply_viscous(u2), G["cns_diff"], ne, p1, ney, 1e-13)
    _check_reduces(op.eval_rhs(u2), G["cns_rhs"], ne, p1, ney, 1e-13)
    # the reference's acoustic wave (eta = 1e-5, Pr 0.75, 12 elements, P = 7): p ~ 1e3 against
    # O(1e2) outputs, so the flux differences cancel ~10 digits (measured 7e-12 on rho u)
    C = golden["cns"]
    ne, P = 12, 7
    p1 = P + 1
    op = dg2d.Op2D(0.0, 1.0, 0.0, 0.3, ne, ney, P, dg2d.NS2D(1.4, 1e-5, 0.75))
    u2 = _lift3(C["op_u"], ne, p1, ney)
    _check_reduces(op.apply_convection(u2), C["op_conv"], ne, p1, ney, 2e-11)
    _check_reduces(op.eval_rhs(u2), C["op_rhs"], ne, p1, ney, 2e-11)


def test_ns2d_viscous_consistency():
    """The NS viscous operator: zero on constant states, conserves mass and
    momentum on a periodic mesh, and decays kinetic energy of a shear wave at
    the Stokes rate nu k^2 (resolved mesh)."""
    op = dg2d.Op2D(0.0, 2 * np.pi, 0.0, 2 * np.pi, 4, 4, 7, dg2d.NS2D(1.4, 1e-2, 0.72))
    X, Y = op.nodes()
    const = np.stack([np.full(X.shape, 1.1), np.full(X.shape, 0.3), np.full(X.shape, -0.2),
                      np.full(X.shape, 2.5)]).reshape(-1)
    assert np.abs(op.apply_viscous(const)).max() < 1e-12
    rho = 1.0 + 0.1 * np.sin(X + 2 * Y)
    u = np.stack([rho, rho * np.sin(Y), rho * 0.2 * np.cos(X), 2.5 + 0.1 * np.cos(X - Y)])
    fv = op.apply_viscous(u.reshape(-1)).reshape(4, 4, 4, 8, 8)
    for c in range(3):
        assert abs(float((fv[c] * op.m2).sum())) < 1e-12
    # shear wave rho = 1, u = sin y: d(rho u)/dt = nu u_yy = -nu sin y
    sw = np.stack([np.ones(X.shape), np.sin(Y), np.zeros(X.shape), np.full(X.shape, 2.5)])
    fv = op.apply_viscous(sw.reshape(-1)).reshape(4, 4, 4, 8, 8)
    assert np.abs(fv[1] + 1e-2 * np.sin(Y)).max() < 1e-6


def test_persson_2d_reduces_to_pinned_1d_sensor():
    """The tensor-product modal sensor on y-invariant data is the 1-D sensor of oracle/dg1d.py
    (itself pinned to the reference's AV goldens, test_oracle_golden.py): only the l = 0 modes
    survive, their (2 / (2l+1)) = 2 factor cancels in the energy ratio, h = max(dx, dy) = dx."""
    from oracle import dg1d
    ne, P, ney = 24, 6, 3
    av = (1.0, 0.7)
    o1 = dg1d.Op1D(0.0, 2.0, ne, P, dg1d.Burgers(1e-3), av=av)
    x = (o1.xl + o1.dx * np.arange(ne))[:, None] + 0.5 * o1.dx * (o1.xi + 1.0)[None, :]
    u1 = 0.3 + np.tanh((x - 1.03) / 0.02) + 0.2 * np.tanh((x - 0.41) / 0.01)   # under-resolved fronts: the ramp is active
    nu1 = o1.persson_viscosity(u1.reshape(-1))
    assert nu1.max() > 0 and (nu1 == 0).any()
    o2 = dg2d.Op2D(0.0, 2.0, 0.0, 0.1, ne, ney, P, dg2d.Burgers2D(1e-3), av=av)
    u2 = np.broadcast_to(u1.reshape(1, 1, ne, 1, P + 1), (1, ney, ne, P + 1, P + 1)).reshape(-1)
    nu2 = o2.persson_viscosity(u2)
    assert nu2.shape == (ney, ne)
    for j in range(ney):
        assert np.abs(nu2[j] - nu1).max() <= 1e-13 * nu1.max()
    # frozen per slab, entering the rhs and the SI coefficient as nu + nu_art (dgsem.py:356-396, 563-571)
    o2.begin_slab(u2, 0.0, 1e-3)
    o1.begin_slab(u1.reshape(-1), 0.0, 1e-3)
    r2 = o2.eval_rhs(u2).reshape(1, ney, ne, P + 1, P + 1)
    r1 = o1.eval_rhs(u1.reshape(-1))
    assert rel(r2[0, 1, :, 2, :].reshape(-1), r1) < 1e-12
    c2 = np.asarray(o2.modified_coeff(u2, 2e-3)).reshape(ney, ne, P + 1, P + 1)
    c1 = np.asarray(o1.modified_coeff(u1.reshape(-1), 2e-3)).reshape(ne, P + 1)
    assert rel(c2[1, :, 3, :], c1) < 1e-14
