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
