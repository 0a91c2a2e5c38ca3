"""GPU-vs-oracle bisection of the 1-D CNS path (diagnostics, needs a GPU)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dg1d, quad, sweeper  # noqa: E402
from paper_2504_18526_b200 import collocation, dgsem, mlsdc, problems, sdc  # noqa: E402
from paper_2504_18526_b200.configs import CNS_CASES  # noqa: E402
from paper_2504_18526_b200.runtime import get_runtime  # noqa: E402

G = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cns.npz"))
rt = get_runtime()
rt.set_cg(1e-14, 1000, 0)


def h(a):
    return a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)


def fr(a, b):
    a, b = h(a).reshape(3, -1), h(b).reshape(3, -1)
    return max(np.linalg.norm(a[c] - b[c]) / np.linalg.norm(b[c]) for c in range(3))


case = sys.argv[1] if len(sys.argv) > 1 else "cns_mlsdc"
w = {c.name: c for c in CNS_CASES}[case]
u0f, dt = G[f"{case}_u0"], float(G[f"{case}_dt"])
prob_o = dg1d.CNS1D(gamma=w.gamma, R_gas=w.R_gas, eta=w.eta, Pr=w.prandtl)
for P in (() if len(sys.argv) > 2 else (w.p_coarse, w.p_fine)):
    op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, w.n_elem, P), problems.CompressibleFlow(eta=w.eta))
    log = []
    oo = dg1d.Op1D(0.0, 1.0, w.n_elem, P, prob_o, cg_log=log)
    xf = quad.gll(w.p_fine + 1)[0]
    xc = quad.gll(P + 1)[0]
    u = np.einsum("ij,cej->cei", quad.lagrange(xf, xc), u0f.reshape(3, w.n_elem, -1)).reshape(-1)
    print(f"P={P} conv", fr(op.apply_convection(u), oo.apply_convection(u)),
          "rhs", fr(op.eval_rhs(u), oo.eval_rhs(u)))
    for a in (0.05 * dt, 0.3 * dt):
        c = op.modified_diffusion_matrix(u, a, "si2")
        co = oo.modified_coeff(u, a)
        print(f"  a={a:.3e} coef", np.abs(h(op.coefficient_field(c)) - co).max() / np.abs(co).max(),
              "diff", fr(op.apply_diffusion(c, u), oo.apply_diffusion(co, u)))
        n0 = rt.status()[2]
        x = op.implicit_solve(c, a, u)
        xo = oo.implicit_solve(co, a, u)
        print("    solve", fr(x, xo), "iters gpu", rt.cg_log()[0][n0:].tolist(), "oracle", log[-1][0])
    # node caches + single-level sweep vs oracle
    rule = collocation.make_nodes("radau_right", 3)
    s = sdc.run_sdc(op, rule, collocation.make_weights(rule), dt, "si2", u, 0.0, 1)
    so = sweeper.run_sdc(oo, sweeper.Rule("radau_right", 3), dt, "si2", u, 0.0, 1)
    print("  sdc1 u", fr(s.u[-1], so.u[-1]), "f", fr(s.f[-1], so.f[-1]), "h1", fr(s.h1[-1], so.h1[-1]))
# MLSDC step
log = []
hg = mlsdc.build_p_hierarchy(lambda P: dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, w.n_elem, P),
                                                         problems.CompressibleFlow(eta=w.eta)),
                             [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
ho = sweeper.build_two_level(lambda lvl: dg1d.Op1D(0.0, 1.0, w.n_elem, w.p_coarse if lvl == "coarse" else w.p_fine,
                                                   prob_o, cg_log=log),
                             sweeper.Rule("radau_right", w.m_coarse), sweeper.Rule("radau_right", w.m_fine))
for nc in (() if len(sys.argv) > 2 else (0, 1, 2)):
    n0 = rt.status()[2]
    log.clear()
    ug = mlsdc.run_mlsdc(hg, u0f, 0.0, dt, nc, strategy="fmg").u[-1]
    uo = sweeper.run_mlsdc(ho, u0f, 0.0, dt, nc).u[-1]
    print("mlsdc cycles", nc, fr(ug, uo), rt.cg_log()[0][n0:].tolist()[:30], [it for it, _ in log][:30])
# single-level SDC of the case, solve by solve
op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, w.n_elem, w.p_fine), problems.CompressibleFlow(eta=w.eta))
rule = collocation.make_nodes("radau_right", w.m_fine)
log = []
oo = dg1d.Op1D(0.0, 1.0, w.n_elem, w.p_fine, prob_o, cg_log=log)
for ns in range(0, w.n_sweeps + 1):
    n0 = rt.status()[2]
    log.clear()
    s = sdc.run_sdc(op, rule, collocation.make_weights(rule), dt, w.scheme, u0f, 0.0, ns)
    so = sweeper.run_sdc(oo, sweeper.Rule("radau_right", w.m_fine), dt, w.scheme, u0f, 0.0, ns)
    it, mg = rt.cg_log()
    it, mg = it[n0:], mg[n0:]
    print("sdc sweeps", ns, fr(s.u[-1], so.u[-1]), it.tolist(), [i for i, _ in log], np.round(mg, 2).tolist())
