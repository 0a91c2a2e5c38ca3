"""Small solves through every barrier-heavy kernel, as a compute-sanitizer target.

usage: compute-sanitizer --tool racecheck|synccheck|memcheck python tools/sanitize_small.py [1d|cns|2d|all]

1d : the cluster-resident PCG (st.async / mbarrier pushes) on 4 and 16 CTAs, and the grid mode
cns: the cluster BiCGStab of CompressibleFlow (DSMEM halo reads, cluster barriers)
2d : the fused single-pass 2-D PCG (TMA bulk staging on mbarriers, split column barrier)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2504_18526_b200 import dgsem, dgsem2d, problems
from paper_2504_18526_b200.runtime import get_runtime

what = sys.argv[1] if len(sys.argv) > 1 else "all"
rt = get_runtime()
rng = np.random.default_rng(0)
if what in ("1d", "all"):
    for ne, P, ctas in ((48, 8, 4), (96, 4, 16), (24, 8, 1), (720, 8, 0)):
        rt.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=ctas)
        op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 2.0 * np.pi, ne, P), problems.Burgers(5e-3))
        x = np.asarray(op.mesh.nodes_x).reshape(-1)
        u = 1.0 + 0.5 * np.sin(x)
        out = op.implicit_solve(op.modified_diffusion_matrix(u, 1e-3, "si2"), 5e-4, np.cos(x))
        print("1d", ne, P, ctas, "iterations", rt.cg_log()[0][-1], float(out.abs().max()))
    rt.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
if what in ("cns", "all"):
    ne, P = 24, 5
    op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, ne, P), problems.CompressibleFlow(1.4, 1e-3, 0.72))
    x = np.asarray(op.mesh.nodes_x)
    rho = 1.0 + 0.1 * np.sin(2 * np.pi * x)
    v = 0.3 * np.cos(2 * np.pi * x)
    p = 1.0 + 0.1 * np.sin(2 * np.pi * x)
    u = np.stack([rho, rho * v, p / 0.4 + 0.5 * rho * v * v]).reshape(-1)
    out = op.implicit_solve(op.modified_diffusion_matrix(u, 1e-3, "si2"), 5e-4, u)
    print("cns iterations", rt.cg_log()[0][-1], float(out.abs().max()))
if what in ("2d", "all"):
    from paper_2504_18526_b200.configs import CFG4
    for nex, ney in ((16, 12), (5, 3), (40, 17)):
        op = dgsem2d.DGOperator2D(dgsem2d.Mesh2D(0.0, CFG4.length, 0.0, CFG4.length, nex, ney, 7), CFG4.gpu_problem())
        X, Y = op.mesh.nodes_xy
        u = op.scatter(CFG4.initial_state(X, Y))
        out = op.implicit_solve(op.modified_diffusion_matrix(u, 1e-3, "si2"), 5e-4, u)
        print("2d", nex, ney, "iterations", rt.cg_log()[0][-1], float(out.abs().max()))
rt.raise_on_failure()
print("done")
