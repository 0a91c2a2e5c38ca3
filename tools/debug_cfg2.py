"""Debug: cfg2 pieces on the GPU vs the oracle, cluster CG in isolation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import dg1d, sweeper as osw, workloads
from paper_2504_18526_b200 import dgsem, problems, sdc, mlsdc, collocation
from paper_2504_18526_b200.configs import CFG2 as w
from paper_2504_18526_b200.runtime import get_runtime
rt = get_runtime()
rng = np.random.default_rng(0)
for ne in (64, 512):
    op = dgsem.DGOperator(dgsem.Mesh1D(w.x_left, w.x_right, ne, 8), problems.Burgers(5e-3))
    orc = dg1d.Op1D(w.x_left, w.x_right, ne, 8, dg1d.Burgers(5e-3))
    rhs = 1 + 0.1 * np.sin(np.arange(op.ndof) * 0.05)
    fld = 0.01 + 0.01 * rng.random((ne, 9))
    xo = orc.implicit_solve(fld, 0.01, rhs)
    for K in (1, 2, 4, 8, 16):
        if ne * 9 / K > 3000: continue
        rt.set_cg(1e-14, 1000, K)
        try:
            x = op.implicit_solve(fld, 0.01, rhs).cpu().numpy()
            print(ne, K, 'err', np.abs(x - xo).max(), 'its', rt.cg_log()[0][-1], orc.cg_log[-1][0], flush=True)
        except Exception as e:
            print(ne, K, 'EXC', e, flush=True)
            rt.reset_status()
rt.set_cg(1e-14, 1000, 0)
