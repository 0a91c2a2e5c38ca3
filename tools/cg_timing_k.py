"""Cluster size sweep of the cfg2 coarse (P=4) and fine (P=8) CG (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2504_18526_b200 import dgsem, problems
from paper_2504_18526_b200.configs import CFG2 as w
from paper_2504_18526_b200.runtime import get_runtime
rt = get_runtime()
for P, Ks in ((4, (0, 7, 8, 10, 12, 16)), (8, (0, 12, 14, 16))):
    for K in Ks:
        rt.set_cg(1e-14, 1000, K)
        op = dgsem.DGOperator(dgsem.Mesh1D(w.x_left, w.x_right, 512, P), problems.Burgers(5e-3))
        op.eager_checks = False
        x = np.sin(np.arange(op.ndof) * 0.01) + 1.0
        coef = dgsem.SICoefficient(op.rt.to_device(x), 1.2e-4)
        xd = op.rt.to_device(x)
        out = torch.empty_like(xd)
        for rep in range(3):
            op.implicit_solve(coef, 1.2e-4, xd, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for rep in range(50):
            op.implicit_solve(coef, 1.2e-4, xd, out=out)
        e1.record()
        torch.cuda.synchronize()
        its = rt.cg_log()[0][-1]
        print(f"P={P} K={K} iters={its} per solve {e0.elapsed_time(e1) * 1e3 / 50:.2f} us")
