"""Setup vs iteration time of the cfg2 fine (P=8) and coarse (P=4) cluster CG
solves, plus the graph-level time per solve (diagnostics)."""
import os, sys, ctypes as C
os.environ["SISDC_CG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2504_18526_b200 import dgsem, problems
from paper_2504_18526_b200.configs import CFG2 as w
from paper_2504_18526_b200.runtime import get_runtime
rt = get_runtime()
rt.set_cg(1e-14, 1000, 0)
ghz = 1.965
for P in (8, 4):
    op = dgsem.DGOperator(dgsem.Mesh1D(w.x_left, w.x_right, 512, P), problems.Burgers(5e-3))
    op.eager_checks = False
    x = np.sin(np.arange(op.ndof) * 0.01) + 1.0
    coef = dgsem.SICoefficient(op.rt.to_device(x), 1.2e-4)
    xd = op.rt.to_device(x)
    out = torch.empty_like(xd)
    for rep in range(3):
        op.implicit_solve(coef, 1.2e-4, xd, out=out)
    torch.cuda.synchronize()
    buf = (C.c_longlong * 80)()
    rt.check(rt.lib.sisdc_ctx_debug_timing(rt.h, buf, 80))
    t = np.array(buf[:], dtype=np.float64)
    k = int(t[65])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for rep in range(20):
        op.implicit_solve(coef, 1.2e-4, xd, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"P={P} iters={k}: tables->x0 halo + r0 {(t[1]-t[0])/ghz/1e3:.2f} us, w0 matvec {(t[2]-t[1])/ghz/1e3:.2f} us, "
          f"setup reduction {(t[3]-t[2])/ghz/1e3:.2f} us, per-iteration {(t[4+k]-t[5])/(k-1)/ghz/1e3 if k>1 else 0:.2f} us, "
          f"kernel (CTA0 clock) {(t[64]-t[0])/ghz/1e3:.2f} us, back-to-back per solve {e0.elapsed_time(e1)*1e3/20:.2f} us")
