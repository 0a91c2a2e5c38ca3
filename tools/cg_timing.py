"""Per-iteration clock64 breakdown of one cluster CG solve (diagnostics)."""
import os, sys, ctypes as C
os.environ["SISDC_CG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2504_18526_b200 import dgsem, problems
from paper_2504_18526_b200.configs import CFG2 as w
from paper_2504_18526_b200.runtime import get_runtime
rt = get_runtime()
for ne, K in ((512, 0), (512, 8), (512, 16), (64, 1), (256, 0)):
    rt.set_cg(1e-14, 1000, K)
    op = dgsem.DGOperator(dgsem.Mesh1D(w.x_left, w.x_right, ne, 8), problems.Burgers(5e-3))
    x = np.sin(np.arange(op.ndof) * 0.01) + 1.0
    coef = dgsem.SICoefficient(op.rt.to_device(x), 2e-4)
    for rep in range(3):
        op.implicit_solve(coef, 2e-4, x)
    buf = (C.c_longlong * 80)()
    rt.check(rt.lib.sisdc_ctx_debug_timing(rt.h, buf, 80))
    t = np.array(buf[:], dtype=np.float64)
    k = int(t[65])
    ghz = 1.965
    print(f"ne={ne} K={K} iters={k}: setup tables->x0halo {(t[1]-t[0])/ghz/1e3:.2f} us, w0 matvec {(t[2]-t[1])/ghz/1e3:.2f} us, "
          f"setup reduction {(t[3]-t[2])/ghz/1e3:.2f} us, per-iteration {(t[4+k]-t[5])/(k-1)/ghz/1e3 if k>1 else 0:.2f} us "
          f"(first {(t[5]-t[3])/ghz/1e3:.2f}), total {(t[64]-t[0])/ghz/1e3:.2f} us")
    d = np.diff(t[70:75])
    print("   iteration 5 cycles: top->sync %d, sync %d, matvec %d, reduction %d, scalars %d" % tuple(np.concatenate([[t[70]-t[9]], d])))
