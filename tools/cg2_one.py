"""Time one 2-D implicit solve (k2_cg) on a BASELINE 2-D level; ncu target.

usage: python tools/cg2_one.py [cfg3|cfg4|cfg5] [P] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_18526_b200 import dgsem, dgsem2d
from paper_2504_18526_b200.configs import WORKLOADS
from paper_2504_18526_b200.runtime import get_runtime

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
w = WORKLOADS[name]
P = int(sys.argv[2]) if len(sys.argv) > 2 else w.p_fine
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rt = get_runtime()
rt.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
npart = int(os.environ.get("SISDC_PART", "0"))   # > 0: split CG of an R-partition operator
op = dgsem2d.DGOperator2D(dgsem2d.Mesh2D(0.0, w.length, 0.0, w.length, w.nex, w.ney, P),
                          w.gpu_problem(),
                          partition=dgsem2d.Partition(npart) if npart > 0 else None)
X, Y = op.mesh.nodes_xy
u = op.scatter(w.initial_state(X, Y))
dt = w.time_step(w.initial_state(X, Y), dgsem.compute_delta(w.p_fine))
a = 0.5 * dt
c = op.modified_diffusion_matrix(u, a, "si2")
out = torch.empty_like(u)
op.eager_checks = False
ts = []
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    op.implicit_solve(c, a, u, out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
its = rt.cg_log()[0][-reps:].tolist()
n = u.numel()
print(f"{name} P={P} n={n} iterations={its} us/solve={[round(t) for t in ts]} "
      f"us/iter={ts[-1] / max(its[-1], 1):.1f} ideal_us/iter(94B/DOF)={94 * n / 6553.6e3:.1f}")
if os.environ.get("SISDC_CG_TIMING") == "1":
    import ctypes as C
    import numpy as np
    buf = (C.c_longlong * 80)()
    rt.check(rt.lib.sisdc_ctx_debug_timing(rt.h, buf, 80))
    t = np.array(buf[:20], dtype=np.float64)
    for b, o in (("block 0", 0), ("block G-1", 10)):
        d = np.diff(t[o:o + 7]) / 1e3
        print(f"  {b} iteration 2 (us): phaseA {d[0]:.1f} sync {d[1]:.1f} phaseB {d[2]:.1f} part {d[3]:.1f} "
              f"sync {d[4]:.1f} total {d[5]:.1f}")
    for b, o in (("block 0", 30), ("block G-1", 40)):
        d = np.diff(np.array(buf[o:o + 5], dtype=np.float64)) / 1e3
        print(f"  {b} setup (us): coef/dinv tiles {d[0]:.1f}, x/p/s init + sync {d[1]:.1f}, "
              f"r0 = b - A x0 + u0 + sync {d[2]:.1f}, w0 = A u0 + reduction {d[3]:.1f}")
    t2 = np.array(buf[20:23], dtype=np.float64)
    if t2[2] > 0:
        print(f"  block0/warp0 phase B per element: wait {t2[0]/t2[2]:.0f} cycles, compute {t2[1]/t2[2]:.0f} cycles "
              f"({int(t2[2])} elements over all solves)")
