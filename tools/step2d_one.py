"""Replay one SI-MLSDC step of a 2-D BASELINE workload (launch-list target).

usage: python tools/step2d_one.py [cfg3|cfg4|cfg5] [warm]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_18526_b200 import dgsem, dgsem2d, mlsdc
from paper_2504_18526_b200.configs import WORKLOADS
from paper_2504_18526_b200.runtime import get_runtime

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rt = get_runtime()
rt.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)


def make_op(P):
    mesh = dgsem2d.Mesh2D(0.0, w.length, 0.0, w.length, w.nex, w.ney, P)
    return dgsem2d.DGOperator2D(mesh, w.gpu_problem())


hier = mlsdc.build_p_hierarchy(make_op, [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
X, Y = hier.fine.ctx.mesh.nodes_xy
u0 = w.initial_state(X, Y)
dt = w.time_step(u0, dgsem.compute_delta(w.p_fine))
g = mlsdc.SlabGraph(hier, u0, 0.0, dt, w.n_cycles, "fmg")
for _ in range(warm):
    g.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.step()
e1.record()
torch.cuda.synchronize()
print(f"{w.name}: one step {e0.elapsed_time(e1):.1f} ms, kernels/step {g.kernels_per_step}")
