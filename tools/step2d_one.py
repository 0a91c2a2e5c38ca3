"""Replay one SI-MLSDC step of a 2-D BASELINE workload (launch-list target).

usage: python tools/step2d_one.py [cfg3|cfg4|cfg5] [warm]
env: SISDC_PART=n (n in-process partitions), SISDC_PART_NCCL=1 (one NCCL rank), SISDC_EAGER=1 (eager
slabs instead of a replayed CUDA graph)
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


part = None
if os.environ.get("SISDC_PART_NCCL") == "1":
    part = dgsem2d.Partition(1, dgsem2d.NcclComm(0, 1))
elif int(os.environ.get("SISDC_PART", "0")) > 0:
    part = dgsem2d.Partition(int(os.environ["SISDC_PART"]))
eager = os.environ.get("SISDC_EAGER") == "1"


def make_op(P):
    mesh = dgsem2d.Mesh2D(0.0, w.length, 0.0, w.length, w.nex, w.ney, P)
    return dgsem2d.DGOperator2D(mesh, w.gpu_problem(), partition=part, eager_checks=not eager)


hier = mlsdc.build_p_hierarchy(make_op, [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
X, Y = hier.fine.ctx.mesh.nodes_xy
u0 = w.initial_state(X, Y)
dt = w.time_step(u0, dgsem.compute_delta(w.p_fine))
u0 = hier.fine.ctx.scatter(u0) if part is not None else u0
if eager:
    class _Eager:
        kernels_per_step = -1

        def __init__(self):
            self.u = rt.to_device(u0).clone()

        def step(self):
            n0 = rt.launch_count()
            sol = mlsdc.run_mlsdc(hier, self.u, 0.0, dt, w.n_cycles, strategy="fmg")
            rt.copy(self.u, sol.u[-1])
            self.kernels_per_step = rt.launch_count() - n0
    g = _Eager()
else:
    g = mlsdc.SlabGraph(hier, u0, 0.0, dt, w.n_cycles, "fmg")
for _ in range(warm):
    g.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.step()
e1.record()
torch.cuda.synchronize()
print(f"{w.name} part={os.environ.get('SISDC_PART_NCCL') and 'nccl1' or os.environ.get('SISDC_PART', 0)} eager={eager} overlap={os.environ.get('SISDC_PART_OVERLAP', 'auto')}: one step {e0.elapsed_time(e1):.1f} ms, kernels/step {g.kernels_per_step}")
