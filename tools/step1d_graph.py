"""Replay the cfg2 SI-MLSDC slab graph a few times (launch-gap measurement
target: ncu --cache-control none sums the per-kernel durations of one replay,
compared with the CUDA-event time of a replay).

usage: python tools/step1d_graph.py [replays]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_18526_b200 import dgsem, mlsdc, problems
from paper_2504_18526_b200.configs import CFG2 as w
from paper_2504_18526_b200.runtime import get_runtime

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rt = get_runtime()
rt.set_cg(rtol=1e-14, maxit=1000)
mk = lambda P: dgsem.DGOperator(dgsem.Mesh1D(w.x_left, w.x_right, w.n_elem, P), problems.Burgers(w.params["nu"]))
hier = mlsdc.build_p_hierarchy(mk, [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
u0 = w.initial_state(dgsem.Mesh1D(w.x_left, w.x_right, w.n_elem, w.p_fine).ref_nodes)
dt, _ = w.time_step(u0, dgsem.compute_delta(w.p_fine))
g = mlsdc.SlabGraph(hier, u0, 0.0, dt, w.n_cycles, "fmg")
for _ in range(3):
    g.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    g.step()
e1.record()
torch.cuda.synchronize()
print(f"kernels per slab {g.kernels_per_step}, {e0.elapsed_time(e1) / reps * 1e3:.1f} us per replay")
