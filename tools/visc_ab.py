"""Time the NS2D viscous operator (and eval_rhs) on a BASELINE 2-D workload, and compare the
tensor-core kernel k2_visc8 with the line-formulated k2_visc (SISDC_VISC_LINE=1 in a child process).

usage: python tools/visc_ab.py [cfg4|cfg5] [reps]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2504_18526_b200 import dgsem2d
from paper_2504_18526_b200.configs import WORKLOADS
from paper_2504_18526_b200.runtime import get_runtime

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
child = os.environ.get("VISC_AB_CHILD")
w = WORKLOADS[name]
rt = get_runtime()
mesh = dgsem2d.Mesh2D(0.0, w.length, 0.0, w.length, w.nex, w.ney, w.p_fine)
op = dgsem2d.DGOperator2D(mesh, w.gpu_problem())
X, Y = mesh.nodes_xy
u = rt.to_device(w.initial_state(X, Y))
out = torch.empty_like(u)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


tv = timed(lambda: op.apply_viscous(u, out=out))
v = out.clone()
tr = timed(lambda: op.eval_rhs(u, out=out))
tag = "line (k2_visc)" if os.environ.get("SISDC_VISC_LINE") == "1" else "tensor-core (k2_visc8)"
print(f"{name} {tag}: apply_viscous {tv:.1f} us, eval_rhs {tr:.1f} us")
if child:
    np.save(child, v.cpu().numpy())
else:
    path = "/tmp/visc_ab_line.npy"
    env = dict(os.environ, SISDC_VISC_LINE="1", VISC_AB_CHILD=path)
    subprocess.run([sys.executable, os.path.abspath(__file__), name, str(reps)], env=env, check=True)
    ref = np.load(path)
    got = v.cpu().numpy()
    print(f"max |k2_visc8 - k2_visc| / max |k2_visc| = {np.abs(got - ref).max() / np.abs(ref).max():.3e}")
