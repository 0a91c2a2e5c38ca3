"""Run one implicit solve per configuration in a fresh process (fault isolation)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2504_18526_b200 import dgsem, problems
from paper_2504_18526_b200.runtime import get_runtime
ne, P, K, zero = %d, %d, %d, %d
rt = get_runtime(); rt.set_cg(1e-14, 1000, K)
op = dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, ne, P), problems.ConvectionDiffusion(1.0, 0.01))
rhs = np.zeros(op.ndof) if zero else np.random.default_rng(0).standard_normal(op.ndof)
x = op.implicit_solve(0.02, 0.05, rhs)
print("ok", ne, P, K, zero, float(x.abs().max()), rt.cg_log()[0][-1:] )
'''
for ne, P, K, zero in [(8, 4, 0, 1), (8, 4, 0, 0), (8, 8, 0, 0), (64, 4, 0, 0), (8, 3, 0, 0), (4, 3, 0, 0), (64, 8, 0, 0), (64, 8, 2, 0), (40, 8, 0, 0)]:
    r = subprocess.run([sys.executable, "-c", CODE % (ROOT, ne, P, K, zero)], capture_output=True, text=True, timeout=120)
    out = (r.stdout + r.stderr).strip().splitlines()
    print(ne, P, K, zero, "->", out[-1] if out else r.returncode, flush=True)
