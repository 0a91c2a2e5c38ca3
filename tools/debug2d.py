import sys, os, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2504_18526_b200 import dgsem, dgsem2d, mlsdc
from paper_2504_18526_b200.configs import CFG3, CFG4
from paper_2504_18526_b200.runtime import get_runtime
rt = get_runtime()
for base in (CFG3, CFG4):
    for ne in (4, 8, 16, 32, 128):
        w = dataclasses.replace(base, nex=ne, ney=ne)
        mk = lambda P: dgsem2d.DGOperator2D(dgsem2d.Mesh2D(0, w.length, 0, w.length, ne, ne, P), dgsem2d.CompressibleEuler2D(w.gamma, w.nu))
        h = mlsdc.build_p_hierarchy(mk, [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
        X, Y = h.fine.ctx.mesh.nodes_xy
        u = w.initial_state(X, Y)
        dt = w.time_step(u, dgsem.compute_delta(w.p_fine))
        msg = []
        for s in range(4):
            rt.reset_status()
            sol = mlsdc.run_mlsdc(h, u, s * dt, dt, w.n_cycles, strategy="fmg")
            bad, fails, _ = rt.status()
            un = sol.u[-1].cpu().numpy()
            msg.append(f"s{s}: bad={bad} fails={fails} finite={np.isfinite(un).all()} rho[{un[:un.size//4].min():.3f},{un[:un.size//4].max():.3f}]")
            if bad >= 0 or not np.isfinite(un).all():
                break
            u = un
        its = rt.cg_log()[0]
        print(base.name[:5], ne, 'dt', f'{dt:.3e}', ' | '.join(msg), 'cg max it', its[-50:].max() if len(its) else None, flush=True)
