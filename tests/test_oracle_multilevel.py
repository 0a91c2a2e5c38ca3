"""The oracle's multilevel engine on three levels (oracle/sweeper.py
v_cycle / start / fas_rhs over an intermediate level) against the
reference's own 3-level goldens (tests/golden/multilevel.npz): the paper's
p-hierarchy {5,10,15} x M {3,5,7} on the Burgers moving front, FMG (c_fmg 1
and 2) and cascade starts, identical pinned-PCG iteration sequence."""
import json

import numpy as np
import pytest

from oracle import dg1d, sweeper
from paper_2504_18526_b200.configs import burgers_front_boundary


def oracle_hierarchy(levels, log):
    ctxs = [dg1d.Op1D(-1.0, 1.0, ne, P, dg1d.Burgers(0.01, boundary=burgers_front_boundary(0.01)),
                      bc="dirichlet", solver="pcg", rtol=1e-14, cg_log=log) for ne, P, _ in levels]
    rules = [sweeper.Rule("radau_right", M) for _, _, M in levels]
    lv = [sweeper.Lev(c, r) for c, r in zip(ctxs, rules)]
    tr = [sweeper.PTransfer(ctxs[i], ctxs[i + 1], rules[i], rules[i + 1]) for i in range(len(levels) - 1)]
    return sweeper.Hier(lv, tr, 2, 1, "incremental", True)


@pytest.mark.parametrize("case", ["p3_fmg1", "p3_fmg2", "p3_cascade"])
def test_oracle_three_level_step(golden_ml, case):
    G = golden_ml
    cfg = json.loads(str(G["config"]))[case]
    levels = json.loads(str(G["levels"]))[cfg[0]]
    log = []
    h = oracle_hierarchy(levels, log)
    sol = sweeper.run_mlsdc(h, G[f"{case}_u0"], 0.0, float(G[f"{case}_dt"]), 3, cfg[1], cfg[2])
    assert [it for it, _ in log] == G[f"{case}_pcg_iters1"].tolist()
    ref = G[f"{case}_pcg_u1"]
    assert np.linalg.norm(sol.u[-1] - ref) / np.linalg.norm(ref) < 1e-12
