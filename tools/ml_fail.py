"""Debug: one march of a paper-table case; print the failure (debug aid)."""
import json
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from tools.paper_table import make_study  # noqa: E402
from paper_2504_18526_b200.runtime import get_runtime  # noqa: E402

rt = get_runtime()
rt.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
G = np.load("tests/golden/multilevel_study.npz")
cfg = json.loads(str(G["config"]))
case, cfl = sys.argv[1], float(sys.argv[2])
lv, start, c_fmg = cfg["cases"][case]
st = make_study(case, cfg["levels"][lv], start, c_fmg)
for k in range(int(sys.argv[3]) + 1):
    n0 = rt.status()[2]
    try:
        u = st.march(cfl, k)
        print(k, "err", st.error(u), flush=True)
    except Exception as e:
        traceback.print_exc()
        its, mg = rt.cg_log()
        its = its[n0:]
        print(k, "FAILED", repr(e), "solves", len(its), "max it", its.max() if len(its) else None,
              "neg", int((its < 0).sum()), "status", rt.status(), flush=True)
