"""Dump the GPU CG iteration sequence of the 3-level golden cases (debug aid)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_multilevel import front_hierarchy  # noqa: E402
from paper_2504_18526_b200 import mlsdc  # noqa: E402
from paper_2504_18526_b200.runtime import get_runtime  # noqa: E402

G = np.load("tests/golden/multilevel.npz")
rt = get_runtime()
rt.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
out = {}
for case in sys.argv[1:]:
    cfg = json.loads(str(G["config"]))[case]
    h, _ = front_hierarchy(json.loads(str(G["levels"]))[cfg[0]])
    n0 = rt.status()[2]
    sol = mlsdc.run_mlsdc(h, G[f"{case}_u0"], 0.0, float(G[f"{case}_dt"]), 3, strategy=cfg[1], c_fmg=cfg[2])
    its, margins = rt.cg_log()
    out[case] = {"its": its[n0:].tolist(), "margins": margins[n0:].tolist(), "ref": G[f"{case}_pcg_iters1"].tolist()}
json.dump(out, open("gpurun_out/ml_dump.json", "w"))
