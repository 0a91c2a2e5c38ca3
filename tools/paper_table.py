"""Reproduce the paper's Burgers moving-front iteration table
(tab:burgers_iterations_cfl_hires) with the GPU study
runner: the reference CLI's cfl-sweep (cli.py:1110-1194) for each row's
hierarchy at CFL 0.5 ... 64, next to the reference CLI's own output
(tests/golden/multilevel_study*.npz, CFL 8-64) and the paper's values.

usage: python tools/paper_table.py [out.md]      (GPU; ~10 min)
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2504_18526_b200 import collocation, dgsem, mlsdc, problems, study  # noqa: E402
from paper_2504_18526_b200.runtime import get_runtime  # noqa: E402

CFL = [0.5, 1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0]
PAPER = {   # PAPER.md:1262-1267, fine-grid iterations until convergence
    "sdc": [3, 4, 4, 5, 6, 7, 11, 14],
    "i3_fmg1": [2, 2, 2, 2, 2, 4, 6, 9],
    "h3_fmg2": [2, 2, 2, 2, 2, 3, 6, 9],
    "h3_fmg1": [2, 2, 2, 2, 2, 4, 6, 9],
    "h3_cascade": [2, 2, 2, 2, 3, 5, 7, 10],
    "p3_fmg1": [3, 4, 4, 4, 4, 9, 9, 10],
}
LABEL = {
    "sdc": "SDC-SI(2,2)_7, 200 el, P 15",
    "i3_fmg1": "MLSDC_{3,5,7}, {200,200,200}, P {15,15,15}, FMG1",
    "h3_fmg2": "MLSDC_{3,5,7}, {50,100,200}, P 15, FMG2",
    "h3_fmg1": "MLSDC_{3,5,7}, {50,100,200}, P 15, FMG1",
    "h3_cascade": "MLSDC_{3,5,7}, {50,100,200}, P 15, cascade",
    "p3_fmg1": "MLSDC_{3,5,7}, {200,200,200}, P {5,10,15}, FMG1",
}
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def make_study(case, levels, start, c_fmg, nu=0.01, t_end=0.1):
    prob, exact = problems.burgers_front_problem(nu)
    if len(levels) == 1:
        ne, P, M = levels[0]
        op = dgsem.DGOperator(dgsem.Mesh1D(-1.0, 1.0, ne, P, bc="dirichlet"), prob)
        rule = collocation.make_nodes("radau_right", M)
        u0 = op.nodal_field(lambda x: exact(x, 0.0)[None])
        ur = op.nodal_field(lambda x: exact(x, t_end)[None])
        return study.SDCStudy(op, rule, collocation.make_weights(rule), "si2", u0, ur, t_end,
                              dgsem.max_wave_speed(op, u0))
    h = mlsdc.build_hierarchy(lambda ne, P: dgsem.DGOperator(dgsem.Mesh1D(-1.0, 1.0, ne, P, bc="dirichlet"), prob),
                              [tuple(x) for x in levels])
    op = h.fine.ctx
    u0 = op.nodal_field(lambda x: exact(x, 0.0)[None])
    ur = op.nodal_field(lambda x: exact(x, t_end)[None])
    return study.MLSDCStudy(h, u0, ur, t_end, dgsem.max_wave_speed(op, u0), strategy=start, c_fmg=c_fmg)


def ref_rows(name, case):
    p = os.path.join(HERE, "tests", "golden", name)
    if not os.path.exists(p):
        return {}
    G = np.load(p)
    out = {}
    for ln in str(G[f"{case}_iterations_csv"]).strip().split("\n")[1:]:
        c = ln.split(",")
        out[float(c[0])] = (c[2], c[4])
    return out


def fmt(stall, status, single):
    if status != "ok":
        return "fail"
    if stall in ("", None):
        return "-"
    return str(int(stall) + (0 if single else 1))


def main():
    out_md = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "gpurun_out", "paper_table.md")
    rt = get_runtime()
    rt.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
    G = np.load(os.path.join(HERE, "tests", "golden", "multilevel_study.npz"))
    cfg = json.loads(str(G["config"]))
    lines = ["| row | source | " + " | ".join(f"CFL {c:g}" for c in CFL) + " |",
             "|---|---|" + "---|" * len(CFL)]
    raw = {}
    for case, (lv, start, c_fmg) in cfg["cases"].items():
        levels = cfg["levels"][lv]
        single = len(levels) == 1
        st = make_study(case, levels, start, c_fmg)
        t0 = time.time()
        with tempfile.TemporaryDirectory() as d:
            pts = study.cfl_sweep(st, CFL, cfg["max_iterations"], out_dir=d)
            raw[case] = {"iterations_csv": open(os.path.join(d, "iterations.csv")).read(),
                         "errors_csv": open(os.path.join(d, "errors.csv")).read()}
        gpu = [fmt("" if p.stall is None else p.stall, p.status, single) for p in pts]
        lu = ref_rows("multilevel_study.npz", case)
        pcg = ref_rows("multilevel_study_pcg.npz", case)
        lines.append(f"| {LABEL[case]} | paper (HiSPEET) | " + " | ".join(map(str, PAPER[case])) + " |")
        lines.append(f"| | this repo (GPU, pinned PCG) | " + " | ".join(gpu) + " |")
        if pcg:
            lines.append(f"| | reference CLI, pinned PCG | " +
                         " | ".join(fmt(*pcg[c], single) if c in pcg else "" for c in CFL) + " |")
        lines.append(f"| | reference CLI, SuperLU | " +
                     " | ".join(fmt(*lu[c], single) if c in lu else "" for c in CFL) + " |")
        print(case, gpu, f"{time.time() - t0:.0f} s", flush=True)
    os.makedirs(os.path.dirname(out_md), exist_ok=True)
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(out_md.replace(".md", ".json"), "w") as f:
        json.dump(raw, f)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
