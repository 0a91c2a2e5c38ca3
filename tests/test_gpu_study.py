"""The reference CLI's own cfl-sweep study (cli.py:1110-1194, wave-packet
convection-diffusion, two p-levels, exact reference) run through the GPU
ensemble dispatch (paper_2504_18526_b200/study.py): the same n_steps, stall
iterations and status per CFL point, and the error series of
errors.csv / iterations.csv to 1e-9 relative (tests/golden/study.npz)."""
import json
import os
import tempfile

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def parse(text):
    lines = text.strip().split("\n")
    return lines[0], [ln.split(",") for ln in lines[1:]]


def test_cfl_sweep_matches_reference_cli(golden):
    from paper_2504_18526_b200 import dgsem, mlsdc, problems, study
    G = golden["study"]
    cfg = json.loads(str(G["config"]))
    pr, lv = cfg["problem"], cfg["levels"]
    prob = problems.ConvectionDiffusion(pr["speed"], pr["nu"])
    exact = problems.wave_packet_exact(pr["nu"], pr["speed"])
    h = mlsdc.build_p_hierarchy(lambda P: dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, lv[1]["n_elem"], P), prob),
                                [lv[0]["degree"], lv[1]["degree"]], [lv[0]["n_nodes"], lv[1]["n_nodes"]])
    op = h.fine.ctx
    u0 = op.nodal_field(lambda x: exact(x, 0.0)[None])
    u_ref = op.nodal_field(lambda x: exact(x, cfg["time"]["t_end"])[None])
    st = study.MLSDCStudy(h, u0, u_ref, cfg["time"]["t_end"], dgsem.max_wave_speed(op, u0))
    with tempfile.TemporaryDirectory() as d:
        pts = study.cfl_sweep(st, cfg["sweep"]["cfl_values"], cfg["sweep"]["max_iterations"], out_dir=d)
        it_text = open(os.path.join(d, "iterations.csv")).read()
        err_text = open(os.path.join(d, "errors.csv")).read()
    assert len(pts) == len(cfg["sweep"]["cfl_values"])
    for mine, ref in ((it_text, str(G["iterations_csv"])), (err_text, str(G["errors_csv"]))):
        h1, rows = parse(mine)
        h2, rrows = parse(ref)
        assert h1 == h2 and len(rows) == len(rrows)
        for a, b in zip(rows, rrows):
            assert a[:3] == b[:3]                     # cfl, n_steps, stall / iteration index
            if len(a) > 4:
                assert a[4] == b[4]                   # status
            assert abs(float(a[3]) - float(b[3])) <= 1e-9 * abs(float(b[3]))


def test_convergence_study_matches_reference_cli(golden):
    """The reference CLI's convergence study (cli.py:1194-1256): one GPU
    SI-MLSDC march per (cfl, element-count family) at fixed iterations;
    n_steps and the error table to 1e-9, observed orders to 1e-7."""
    import math
    from paper_2504_18526_b200 import dgsem, mlsdc, problems, study
    G = golden["study"]
    cfg = json.loads(str(G["conv_config"]))
    pr, lv = cfg["problem"], cfg["levels"]
    prob = problems.ConvectionDiffusion(pr["speed"], pr["nu"])
    exact = problems.wave_packet_exact(pr["nu"], pr["speed"])
    t_end = cfg["time"]["t_end"]

    def run_job(n_elems, cfl):
        h = mlsdc.build_p_hierarchy(lambda P: dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, n_elems[-1], P), prob),
                                    [lv[0]["degree"], lv[1]["degree"]], [lv[0]["n_nodes"], lv[1]["n_nodes"]])
        op = h.fine.ctx
        u0 = op.nodal_field(lambda x: exact(x, 0.0)[None])
        lam = dgsem.max_wave_speed(op, u0)
        dt0 = dgsem.dt_from_cfl(cfl, op.mesh.dx, lam, op.mesh.degree)
        n = max(1, math.ceil(t_end / dt0 - 1e-12))
        u = mlsdc.integrate_mlsdc(h, u0, 0.0, t_end / n, n, cfg["method"]["iterations"], strategy="fmg")
        ref = op.nodal_field(lambda x: exact(x, t_end)[None])
        return n, op.norm_l2(u - ref) / op.norm_l2(ref)
    with tempfile.TemporaryDirectory() as d:
        study.convergence(run_job, cfg["convergence"]["element_counts"], cfg["convergence"]["cfl_values"], out_dir=d)
        mine_e = open(os.path.join(d, "errors.csv")).read()
        mine_o = open(os.path.join(d, "orders.csv")).read()
    for mine, ref, tol in ((mine_e, str(G["conv_errors_csv"]), 1e-9), (mine_o, str(G["conv_orders_csv"]), 1e-7)):
        h1, rows = parse(mine)
        h2, rrows = parse(ref)
        assert h1 == h2 and len(rows) == len(rrows)
        for a, b in zip(rows, rrows):
            assert a[:-1] == b[:-1]
            assert abs(float(a[-1]) - float(b[-1])) <= tol * abs(float(b[-1]))


def test_failed_point_does_not_poison_later_points(golden):
    """A CFL point whose march fails (non-finite state -> SolverError latched
    on the device) must not turn later points on the same rank into failures:
    each march is independent, as in the reference CLI (cli.py:1110-1138)."""
    from paper_2504_18526_b200 import dgsem, mlsdc, problems, study
    G = golden["study"]
    cfg = json.loads(str(G["config"]))
    pr, lv = cfg["problem"], cfg["levels"]
    prob = problems.ConvectionDiffusion(pr["speed"], pr["nu"])
    exact = problems.wave_packet_exact(pr["nu"], pr["speed"])
    h = mlsdc.build_p_hierarchy(lambda P: dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, lv[1]["n_elem"], P), prob),
                                [lv[0]["degree"], lv[1]["degree"]], [lv[0]["n_nodes"], lv[1]["n_nodes"]])
    op = h.fine.ctx
    u0 = op.nodal_field(lambda x: exact(x, 0.0)[None])
    u_ref = op.nodal_field(lambda x: exact(x, cfg["time"]["t_end"])[None])
    cfl_bad, cfl_good = 1.0, float(cfg["sweep"]["cfl_values"][0])

    class Poisoned(study.MLSDCStudy):
        def march(self, cfl, k):
            if cfl == cfl_bad:
                good = self.u0
                self.u0 = good * float("nan")
                try:
                    return super().march(cfl, k)
                finally:
                    self.u0 = good
            return super().march(cfl, k)

    st = Poisoned(h, u0, u_ref, cfg["time"]["t_end"], dgsem.max_wave_speed(op, u0))
    pts = study.cfl_sweep(st, [cfl_bad, cfl_good], 3)
    assert pts[0].status == "failed"
    clean = study.cfl_sweep(study.MLSDCStudy(h, u0, u_ref, cfg["time"]["t_end"], dgsem.max_wave_speed(op, u0)),
                            [cfl_good], 3)[0]
    assert pts[1].status == clean.status != "failed"
    assert pts[1].errors == clean.errors
