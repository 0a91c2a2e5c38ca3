"""CPU tests of the ensemble study dispatch (SURVEY 8f.4,
paper_2504_18526_b200/study.py): the stall rule and CSV format restate the
reference's (checked against the reference CLI's own cfl-sweep output,
tests/golden/study.npz), and the round-robin dispatch over a 2-rank gloo
group gathers every point in order with no point run twice."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_18526_b200 import study


def test_converged_iteration_rule():
    assert study.converged_iteration([1.0, 0.5, 0.48]) == 2
    assert study.converged_iteration([1.0, 0.0, 0.0]) == 2
    assert study.converged_iteration([1.0, 2.0, 4.0]) is None
    with pytest.raises(ValueError):
        study.converged_iteration([1.0])


def test_csv_format_matches_reference(golden):
    G = golden["study"]
    text = str(G["iterations_csv"])
    lines = text.strip().split("\n")
    assert lines[0] == "cfl,n_steps,converged_iteration,error,status"
    rows = []
    for ln in lines[1:]:
        c, n, s, e, st = ln.split(",")
        rows.append((float(c), int(n), "" if s == "" else int(s), float(e), st))
    with tempfile.TemporaryDirectory() as d:
        study.write_csv(os.path.join(d, "it.csv"), ("cfl", "n_steps", "converged_iteration", "error", "status"), rows)
        assert open(os.path.join(d, "it.csv")).read() == text   # byte-identical round trip


class FakeStudy:
    """Deterministic error series per CFL (no GPU): e_k = cfl * 0.5^k + 0.01."""

    def steps(self, cfl):
        return 0.1 / max(1, int(4 / cfl)), max(1, int(4 / cfl))

    def march(self, cfl, k):
        if cfl > 7.0:
            raise study.SolverError("diverged")
        return cfl * 0.5 ** k + 0.01

    def error(self, u):
        return float(u)


def _worker(rank, world, port, out_dir, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []

    def sweep(st, c, m):
        calls.append(c)
        return study.sweep_one_cfl(st, c, m)
    pts = study.cfl_sweep(FakeStudy, [0.5, 1.0, 2.0, 4.0, 8.0], 6, out_dir=out_dir, sweep_fn=sweep)
    q.put((rank, calls, [(p.cfl, p.n_steps, p.errors, p.stall, p.status, p.rank) for p in pts]))
    dist.barrier()
    dist.destroy_process_group()


def test_round_robin_dispatch_over_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        procs = [ctx.Process(target=_worker, args=(r, 2, port, d, q)) for r in range(2)]
        for p in procs:
            p.start()
        res = dict((r, (c, pts)) for r, c, pts in [q.get(timeout=60) for _ in range(2)])
        for p in procs:
            p.join(timeout=60)
        assert res[0][0] == [0.5, 2.0, 8.0] and res[1][0] == [1.0, 4.0]   # point i on rank i % 2
        assert res[0][1] == res[1][1]                                       # every rank gets the full list
        pts = res[0][1]
        assert [p[5] for p in pts] == [0, 1, 0, 1, 0]
        assert pts[-1][4] == "failed" and pts[-1][2] == []
        serial = [study.sweep_one_cfl(FakeStudy(), c, 6) for c in (0.5, 1.0, 2.0, 4.0, 8.0)]
        assert [(p[2], p[3], p[4]) for p in pts] == [(s.errors, s.stall, s.status) for s in serial]
        it = open(os.path.join(d, "iterations.csv")).read().strip().split("\n")
        assert it[0] == "cfl,n_steps,converged_iteration,error,status" and len(it) == 6
        assert it[-1] == "8,1,,nan,failed"


def test_observed_order_and_convergence_csv(golden):
    """observed_order restates analysis.py:291-297; the orders.csv the
    dispatch writes from the reference's own error table equals the
    reference CLI's orders.csv byte for byte."""
    G = golden["study"]
    import json
    cfg = json.loads(str(G["conv_config"]))
    rows = [ln.split(",") for ln in str(G["conv_errors_csv"]).strip().split("\n")[1:]]
    table = {(float(r[0]), tuple(cfg["convergence"]["element_counts"][int(r[1])])): (int(r[3]), float(r[4]))
             for r in rows}
    with tempfile.TemporaryDirectory() as d:
        study.convergence(lambda ne, c: table[(c, tuple(ne))], cfg["convergence"]["element_counts"],
                          cfg["convergence"]["cfl_values"], out_dir=d)
        assert open(os.path.join(d, "orders.csv")).read() == str(G["conv_orders_csv"])
        assert open(os.path.join(d, "errors.csv")).read() == str(G["conv_errors_csv"])
    assert study.observed_order(0.4, 0.1, 2.0) == 2.0
    with pytest.raises(ValueError):
        study.observed_order(0.0, 0.1)
