"""Ensemble dispatch of independent study points across GPUs.

The reference's CFL-sweep study (``cli.py:1110-1194``; the convergence study
``cli.py:1194-1256`` is dispatched the same way, ``convergence``) computes, for every
CFL value, the error-vs-iterations series of a march to t_end and the
iteration at which it stalls (``analysis.converged_iteration``,
``analysis.py:300-314``); its points are independent, and the reference runs
them serially or on host threads.  Here every point runs through the GPU
SI-MLSDC (or single-level SDC) path, the points are dealt round-robin over the
ranks of a ``torch.distributed`` process group (one process per GPU, no data
path collective: results are gathered once at the end), and rank 0 writes
``errors.csv`` / ``iterations.csv`` in the reference's exact format
(``cli.py:688-704,1160-1176``), so existing tooling reads them unchanged.

Only the sweep dispatch is built; config parsing, manifests and the other
studies stay with the reference's CLI (out of the sweep path).
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, List, Optional, Sequence

import numpy as np

from ._lib import SolverError

__all__ = ["converged_iteration", "observed_order", "write_csv", "SweepPoint", "MLSDCStudy", "SDCStudy",
           "sweep_one_cfl", "cfl_sweep", "convergence"]


def converged_iteration(error_series, threshold: float = 0.1) -> Optional[int]:
    """First index whose relative change from the previous entry falls below
    threshold; None when the series never settles (``analysis.py:300-314``)."""
    e = [float(x) for x in error_series]
    if len(e) < 2:
        raise ValueError("need at least two error entries")
    for k in range(1, len(e)):
        prev = e[k - 1]
        if prev == 0.0:
            change = 0.0 if e[k] == 0.0 else np.inf
        else:
            change = abs(e[k] - prev) / abs(prev)
        if change < threshold:
            return k
    return None


def _fmt(v) -> str:
    """``cli.py:688-695``: 17 significant digits for floats."""
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return format(float(v), ".17g")
    return str(v)


def write_csv(path, header, rows) -> str:
    """One deterministic CSV (``cli.py:698-704``); returns its sha256."""
    lines = [",".join(header)]
    for row in rows:
        lines.append(",".join(_fmt(v) for v in row))
    data = ("\n".join(lines) + "\n").encode()
    Path(path).write_bytes(data)
    return hashlib.sha256(data).hexdigest()


@dataclass
class SweepPoint:
    cfl: float
    n_steps: int
    errors: List[float] = field(default_factory=list)
    stall: Optional[int] = None
    status: str = "ok"
    rank: int = 0


def _steps(t_end: float, cfl: float, dx: float, lam: float, degree: int):
    from .dgsem import dt_from_cfl
    dt0 = dt_from_cfl(cfl, dx, lam, degree)
    n = max(1, math.ceil(t_end / dt0 - 1e-12))   # cli.py:1116-1117
    return t_end / n, n


class _Study:
    def __init__(self, op, u0, u_ref, t_end: float, lam: float):
        self.op, self.u0, self.u_ref = op, op.rt.to_device(u0), op.rt.to_device(u_ref)
        self.t_end, self.lam = float(t_end), float(lam)

    def steps(self, cfl: float):
        return _steps(self.t_end, cfl, self.op.mesh.dx, self.lam, self.op.mesh.degree)

    def error(self, u) -> float:
        """``cli._rel_l2`` (``cli.py:861-864``): mass-weighted relative L2."""
        den = self.op.norm_l2(self.u_ref)
        err = self.op.norm_l2(u - self.u_ref)
        return err if den == 0 else err / den


class MLSDCStudy(_Study):
    """One march = integrate_mlsdc with k V-cycles per step (``cli._march``,
    ``cli.py:849-858``) on a GPU hierarchy."""

    def __init__(self, hierarchy, u0, u_ref, t_end: float, lam: float, strategy: str = "fmg", c_fmg: int = 1):
        super().__init__(hierarchy.fine.ctx, u0, u_ref, t_end, lam)
        self.hier, self.strategy, self.c_fmg = hierarchy, strategy, c_fmg

    def march(self, cfl: float, k: int):
        from .mlsdc import integrate_mlsdc
        dt, n = self.steps(cfl)
        self.op.rt.reset_status()   # each march is independent (cli.py:1110-1138): clear latched failures
        return integrate_mlsdc(self.hier, self.u0, 0.0, dt, n, k, strategy=self.strategy, c_fmg=self.c_fmg)


class SDCStudy(_Study):
    """One march = n_steps single-level run_sdc slabs with k sweeps
    (``cli._march_single``, ``cli.py:839-846``)."""

    def __init__(self, op, rule, weights, scheme, u0, u_ref, t_end: float, lam: float, form="incremental",
                 start="predictor"):
        super().__init__(op, u0, u_ref, t_end, lam)
        self.rule, self.weights, self.scheme, self.form, self.start = rule, weights, scheme, form, start

    def march(self, cfl: float, k: int):
        from .sdc import run_sdc
        dt, n = self.steps(cfl)
        self.op.rt.reset_status()   # each march is independent (cli.py:1110-1138): clear latched failures
        u, t = self.u0, 0.0
        for _ in range(n):
            u = run_sdc(self.op, self.rule, self.weights, dt, self.scheme, u, t, k, form=self.form,
                        start=self.start).end_value.clone()
            t += dt
        self.op.rt.raise_on_failure()
        return u


def sweep_one_cfl(study, cfl: float, max_iterations: int) -> SweepPoint:
    """Error-vs-iterations series at one CFL, stopping once it stalls
    (``cli._sweep_one_cfl``, ``cli.py:1110-1138``)."""
    _, n_steps = study.steps(cfl)
    pt = SweepPoint(float(cfl), int(n_steps))
    for k in range(max_iterations + 1):
        try:
            u = study.march(cfl, k)
        except (SolverError, ValueError):   # a state leaving the admissible set is a solver failure
            pt.status = "failed"
            break
        e = study.error(u)
        if not np.isfinite(e):
            pt.status = "failed"
            break
        pt.errors.append(float(e))
        if len(pt.errors) >= 2 and converged_iteration(pt.errors) is not None:
            break
    pt.stall = converged_iteration(pt.errors) if len(pt.errors) >= 2 else None
    return pt


def _group():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist, dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return None, 0, 1


def cfl_sweep(study_or_factory, cfl_values: Sequence[float], max_iterations: int = 25,
              out_dir=None, sweep_fn: Callable = sweep_one_cfl) -> List[SweepPoint]:
    """Run the sweep with point i on rank i % world (every rank's GPU holds its
    own study objects: ``study_or_factory`` is a study or a zero-argument
    callable building one on the rank).  All ranks return the full ordered
    list; rank 0 writes errors.csv / iterations.csv into ``out_dir``
    (``cli.py:1160-1176``) and returns {file: sha256} in ``cfl_sweep.outputs``."""
    dist, rank, world = _group()
    mine = [(i, float(c)) for i, c in enumerate(cfl_values) if i % world == rank]
    study = None
    res = {}
    for i, c in mine:
        if study is None:
            is_study = hasattr(study_or_factory, "march") and not isinstance(study_or_factory, type)
            study = study_or_factory if is_study else study_or_factory()
        pt = sweep_fn(study, c, max_iterations)
        pt.rank = rank
        res[i] = pt
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        for part in gathered:
            res.update(part)
    points = [res[i] for i in range(len(cfl_values))]
    cfl_sweep.outputs = {}
    if out_dir is not None and rank == 0:
        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        err_rows, it_rows = [], []
        for p in points:
            for k, e in enumerate(p.errors):
                err_rows.append((p.cfl, p.n_steps, k, e))
            e_at = p.errors[p.stall] if p.stall is not None else (p.errors[-1] if p.errors else math.nan)
            it_rows.append((p.cfl, p.n_steps, "" if p.stall is None else p.stall, e_at, p.status))
        cfl_sweep.outputs = {
            "errors.csv": write_csv(out / "errors.csv", ("cfl", "n_steps", "iterations", "error"), err_rows),
            "iterations.csv": write_csv(out / "iterations.csv",
                                        ("cfl", "n_steps", "converged_iteration", "error", "status"), it_rows),
        }
    return points


def observed_order(e_coarse: float, e_fine: float, ratio: float = 2.0) -> float:
    """log(e_c / e_f) / log(ratio) (``analysis.py:291-297``)."""
    if e_coarse <= 0.0 or e_fine <= 0.0:
        raise ValueError("observed order needs strictly positive errors")
    if ratio <= 1.0:
        raise ValueError("refinement ratio must exceed 1")
    return float(np.log(e_coarse / e_fine) / np.log(ratio))


def convergence(run_job: Callable, element_counts: Sequence[Sequence[int]], cfl_values: Sequence[float],
                out_dir=None):
    """The reference's convergence study (``cli.py:1194-1256``): one job per
    (cfl, element-count family), each a full march at fixed iterations whose
    terminal error against the exact solution is returned by
    ``run_job(n_elems, cfl) -> (n_steps, error)`` on the rank that owns it
    (job j on rank j % world); rank 0 writes errors.csv / orders.csv in the
    reference's format.  Returns the ordered [(cfl, family, n_elem_fine,
    n_steps, error)] rows on every rank."""
    dist, rank, world = _group()
    jobs = [(fi, tuple(ne), float(c)) for c in cfl_values for fi, ne in enumerate(element_counts)]
    res = {}
    for j, (fi, ne, c) in enumerate(jobs):
        if j % world == rank:
            n_steps, err = run_job(ne, c)
            res[j] = (c, fi, ne[-1], int(n_steps), float(err))
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        for part in gathered:
            res.update(part)
    err_rows = [res[j] for j in range(len(jobs))]
    convergence.outputs = {}
    if out_dir is not None and rank == 0:
        table = {(r[0], r[1]): (r[2], r[4]) for r in err_rows}
        order_rows = []
        for c in cfl_values:
            c = float(c)
            for fi in range(1, len(element_counts)):
                ne_c, e_c = table[(c, fi - 1)]
                ne_f, e_f = table[(c, fi)]
                if e_c <= 0 or e_f <= 0:
                    order_rows.append((c, fi - 1, fi, ""))
                    continue
                order_rows.append((c, fi - 1, fi, observed_order(e_c, e_f, ratio=ne_f / ne_c)))
        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        convergence.outputs = {
            "errors.csv": write_csv(out / "errors.csv", ("cfl", "family", "n_elem_fine", "n_steps", "error"),
                                    err_rows),
            "orders.csv": write_csv(out / "orders.csv", ("cfl", "family_coarse", "family_fine", "order"),
                                    order_rows),
        }
    return err_rows
