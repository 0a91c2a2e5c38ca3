"""Element-row partitioned 2-D path on one GPU.

A partitioned operator with R local partitions (the single-GPU emulation of R
ranks: halo exchange and CG allreduce as device copies and fixed-order sums)
and a 1-rank NCCL operator (halo by NCCL send/recv to itself, allreduce by
NCCL) against the single-domain path:
  * operators (convection, SIP, eval_rhs, coefficient field, node caches) are
    per-node identical, so they agree BITWISE;
  * the split Chronopoulos-Gear CG reduces in a different order than the
    cooperative k2_cg: solutions <= 1e-13 relative, identical iterations;
  * one SI-MLSDC step: <= 1e-11 relative L2 vs the single domain and the 2-D
    restatement, identical CG iteration sequence.
"""
import dataclasses

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_2504_18526_b200.configs import CFG3, CFG4  # noqa: E402


def small(w, nex, ney=None):
    return dataclasses.replace(w, nex=nex, ney=ney or nex)


@pytest.fixture(scope="module")
def rt():
    from paper_2504_18526_b200.runtime import get_runtime
    r = get_runtime()
    r.set_cg(rtol=1e-14, maxit=1000, cluster_ctas=0)
    return r


@pytest.fixture(scope="module")
def comm1(rt):
    from paper_2504_18526_b200 import dgsem2d
    return dgsem2d.NcclComm(0, 1)


def ops(w, P, partition):
    from paper_2504_18526_b200 import dgsem2d
    L = w.length
    mesh = dgsem2d.Mesh2D(0.0, L, 0.0, L, w.nex, w.ney, P)
    prob = w.gpu_problem()
    one = dgsem2d.DGOperator2D(mesh, prob)
    part = dgsem2d.DGOperator2D(mesh, prob, partition=partition)
    X, Y = mesh.nodes_xy
    return one, part, w.initial_state(X, Y)


def glob(op, v):
    return op.gather(v).reshape(-1)


def parts(comm1):
    from paper_2504_18526_b200.dgsem2d import Partition
    return [Partition(1), Partition(2), Partition(3), Partition(4), Partition(1, comm1)]


@pytest.mark.parametrize("P", [7, 3])
def test_partitioned_operators_bitwise(rt, comm1, P):
    w = small(CFG4, 5, 8)
    for part in parts(comm1):
        one, op, u = ops(w, P, part)
        us = op.scatter(u)
        assert np.array_equal(glob(op, op.apply_convection(us)), one.apply_convection(u).cpu().numpy())
        assert np.array_equal(glob(op, op.eval_rhs(us)), one.eval_rhs(u).cpu().numpy())
        c1, cp = one.modified_diffusion_matrix(u, 3e-3, "si2"), op.modified_diffusion_matrix(us, 3e-3, "si2")
        assert np.array_equal(glob(op, op.apply_diffusion(cp, us)), one.apply_diffusion(c1, u).cpu().numpy())
        assert np.array_equal(glob(op, op.apply_diffusion(0.0123, us)), one.apply_diffusion(0.0123, u).cpu().numpy())
        # coefficient field: scalar layout (rows + 2 per partition)
        cf = op.coefficient_field(cp).view(op.slab_rows, w.nex, P + 1, P + 1)
        ref = one.coefficient_field(c1).view(w.ney, w.nex, P + 1, P + 1).cpu().numpy()
        r = 0
        for rb, rows, _ in op.parts:
            assert np.array_equal(cf[r + 1:r + 1 + rows].cpu().numpy(), ref[rb:rb + rows])
            r += rows + 2


def test_partitioned_node_caches_bitwise(rt, comm1):
    """Fused node caches (f, h1, h2 over all M nodes, P = 7 tensor-core path)."""
    from paper_2504_18526_b200 import sdc
    from paper_2504_18526_b200.collocation import make_nodes
    w = small(CFG4, 4, 6)
    rule = make_nodes("radau_right", 3)
    dt = 2e-3
    for part in parts(comm1):
        one, op, u = ops(w, 7, part)
        rng = np.random.default_rng(7)
        nodes = [u * (1.0 + 1e-3 * rng.standard_normal(u.shape)) for _ in range(3)]
        s1 = sdc.from_nodes(one, rule, dt, "si2", u, 0.0, np.stack(nodes))
        sp = sdc.from_nodes(op, rule, dt, "si2", op.scatter(u), 0.0,
                            np.stack([op.scatter(x).cpu().numpy() for x in nodes]))
        for a, b in ((s1.f, sp.f), (s1.h1, sp.h1), (s1.h2, sp.h2)):
            for m in range(3):
                assert np.array_equal(glob(op, b[m]), a[m].cpu().numpy())


@pytest.mark.parametrize("nex,ney,P", [(6, 8, 7), (5, 7, 3), (6, 8, 3), (2, 16, 3), (34, 12, 3)])
def test_partitioned_implicit_solve(rt, comm1, nex, ney, P):
    w = small(CFG4, nex, ney)
    for part in parts(comm1):
        one, op, u = ops(w, P, part)
        us = op.scatter(u)
        for a in (2e-3, 5e-2):
            n0 = rt.status()[2]
            x1 = one.implicit_solve(one.modified_diffusion_matrix(u, a, "si2"), a, u)
            it1 = rt.cg_log()[0][n0:].tolist()
            n0 = rt.status()[2]
            xp = op.implicit_solve(op.modified_diffusion_matrix(us, a, "si2"), a, us)
            itp = rt.cg_log()[0][n0:].tolist()
            assert itp == it1, (part, a)
            ref = x1.cpu().numpy()
            assert np.abs(glob(op, xp) - ref).max() / np.abs(ref).max() < 1e-13
    rt.raise_on_failure()


def test_partitioned_zero_rhs(rt):
    from paper_2504_18526_b200 import dgsem2d
    w = small(CFG4, 4, 4)
    one, op, u = ops(w, 7, dgsem2d.Partition(2))
    z = rt.zeros(op.ndof)
    n0 = rt.status()[2]
    x = op.implicit_solve(op.modified_diffusion_matrix(op.scatter(u), 1e-3, "si2"), 1e-3, z)
    assert rt.cg_log()[0][n0:].tolist() == [0]
    assert np.all(glob(op, x) == 0.0)


def run_step(w, partition, rt):
    from paper_2504_18526_b200 import dgsem, dgsem2d, mlsdc
    L = w.length
    mk = lambda P: dgsem2d.DGOperator2D(dgsem2d.Mesh2D(0.0, L, 0.0, L, w.nex, w.ney, P),
                                        w.gpu_problem(), partition=partition)
    h = mlsdc.build_p_hierarchy(mk, [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
    X, Y = h.fine.ctx.mesh.nodes_xy
    u0 = w.initial_state(X, Y)
    dt = w.time_step(u0, dgsem.compute_delta(w.p_fine))
    n0 = rt.status()[2]
    sol = mlsdc.run_mlsdc(h, h.fine.ctx.scatter(u0), 0.0, dt, w.n_cycles, strategy="fmg")
    rt.raise_on_failure()
    return h.fine.ctx.gather(sol.u[-1]).reshape(-1), rt.cg_log()[0][n0:].tolist()


@pytest.mark.parametrize("base,nex,ney", [(CFG4, 5, 6), (CFG3, 4, 5)])
def test_partitioned_mlsdc_step(rt, comm1, base, nex, ney):
    """One SI-MLSDC step (P 7/3, 3 V-cycles): every partition count and the
    NCCL path agree with the single domain to <= 1e-11 with identical CG
    iteration sequences."""
    from paper_2504_18526_b200 import dgsem2d
    w = small(base, nex, ney)
    ref, its = run_step(w, None, rt)
    for part in [dgsem2d.Partition(2), dgsem2d.Partition(3), dgsem2d.Partition(ney), dgsem2d.Partition(1, comm1)]:
        u, itp = run_step(w, part, rt)
        assert itp == its, part
        assert np.linalg.norm(u - ref) / np.linalg.norm(ref) < 1e-11, part


def test_partitioned_slab_graph_replays_like_eager(rt, comm1):
    """A partitioned slab is CUDA-graph capturable: inside a capture the split solve records a
    fixed-length iteration batch (kernels return at once after convergence, the closing scalar
    kernel latches a failure if the batch was too short).  A replay equals the eager slab bitwise,
    with the same CG iteration log, for in-process partitions and one NCCL rank."""
    from paper_2504_18526_b200 import dgsem, dgsem2d, mlsdc
    w = small(CFG4, 5, 6)
    for part in (dgsem2d.Partition(2), dgsem2d.Partition(1, comm1)):
        h = mlsdc.build_p_hierarchy(
            lambda P: dgsem2d.DGOperator2D(dgsem2d.Mesh2D(0.0, w.length, 0.0, w.length, w.nex, w.ney, P),
                                           w.gpu_problem(), partition=part),
            [w.p_coarse, w.p_fine], [w.m_coarse, w.m_fine])
        fine = h.fine.ctx
        X, Y = fine.mesh.nodes_xy
        u0 = w.initial_state(X, Y)
        dt = w.time_step(u0, dgsem.compute_delta(w.p_fine))
        us = fine.scatter(u0)
        n0 = rt.status()[2]
        eager = mlsdc.run_mlsdc(h, us, 0.0, dt, w.n_cycles, strategy="fmg").u[-1].clone()
        its_e = rt.cg_log()[0][n0:].tolist()
        g = mlsdc.SlabGraph(h, us, 0.0, dt, w.n_cycles, "fmg")
        n1 = rt.status()[2]
        g.step()
        rt.synchronize()
        assert rt.cg_log()[0][n1:].tolist() == its_e
        assert bool((g.u == eager).all())
        rt.raise_on_failure()


@pytest.mark.parametrize("nex,ney,nparts,P", [(4, 48, -1, 7), (3, 25, -1, 7), (4, 50, 2, 7), (4, 96, -1, 3), (6, 100, 2, 3)])
def test_partitioned_solve_halo_overlap(rt, comm1, monkeypatch, nex, ney, nparts, P):
    """Partitions of >= 3 bands (24+ element rows) run the fused iteration with the halo overlapped:
    the exchange and the two ghost-row bands on the operator's second stream, the interior bands on
    the main stream (part2d.cu iterate_fused).  Same iterations as the single domain, <= 1e-13, for
    in-process partitions and one NCCL rank (nparts -1; packed send / receive buffers), eager and
    replayed from a CUDA graph (solves within the captured batch of 32 iterations).  Single-GPU
    runs overlap only under SISDC_PART_OVERLAP=1 (read per solve): there is no transfer to hide."""
    import torch
    monkeypatch.setenv("SISDC_PART_OVERLAP", "1")
    from paper_2504_18526_b200 import dgsem2d
    w = small(CFG4, nex, ney)
    part = dgsem2d.Partition(1, comm1) if nparts < 0 else dgsem2d.Partition(nparts)
    one, op, u = ops(w, P, part)   # P = 3: the fused 2 x 2-tile pass (even rows per partition), bands of 16 rows
    us = op.scatter(u)
    for a in (2e-3, 5e-2):
        n0 = rt.status()[2]
        x1 = one.implicit_solve(one.modified_diffusion_matrix(u, a, "si2"), a, u)
        it1 = rt.cg_log()[0][n0:].tolist()
        cp = op.modified_diffusion_matrix(us, a, "si2")
        n0 = rt.status()[2]
        xp = op.implicit_solve(cp, a, us).clone()
        assert rt.cg_log()[0][n0:].tolist() == it1, (part, a)
        ref = x1.cpu().numpy()
        assert np.abs(glob(op, xp) - ref).max() / np.abs(ref).max() < 1e-13
        if it1[0] > 30:
            continue
        # the same solve captured (fixed-length batch, both streams inside the capture) and replayed
        out = torch.empty_like(us)
        rt.synchronize()
        g = torch.cuda.CUDAGraph()
        stream = torch.cuda.Stream(device=rt.device)
        stream.wait_stream(torch.cuda.current_stream(rt.device))
        op.eager_checks = False          # no status read-back inside a capture (as SlabGraph's sweeps)
        with torch.cuda.graph(g, stream=stream):
            rt.bind_stream()
            op.implicit_solve(cp, a, us, out=out)
        op.eager_checks = True
        rt.bind_stream()
        n0 = rt.status()[2]
        g.replay()
        rt.synchronize()
        assert rt.cg_log()[0][n0:].tolist() == it1
        assert bool((out == xp).all())
    rt.raise_on_failure()
