"""Host-side setup of the product package: collocation tables, transfer
matrices, delta(P), workload generators -- against the reference goldens."""
import numpy as np
import pytest

from paper_2504_18526_b200 import collocation as col
from paper_2504_18526_b200.configs import CFG1, CFG2
from paper_2504_18526_b200.dgsem import compute_delta, dt_from_cfl, Mesh1D
from paper_2504_18526_b200.transfer import build_spatial_p_transfer, build_temporal_transfer


def test_collocation_tables(golden):
    G = golden["tables"]
    for M in (1, 2, 3, 4, 5, 7):
        r = col.make_nodes("radau_right", M)
        w = col.make_weights(r)
        assert np.abs(r.tau - G[f"radau_tau_{M}"]).max() < 1e-15
        assert np.abs(w.w_nn - G[f"radau_wnn_{M}"]).max() < 1e-14
        assert np.abs(w.w_0n - G[f"radau_w0n_{M}"]).max() < 1e-14
    for M in (2, 3, 5):
        assert np.abs(col.make_nodes("lobatto", M).tau - G[f"lobatto_tau_{M}"]).max() < 1e-15
    for P in (3, 4, 7, 8):
        x, w = col.gauss_lobatto(P + 1)
        assert np.abs(x - G[f"gll_x_{P}"]).max() < 1e-15
        assert np.abs(w - G[f"gll_w_{P}"]).max() < 1e-15
        assert abs(compute_delta(P) - float(G[f"delta_{P}"])) < 1e-12


def test_transfer_matrices(golden):
    G = golden["tables"]
    for pc, pf in ((4, 8), (3, 7)):
        s = build_spatial_p_transfer(pc, pf, 1)
        assert np.abs(s.blocks["interp"] - G[f"psp_interp_{pc}_{pf}"]).max() < 1e-14
        assert np.abs(s.blocks["project"] - G[f"psp_project_{pc}_{pf}"]).max() < 1e-14
        assert np.array_equal(s.blocks["restrict"], s.blocks["interp"].T)
    for mc, mf in ((2, 4), (3, 5), (2, 5)):
        p = build_temporal_transfer(col.make_nodes("radau_right", mc), col.make_nodes("radau_right", mf))
        assert np.abs(p.interp - G[f"t_interp_{mc}_{mf}"]).max() < 1e-14
        assert np.abs(p.project - G[f"t_project_{mc}_{mf}"]).max() < 1e-14
        assert np.array_equal(p.restrict, p.interp.T)


def test_workloads(golden):
    G = golden["trajectories"]
    for tag, w in (("cfg1", CFG1), ("cfg2", CFG2)):
        mesh = Mesh1D(w.x_left, w.x_right, w.n_elem, w.p_fine)
        u0 = w.initial_state(mesh.ref_nodes)
        assert np.abs(u0 - G[f"{tag}_u0"]).max() < 1e-14
        dt, n = w.time_step(u0, compute_delta(w.p_fine))
        assert abs(dt - float(G[f"{tag}_dt"])) < 1e-17
        if tag == "cfg2":
            assert n == int(G["cfg2_nsteps_total"]) and abs(n * dt - 1.5) < 1e-12
    assert CFG1.dof_sweeps_per_step()[0] == 576 * 4 * 6 + 320 * 2 * 12
    assert CFG2.dof_sweeps_per_step()[0] == 4608 * 5 * 4 + 2560 * 3 * 8


def test_mesh_validation():
    with pytest.raises(ValueError):
        Mesh1D(1.0, 0.0, 4, 3)
    with pytest.raises(ValueError):
        Mesh1D(0.0, 1.0, 0, 3)
    with pytest.raises(ValueError):
        Mesh1D(0.0, 1.0, 4, 3, bc="outflow")
    assert dt_from_cfl(2.0, 0.1, 1.0, 8) == pytest.approx(2.0 * 0.1 / (2 * compute_delta(8)))


def test_h_transfer_blocks_match_reference(golden):
    """Host-side h-transfer blocks (transfer.py:248-317) applied per parent
    element reproduce the reference's apply() for every jump policy and the l2
    projection; the p-transfer l2 projection likewise."""
    import numpy as np
    from paper_2504_18526_b200.transfer import build_spatial_h_transfer, build_spatial_p_transfer
    G = golden["htransfer"]
    for pol, kind in (("linear_blend", "embedded"), ("average", "embedded"), ("linear_blend", "l2")):
        st = build_spatial_h_transfer(6, 5, 1, kind, pol)
        tag = f"h_{pol}_{kind}"
        uc, uf = G[f"{tag}_uc"], G[f"{tag}_uf"]
        I, P, R = st.blocks["interp"], st.blocks["project"], st.blocks["restrict"]
        got = {"interp": np.einsum("ij,ej->ei", I, uc.reshape(6, 6)).reshape(-1),
               "project": np.einsum("ij,ej->ei", P, uf.reshape(6, 12)).reshape(-1),
               "restrict": np.einsum("ij,ej->ei", R, uf.reshape(6, 12)).reshape(-1)}
        for d, v in got.items():
            assert np.abs(v - G[f"{tag}_{d}"]).max() < 1e-13, (tag, d)
    sp = build_spatial_p_transfer(3, 7, 5, 1, "l2")
    v = np.einsum("ij,ej->ei", sp.blocks["project"], G["p_l2_uf"].reshape(5, 8)).reshape(-1)
    assert np.abs(v - G["p_l2_project"]).max() < 1e-13


def test_nvtx_ranges_wrap_the_sweep_entry_points(monkeypatch):
    """SISDC_NVTX=1 puts every host entry point of the sweep path in a named NVTX range."""
    import importlib
    import torch
    from paper_2504_18526_b200 import trace
    calls = []
    monkeypatch.setattr(torch.cuda.nvtx, "range_push", lambda n: calls.append(("push", n)))
    monkeypatch.setattr(torch.cuda.nvtx, "range_pop", lambda: calls.append(("pop", None)))
    monkeypatch.setattr(trace, "ENABLED", True)
    f = trace.traced("sisdc.unit")(lambda x: x + 1)
    assert f(1) == 2 and calls == [("push", "sisdc.unit"), ("pop", None)]
    with pytest.raises(ZeroDivisionError):
        trace.traced("sisdc.err")(lambda: 1 / 0)()
    assert calls[-1] == ("pop", None)          # the range closes on exceptions too
    monkeypatch.setattr(trace, "ENABLED", False)
    g = lambda: 0                               # noqa: E731
    assert trace.traced("x")(g) is g            # disabled: the function itself, no wrapper
    from paper_2504_18526_b200 import mlsdc, sdc
    src = open(mlsdc.__file__).read() + open(sdc.__file__).read()
    for name in ("v_cycle", "start", "run_mlsdc", "sweep", "predict", "solve"):
        assert f'@traced("sisdc.{name}")' in src
