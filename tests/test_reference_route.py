"""The reference's OWN solver path with its implicit solve routed through the
C-ABI: the unmodified reference package (oracle/_ref, built by
oracle/build_ref.py) runs ``sisdc.mlsdc.run_mlsdc`` with
``DGOperator.implicit_solve`` patched by the reference-side binding of
INTEGRATION.md (integration/sisdc_b200_binding.py, executed as written).
One SI-MLSDC step of cfg1 and cfg2 agrees with the unpatched reference
(SuperLU) to <= 1e-11 relative L2 (north-star tolerance)."""
import importlib.util
import os

import numpy as np
import pytest

from conftest import REPO, gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def binding():
    spec = importlib.util.spec_from_file_location("sisdc_b200_binding",
                                                  os.path.join(REPO, "integration", "sisdc_b200_binding.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_reference_run_mlsdc_through_cabi(cfg):
    from oracle import build_ref, refrun
    if not build_ref.installed():
        pytest.fail("oracle/_ref is missing: run oracle/build_ref.py in the build container (it ships with the repo)")
    sisdc = build_ref.import_reference()
    import sisdc.mlsdc  # noqa: F401
    from paper_2504_18526_b200 import _lib
    from paper_2504_18526_b200.configs import WORKLOADS
    w = WORKLOADS[cfg]
    _, u0, dt, _ = refrun.initial(w)
    u_lu = sisdc.mlsdc.run_mlsdc(refrun.build_hierarchy(w), u0, 0.0, dt, w.n_cycles, strategy="fmg").end_value
    b = binding()
    calls = []
    L = b.install(sisdc, _lib.LIB_PATH)
    try:
        orig_solve = L.solve

        def counting(*a):
            calls.append(1)
            return orig_solve(*a)
        L.solve = counting
        u_gpu = sisdc.mlsdc.run_mlsdc(refrun.build_hierarchy(w), u0, 0.0, dt, w.n_cycles,
                                      strategy="fmg").end_value
    finally:
        b.uninstall(sisdc)
    assert len(calls) > 50                       # every implicit substep went through the C-ABI
    err = np.linalg.norm(u_gpu - u_lu) / np.linalg.norm(u_lu)
    assert err <= 1e-11, err
