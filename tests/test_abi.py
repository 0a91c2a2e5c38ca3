"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
public header declares (no compute calls: this runs without a GPU)."""
import ctypes as C
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "sisdc_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sisdc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2504_18526_b200 import build, _lib
    build.build()
    return _lib.load()


def test_header_symbols_bound_and_exported(lib):
    from paper_2504_18526_b200._lib import SIGNATURES
    names = declared()
    assert len(names) >= 30
    missing_bind = [n for n in names if n not in SIGNATURES]
    assert not missing_bind, missing_bind
    for n in names:
        assert hasattr(lib, n), n
    assert set(SIGNATURES) <= set(names)


def test_abi_version(lib):
    assert lib.sisdc_abi_version() == 2


def test_sm100a_cubin():
    """The shared library carries sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    from paper_2504_18526_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_is_a_clean_error(lib):
    """Without a GPU the context constructor fails with an error code, never
    silently succeeding (there is no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = lib.sisdc_ctx_create(0, C.byref(h))
    assert rc != 0


def test_product_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_18526_b200 import dgsem, problems
    from paper_2504_18526_b200._lib import LibraryError
    with pytest.raises(LibraryError):
        dgsem.DGOperator(dgsem.Mesh1D(0.0, 1.0, 4, 3), problems.ConvectionDiffusion(1.0, 0.01))


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2504_18526_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_reference_binding_structs_match_library(lib):
    """The reference-side ctypes binding shown in INTEGRATION.md
    (integration/sisdc_b200_binding.py) mirrors the header's PODs byte for
    byte (ABI v2: 13-field sisdc_op1d_desc)."""
    import importlib.util
    from paper_2504_18526_b200 import _lib
    spec = importlib.util.spec_from_file_location("sisdc_b200_binding",
                                                  os.path.join(REPO, "integration", "sisdc_b200_binding.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert lib.sisdc_struct_size(0) == C.sizeof(b.Desc) == C.sizeof(_lib.Op1DDesc)
    assert lib.sisdc_struct_size(2) == C.sizeof(b.Coef) == C.sizeof(_lib.Coef)
    assert lib.sisdc_struct_size(1) == C.sizeof(_lib.Op2DDesc)
    assert [f[0] for f in b.Desc._fields_] == [f[0] for f in _lib.Op1DDesc._fields_]
    # INTEGRATION.md embeds the binding verbatim
    doc = open(os.path.join(REPO, "INTEGRATION.md")).read()
    assert open(os.path.join(REPO, "integration", "sisdc_b200_binding.py")).read().strip() in doc
