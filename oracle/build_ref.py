"""Install the UNMODIFIED reference package into ``oracle/_ref`` (TEST / BENCH
INFRASTRUCTURE ONLY -- the product package never imports it).

The reference (``/root/reference/pkg``, pure Python: ``sisdc``) is built with
its own ``pyproject.toml`` by pip, offline, from a scratch copy under /tmp
(``/root/reference`` is read-only), into ``oracle/_ref`` (git-ignored, NOT
gpurun-ignored: it travels to the GPU box, where ``/root/reference`` does not
exist).  Nothing is copied into the repo's history.

``bench.py --impl reference`` and the ``cpu_baseline`` leg time this install
through the reference's own public API (``sisdc.mlsdc.run_mlsdc`` with its
SuperLU implicit solve, ``dgsem.py:503-533``); ``tests/test_reference_route.py``
routes its ``DGOperator.implicit_solve`` through the C-ABI.

    python oracle/build_ref.py [--force]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg"
TARGET = os.path.join(HERE, "_ref")


def installed() -> bool:
    return os.path.isfile(os.path.join(TARGET, "sisdc", "mlsdc.py"))


def build(force: bool = False) -> str | None:
    """Build the install if the reference source is present (build container
    only); returns the target directory or None when neither exists."""
    if installed() and not force:
        return TARGET
    if not os.path.isdir(REF_SRC):
        return TARGET if installed() else None
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_SRC, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache"))
        if os.path.isdir(TARGET):
            shutil.rmtree(TARGET)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--target", TARGET, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("pip install of the reference failed")
    return TARGET


def import_reference():
    """Import the installed reference package ``sisdc`` (raises ImportError
    when oracle/_ref was not built)."""
    if not installed():
        raise ImportError("oracle/_ref is not built (python oracle/build_ref.py in the build container)")
    if TARGET not in sys.path:
        sys.path.insert(0, TARGET)
    import sisdc  # noqa: F401
    if not os.path.abspath(sisdc.__file__).startswith(TARGET):
        raise ImportError(f"sisdc resolved to {sisdc.__file__}, not the oracle/_ref install")
    return sisdc


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
