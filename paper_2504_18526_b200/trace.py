"""NVTX ranges per slab / V-cycle / sweep / implicit solve (tracing).

``SISDC_NVTX=1`` wraps the host entry points of the sweep path in
``torch.cuda.nvtx`` ranges, so that an Nsight Systems / ncu ``--nvtx`` capture
groups the kernels by algorithmic phase; without it ``traced`` returns the
function unchanged (no per-call cost on the launch-bound 1-D path).
"""
from __future__ import annotations

import functools
import os

ENABLED = os.environ.get("SISDC_NVTX", "0") == "1"


def traced(name: str):
    def deco(fn):
        if not ENABLED:
            return fn
        import torch

        @functools.wraps(fn)
        def wrapper(*a, **k):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **k)
            finally:
                torch.cuda.nvtx.range_pop()
        return wrapper
    return deco
