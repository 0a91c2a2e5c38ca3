"""Per-device runtime: the native context, stream binding and status checks."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import LibraryError, SolverError

_RUNTIMES: dict = {}


class Runtime:
    """One libsisdc context per CUDA device (one process drives one GPU)."""

    def __init__(self, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise LibraryError("no CUDA device: the sweep path runs only on the GPU (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.sisdc_ctx_create(device, C.byref(h))
        if rc:
            raise LibraryError(f"sisdc_ctx_create failed ({rc})")
        self.h = h
        self._stream = None
        self.rtol = 1e-14
        self.maxit = 1000
        self.cluster_ctas = 0
        self.bind_stream()

    def __del__(self):
        try:
            self.lib.sisdc_ctx_destroy(self.h)
        except Exception:
            pass

    # ------------------------------------------------------------ plumbing
    def bind_stream(self):
        s = self.torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            self.lib.sisdc_ctx_set_stream(self.h, C.c_void_p(s))
            self._stream = s

    def check(self, rc: int, what: str = ""):
        if rc == 0:
            return
        msg = (self.lib.sisdc_ctx_last_error(self.h) or b"").decode()
        if rc in (_lib.ERR_NONFINITE, _lib.ERR_NOCONV):
            raise SolverError(f"{what}: {msg}")
        if rc == _lib.ERR_ARG:
            raise ValueError(f"{what}: {msg}")
        raise LibraryError(f"{what}: error {rc}: {msg}")

    def set_cg(self, rtol: float = 1e-14, maxit: int = 1000, cluster_ctas: int = 0):
        self.check(self.lib.sisdc_ctx_set_cg(self.h, float(rtol), int(maxit), int(cluster_ctas)), "set_cg")
        self.rtol, self.maxit, self.cluster_ctas = rtol, maxit, cluster_ctas

    def synchronize(self):
        self.check(self.lib.sisdc_ctx_synchronize(self.h), "synchronize")

    def reset_status(self):
        self.bind_stream()
        self.check(self.lib.sisdc_ctx_reset_status(self.h), "reset_status")

    def reset_log(self):
        """Forget the per-solve CG log (the device counter restarts at 0); the log keeps the first
        2^20 solves after a reset, so long sessions (studies, test suites) reset it per run."""
        self.bind_stream()
        self.check(self.lib.sisdc_ctx_reset_log(self.h), "reset_log")

    def status(self):
        e, f, n = C.c_int(), C.c_int(), C.c_int()
        self.check(self.lib.sisdc_ctx_status(self.h, C.byref(e), C.byref(f), C.byref(n)), "status")
        return e.value, f.value, n.value

    def raise_on_failure(self):
        """Map latched device failures to the reference's SolverError
        (``dgsem.py:348-351``, ``:530-533``)."""
        bad, fails, _ = self.status()
        if bad >= 0:
            raise SolverError(f"non-finite right-hand side in element {bad}")
        if fails > 0:
            raise SolverError(f"implicit CG solve did not converge within {self.maxit} iterations "
                              f"({fails} solve(s))")

    def cg_log(self):
        n = C.c_int()
        self.check(self.lib.sisdc_ctx_cg_log(self.h, 0, None, None, C.byref(n)), "cg_log")
        cnt = min(n.value, 1 << 20)   # Ctx::log_cap
        it = (C.c_int * max(cnt, 1))()
        mg = (C.c_double * max(cnt, 1))()
        self.check(self.lib.sisdc_ctx_cg_log(self.h, cnt, it, mg, C.byref(n)), "cg_log")
        return np.array(it[:cnt], dtype=np.int64), np.array(mg[:cnt])

    def launch_count(self) -> int:
        return int(self.lib.sisdc_ctx_launch_count(self.h))

    def copy(self, dst, src):
        self.bind_stream()
        self.check(self.lib.sisdc_copy(self.h, dst.data_ptr(), src.data_ptr(), dst.numel()), "copy")

    def lincomb(self, out, *terms):
        """out = sum c_k v_k over up to four (c, v) pairs, on the device."""
        if not 1 <= len(terms) <= 4:
            raise ValueError("one to four terms")
        cs = (C.c_double * 4)(*([float(c) for c, _ in terms] + [0.0] * (4 - len(terms))))
        vs = [v.data_ptr() for _, v in terms] + [None] * (4 - len(terms))
        self.bind_stream()
        self.check(self.lib.sisdc_lincomb(self.h, out.numel(), cs, *vs, out.data_ptr()), "lincomb")
        return out

    # ------------------------------------------------------------- buffers
    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64, device=self.device)

    def zeros(self, *shape):
        return self.torch.zeros(*shape, dtype=self.torch.float64, device=self.device)

    def to_device(self, a):
        t = self.torch
        if isinstance(a, t.Tensor):
            if a.device == self.device and a.dtype == t.float64:
                return a.contiguous()
            return a.to(device=self.device, dtype=t.float64).contiguous()
        return t.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.device)


def get_runtime(device: int = 0) -> Runtime:
    rt = _RUNTIMES.get(device)
    if rt is None:
        rt = Runtime(device)
        _RUNTIMES[device] = rt
    return rt
