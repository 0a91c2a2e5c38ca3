"""Reference-side binding: route the reference's ``DGOperator.implicit_solve``
(``pkg/src/sisdc/dgsem.py:503-533``, SuperLU + defect iteration) through the
B200 library's C ABI (``include/sisdc_b200.h``: ``sisdc_implicit_solve``,
the pinned Jacobi-PCG / element-block BiCGStab).

This is the file a maintainer of the reference adds (as ``sisdc/_b200.py``)
to switch the implicit substeps of an unmodified ``sisdc`` run to the GPU;
INTEGRATION.md shows it and ``tests/test_reference_route.py`` executes it
exactly as written, against the reference installed in ``oracle/_ref``.

    import sisdc, sisdc_b200_binding as b
    b.install(sisdc, "/path/to/libsisdc_b200.so")   # patches DGOperator.implicit_solve
    ... sisdc.mlsdc.run_mlsdc(...) ...               # implicit solves now run on the GPU
    b.uninstall(sisdc)

Only plain ctypes, numpy and a CUDA allocator (torch tensors as device
buffers) are used; the structs mirror the header and are checked against the
library's ``sisdc_struct_size``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

PERIODIC, DIRICHLET = 0, 1
CONVDIFF, BURGERS, CNS1D = 0, 1, 5
COEF_CONST, COEF_FIELD, COEF_MATRIX = 1, 2, 5


class Coef(C.Structure):          # sisdc_coef
    _fields_ = [("kind", C.c_int), ("value", C.c_double), ("ptr", C.c_void_p)]


class Desc(C.Structure):          # sisdc_op1d_desc (ABI version 2: 13 fields)
    _fields_ = [("n_elem", C.c_int), ("degree", C.c_int), ("ncomp", C.c_int), ("bc", C.c_int),
                ("problem", C.c_int), ("x_left", C.c_double), ("x_right", C.c_double),
                ("speed", C.c_double), ("nu", C.c_double), ("penalty", C.c_double),
                ("gamma", C.c_double), ("eta", C.c_double), ("prandtl", C.c_double)]


class _Lib:
    def __init__(self, path: str, device: int = 0):
        import torch
        self.torch = torch
        self.device = device
        lib = C.CDLL(path)
        lib.sisdc_abi_version.restype = C.c_int
        lib.sisdc_struct_size.argtypes = [C.c_int]
        lib.sisdc_struct_size.restype = C.c_int
        if lib.sisdc_abi_version() != 2:
            raise RuntimeError("libsisdc_b200: ABI version mismatch")
        for which, st in ((0, Desc), (2, Coef)):
            if lib.sisdc_struct_size(which) != C.sizeof(st):
                raise RuntimeError(f"libsisdc_b200: {st.__name__} layout mismatch")
        lib.sisdc_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        lib.sisdc_ctx_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        lib.sisdc_ctx_set_cg.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int]
        lib.sisdc_ctx_last_error.argtypes = [C.c_void_p]
        lib.sisdc_ctx_last_error.restype = C.c_char_p
        lib.sisdc_ctx_status.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 3
        lib.sisdc_ctx_reset_status.argtypes = [C.c_void_p]
        lib.sisdc_op1d_create.argtypes = [C.c_void_p, C.POINTER(Desc), C.POINTER(C.c_void_p)]
        lib.sisdc_op1d_destroy.argtypes = [C.c_void_p]
        lib.sisdc_op1d_destroy.restype = None
        lib.sisdc_implicit_solve.argtypes = [C.c_void_p, Coef, C.c_double, C.c_void_p, C.c_double,
                                             C.c_void_p]
        self.lib = lib
        self.ctx = C.c_void_p()
        self._check(lib.sisdc_ctx_create(device, C.byref(self.ctx)), "ctx_create")
        self.stream = torch.cuda.Stream(device=device)
        self._check(lib.sisdc_ctx_set_stream(self.ctx, C.c_void_p(self.stream.cuda_stream)), "set_stream")
        self._check(lib.sisdc_ctx_set_cg(self.ctx, 1e-14, 1000, 0), "set_cg")

    def _check(self, rc, what):
        if rc != 0:
            msg = self.lib.sisdc_ctx_last_error(self.ctx) if self.ctx else b""
            raise RuntimeError(f"libsisdc_b200 {what}: status {rc}: {(msg or b'').decode()}")

    def op_handle(self, op):
        """One library operator per reference DGOperator (periodic meshes;
        ConvectionDiffusion, Burgers, CompressibleFlow)."""
        h = getattr(op, "_b200_handle", None)
        if h is not None:
            return h
        prob = op.problem
        name = type(prob).__name__
        kind = {"ConvectionDiffusion": CONVDIFF, "Burgers": BURGERS, "CompressibleFlow": CNS1D}.get(name)
        if kind is None or op.mesh.bc != "periodic" or op.av is not None or getattr(prob, "source", None):
            return None
        d = Desc(op.mesh.n_elem, op.mesh.degree, op.ncomp, PERIODIC, kind, op.mesh.x_left, op.mesh.x_right,
                 float(getattr(prob, "speed", 0.0) or 0.0), float(getattr(prob, "nu", 0.0) or 0.0),
                 float(op.mu0 * op.mesh.dx / op.p1 ** 2),
                 float(getattr(prob, "gamma", 1.4)), float(getattr(prob, "eta", 0.0) or 0.0),
                 float(getattr(prob, "Pr", 0.75)))
        h = C.c_void_p()
        self._check(self.lib.sisdc_op1d_create(self.ctx, C.byref(d), C.byref(h)), "op1d_create")
        op._b200_handle = h
        return h

    def solve(self, op, coeff, a, rhs, t):
        torch = self.torch
        h = self.op_handle(op)
        if h is None:
            return None
        dev = torch.device("cuda", self.device)
        with torch.cuda.stream(self.stream):
            r = torch.as_tensor(np.ascontiguousarray(rhs, dtype=np.float64).reshape(-1), device=dev)
            x = torch.empty_like(r)
            keep = None
            if np.isscalar(coeff):
                c = Coef(COEF_CONST, float(coeff), None)
            else:
                arr = np.asarray(coeff, dtype=np.float64)
                keep = torch.as_tensor(np.ascontiguousarray(arr).reshape(-1), device=dev)
                c = Coef(COEF_FIELD if arr.ndim == 2 else COEF_MATRIX, 0.0, keep.data_ptr())
            self.lib.sisdc_ctx_reset_status(self.ctx)
            self._check(self.lib.sisdc_implicit_solve(h, c, float(a), r.data_ptr(), float(t), x.data_ptr()),
                        "implicit_solve")
            bad, fails, n = C.c_int(), C.c_int(), C.c_int()
            self._check(self.lib.sisdc_ctx_status(self.ctx, C.byref(bad), C.byref(fails), C.byref(n)), "status")
            out = x.cpu().numpy()
            del keep
        if fails.value > 0:
            return "noconv"
        return out.reshape(np.shape(rhs))


_state = {}


def install(sisdc, lib_path: str, device: int = 0):
    """Patch ``sisdc.dgsem.DGOperator.implicit_solve``; configurations the
    library does not build (Dirichlet faces, AV, source terms) keep the
    original SuperLU path."""
    L = _Lib(lib_path, device)
    cls = sisdc.dgsem.DGOperator
    orig = cls.implicit_solve

    def implicit_solve(self, coeff, a, rhs, t=0.0):
        if a == 0.0:                        # dgsem.py:505-506: the same rhs object
            return rhs
        rhs_a = np.asarray(rhs)
        if not (self._mass_flat * rhs_a.reshape(-1)).any():   # dgsem.py:509-511
            return np.zeros_like(rhs_a)
        x = L.solve(self, coeff, a, rhs_a, t)
        if x is None:
            return orig(self, coeff, a, rhs, t)
        if isinstance(x, str):
            raise sisdc.dgsem.SolverError("implicit solve did not converge (libsisdc_b200 pinned Krylov solver)")
        return x

    cls.implicit_solve = implicit_solve
    _state["orig"], _state["lib"] = orig, L
    return L


def uninstall(sisdc):
    if "orig" in _state:
        sisdc.dgsem.DGOperator.implicit_solve = _state.pop("orig")
        _state.pop("lib", None)
