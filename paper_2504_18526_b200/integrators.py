"""The operator interface the sweeps are written against (``integrators.py:29-60``)."""
from __future__ import annotations

from typing import Any, Literal, Protocol

Scheme = Literal["euler", "si1", "si2"]


class OperatorContext(Protocol):
    """What a spatial discretisation provides to the time integrators.

    States are flat device vectors (torch float64 CUDA tensors); the
    coefficient returned by ``modified_diffusion_matrix`` is opaque and only
    passed back into ``apply_diffusion`` and ``implicit_solve``.
    """

    def eval_rhs(self, u, t: float): ...

    def apply_convection(self, u, t: float = 0.0): ...

    def modified_diffusion_matrix(self, u, dt_m: float, scheme: Scheme) -> Any: ...

    def apply_diffusion(self, coeff: Any, u, t: float = 0.0): ...

    def implicit_solve(self, coeff: Any, a: float, rhs, t: float = 0.0): ...

    def apply_source(self, u, t: float): ...
