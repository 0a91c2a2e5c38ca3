"""Problem descriptors (``problems.py:25-82,160-240`` of the reference).

The pointwise physics -- flux, wave speed, convective Jacobian A_c and
diffusion coefficient A_d -- is evaluated inside the sm_100a kernels
(``csrc/sisdc_dev.cuh``); these objects carry the parameters and the
attributes the sweeper and the operator read (``ncomp``, ``is_linear``,
``source``, ``boundary_state``).
"""
from __future__ import annotations


class ConvectionDiffusion:
    """u_t + v u_x = nu u_xx, constant coefficients (``problems.py:25-52``)."""

    ncomp = 1
    is_linear = True
    source = None
    kind = "convdiff"

    def __init__(self, speed: float = 1.0, nu: float = 0.0, boundary=None):
        if nu < 0:
            raise ValueError("diffusion coefficient must be nonnegative")
        self.speed = float(speed)
        self.nu = float(nu)
        self.boundary_state = boundary

    def conv_jacobian_const(self):
        return self.speed


class Burgers:
    """u_t + (u^2/2)_x = nu u_xx (``problems.py:55-82``).  ``source`` is the
    reference's host callable src(x, t, u); ``source_depends_on_state=False``
    declares a known forcing src(x, t) (manufactured solutions): its node values
    are then tabulated per time on the device and the state never leaves the GPU."""

    ncomp = 1
    is_linear = False
    kind = "burgers"

    def __init__(self, nu: float = 0.0, source=None, boundary=None, source_depends_on_state: bool = True):
        if nu < 0:
            raise ValueError("diffusion coefficient must be nonnegative")
        self.nu = float(nu)
        self.source = source
        self.source_depends_on_state = bool(source_depends_on_state)
        self.boundary_state = boundary
        self.speed = 0.0


class CompressibleFlow:
    """1-D compressible Navier-Stokes in conservative variables (rho, rho v,
    rho E) (``problems.py:160-240``); eta = 0 is Euler.  Built on periodic
    meshes; the SI coefficient (dt_m/2) A_c(u_b)^2 + A_d(u_b) (+nu_art) is a
    3x3 matrix per node, so the implicit solve is the pinned block-Jacobi
    BiCGStab (``oracle/cg.py``) instead of the CG."""

    ncomp = 3
    is_linear = False
    source = None
    kind = "cns"
    speed = 0.0
    nu = 0.0

    def __init__(self, gamma: float = 1.4, R_gas: float = 287.28, eta: float = 0.0, Pr: float = 0.75,
                 boundary=None):
        if gamma <= 1.0:
            raise ValueError("gamma must exceed 1")
        if Pr <= 0:
            raise ValueError("Prandtl number must be positive")
        if eta < 0:
            raise ValueError("viscosity must be nonnegative")
        self.gamma = float(gamma)
        self.R_gas = float(R_gas)
        self.eta = float(eta)
        self.Pr = float(Pr)
        self.boundary_state = boundary

    @property
    def viscous(self) -> bool:
        return self.eta > 0


def burgers_front_exact(nu: float):
    """Viscous front u = 1 - tanh((x + 1/2 - t) / (2 nu)) (``problems.py:268-277``)."""
    import numpy as np
    nu = float(nu)

    def exact(x, t=0.0):
        return 1.0 - np.tanh((np.asarray(x) + 0.5 - t) / (2.0 * nu))

    return exact


def burgers_front_problem(nu: float):
    """Burgers with the exact front's trace data on [-1, 1] (``problems.py:280-291``):
    returns (problem, exact)."""
    import numpy as np
    exact = burgers_front_exact(nu)

    def boundary(t):
        return np.array([exact(-1.0, t)]), np.array([exact(1.0, t)])

    return Burgers(nu, boundary=boundary), exact


def wave_packet_exact(nu, speed: float = 1.0, wave_numbers=None, amplitudes=None, shifts=None):
    """Decaying multi-mode packet, exact for constant-coefficient
    convection-diffusion on a periodic unit interval (``problems.py:247-270``;
    the reference's default modes).  exact(x, t) = sum_j a_j exp(-k_j^2 nu t)
    sin(k_j (x - s_j - v t))."""
    import numpy as np
    kap = np.asarray(2.0 * np.pi * np.array([1.0, 3.0, 5.0, 7.0, 9.0, 12.0, 15.0])
                     if wave_numbers is None else wave_numbers, dtype=float)
    amp = np.asarray(np.array([1.00, 1.50, 1.80, 1.70, 1.50, 1.30, 1.15])
                     if amplitudes is None else amplitudes, dtype=float)
    sft = np.asarray(np.array([0.00, 0.05, 0.10, 0.15, 0.20, 0.30, 0.18]) if shifts is None else shifts,
                     dtype=float)
    nu, speed = float(nu), float(speed)

    def exact(x, t=0.0):
        x = np.asarray(x)
        phase = kap.reshape((-1,) + (1,) * x.ndim) * (x[None] - sft.reshape((-1,) + (1,) * x.ndim) - speed * t)
        decay = np.exp(-(kap ** 2) * nu * t)
        return np.tensordot(amp * decay, np.sin(phase), axes=(0, 0))

    return exact
