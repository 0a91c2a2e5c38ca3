"""BASELINE.json workloads: seeded synthetic initial data and pinned schedules.

These are *inputs*, shared by the CUDA path, the tests and the CPU oracle.
The generators and the open parameters BASELINE.json leaves (seeds, dt for
config 2, the MLSDC schedule) are pinned here and recorded in DESIGN.md:

* schedule: SI(2), incremental, Radau-right, FMG start (== cascade for two
  levels), N_c = 2, N_s = 1, 5 V-cycles + closing fine sweep -- the
  reference CLI defaults (``cli.py:273-295``).  6 fine sweeps per step.
* cfg1: conv-diff, 64 el, P 8/4, M 4/2, a=1, nu=1e-2, CFL 1 on |a|.
* cfg2: Burgers, 512 el, P 8/4, M 5/3, nu=5e-3, CFL 1 on max|u0|, run to
  t = 1.5 with the reference's step rule n = ceil(t_end/dt0), dt = t_end/n
  (``cli.py:825-836``), **3 V-cycles** + closing sweep (4 fine sweeps per
  step).  With the CLI default of 5 (or 4) cycles the reference itself
  diverges on this hierarchy after 8 (12) steps at any CFL: an interface-jump
  mode at max|u| is amplified by ~1.75 per V-cycle ("cfg2
  schedule").  2 and 3 cycles run stably to t = 1.5 and agree to 4e-13; the
  paper's own Burgers runs converge in 1 cycle + closing sweep at CFL <= 4
  (PAPER.md:1257-1269).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class Workload1D:
    name: str
    problem: str          # "convdiff" | "burgers"
    n_elem: int
    p_fine: int
    p_coarse: int
    m_fine: int
    m_coarse: int
    params: dict
    seed: int
    cfl: float = 1.0
    t_end: float = None
    n_steps: int = None
    n_cycles: int = 5
    x_left: float = 0.0
    x_right: float = TWO_PI

    @property
    def dx(self):
        return (self.x_right - self.x_left) / self.n_elem

    def nodes_x(self, degree, gll_nodes):
        e = self.x_left + self.dx * np.arange(self.n_elem)
        return e[:, None] + 0.5 * self.dx * (np.asarray(gll_nodes) + 1.0)[None, :]

    def initial_state(self, gll_nodes):
        """Seeded IC on the fine GLL nodes, flat (1, ne, P+1)."""
        x = self.nodes_x(self.p_fine, gll_nodes)
        rng = np.random.default_rng(self.seed)
        if self.problem == "convdiff":
            ks = np.sort(rng.choice(np.arange(2, 9), 4, replace=False))
            amps = rng.normal(0.0, 0.1, 4)
            u = np.sin(x) + sum(a * np.sin(k * x) for k, a in zip(ks, amps))
        elif self.problem == "burgers":
            amps = rng.normal(0.0, 0.01, 15)
            u = 1.0 + 0.5 * np.sin(x) + sum(a * np.sin(k * x) for k, a in zip(range(2, 17), amps))
        else:
            raise ValueError(self.problem)
        return np.ascontiguousarray(u.reshape(-1), dtype=np.float64)

    def time_step(self, u0, delta_p):
        """(dt, n_steps) -- ``cli.py:825-836`` semantics with CFL on the
        convective wave speed; delta_p = compute_delta(p_fine)."""
        lam = abs(self.params["speed"]) if self.problem == "convdiff" else float(np.max(np.abs(u0)))
        dt0 = self.cfl * self.dx / (2.0 * delta_p * lam)
        if self.n_steps is not None:
            return dt0, self.n_steps
        n = max(1, math.ceil(self.t_end / dt0 - 1e-12))
        return self.t_end / n, n

    def dof(self):
        return self.n_elem * (self.p_fine + 1), self.n_elem * (self.p_coarse + 1)

    def dof_sweeps_per_step(self):
        """U = sum_l N_l M_l passes_l: 6 fine sweeps, 12 coarse
        passes (1 predictor + 1 FMG sweep + 2 per cycle)."""
        nf, nc = self.dof()
        fine_passes = self.n_cycles + 1
        coarse_passes = 2 + 2 * self.n_cycles
        return nf * self.m_fine * fine_passes + nc * self.m_coarse * coarse_passes, \
            nf * self.m_fine * fine_passes


CFG1 = Workload1D("cfg1_convdiff_64el_P8", "convdiff", 64, 8, 4, 4, 2,
                  {"speed": 1.0, "nu": 1e-2}, seed=1, n_steps=100)
CFG2 = Workload1D("cfg2_burgers_512el_P8", "burgers", 512, 8, 4, 5, 3,
                  {"nu": 5e-3}, seed=2, t_end=1.5, n_cycles=3)

WORKLOADS = {"cfg1": CFG1, "cfg2": CFG2}


# ---------------------------------------------------------------- 2-D (cfgs 3-5)
@dataclass(frozen=True)
class Workload2D:
    """2-D compressible Euler / NS workloads (BASELINE configs 3-5; no
    reference implementation).  Seeded synthetic ICs:
    isentropic vortex (cfg3) and the double shear layer (cfgs 4-5)."""
    name: str
    kind: str            # "vortex" | "shear"
    nex: int
    ney: int
    p_fine: int
    p_coarse: int
    m_fine: int
    m_coarse: int
    length: float
    seed: int
    gamma: float = 1.4
    eta: float = 0.0          # dynamic viscosity (rho = 1: 1/Re); 0 -> Euler
    prandtl: float = 0.72
    mach: float = 0.1
    cfl: float = 1.0
    n_cycles: int = 3
    n_steps: int = 20
    length_y: float = None   # None: square domain; set for one rank's share of a mesh (tools/scaling_estimate.py)

    @property
    def ncomp(self):
        return 4

    def gpu_problem(self):
        """CompressibleNS2D (Stokes stress + Fourier heat flux, eta, Pr) for the
        viscous configs, CompressibleEuler2D for cfg3."""
        from . import dgsem2d
        if self.eta > 0:
            return dgsem2d.CompressibleNS2D(self.gamma, self.eta, self.prandtl)
        return dgsem2d.CompressibleEuler2D(self.gamma, 0.0)

    @property
    def ly(self):
        return self.length if self.length_y is None else self.length_y

    def dof(self):
        nf = 4 * self.nex * self.ney * (self.p_fine + 1) ** 2
        nc = 4 * self.nex * self.ney * (self.p_coarse + 1) ** 2
        return nf, nc

    def dof_sweeps_per_step(self):
        nf, nc = self.dof()
        return nf * self.m_fine * (self.n_cycles + 1) + nc * self.m_coarse * (2 + 2 * self.n_cycles), \
            nf * self.m_fine * (self.n_cycles + 1)

    def initial_state(self, X, Y):
        """Conservative (rho, rho u, rho v, rho E) on node arrays X, Y (ney, nex, p1, p1)."""
        g = self.gamma
        rng = np.random.default_rng(self.seed)
        if self.kind == "vortex":
            x0, y0 = rng.uniform(0.25 * self.length, 0.75 * self.length, 2)
            beta = 5.0
            r2 = (X - x0) ** 2 + (Y - y0) ** 2
            e = np.exp(0.5 * (1.0 - r2))
            u = 1.0 - beta / (2.0 * math.pi) * (Y - y0) * e
            v = 1.0 + beta / (2.0 * math.pi) * (X - x0) * e
            T = 1.0 - (g - 1.0) * beta ** 2 / (8.0 * g * math.pi ** 2) * np.exp(1.0 - r2)
            rho = T ** (1.0 / (g - 1.0))
            p = rho ** g
        else:
            delta = 0.05
            u = np.where(Y <= math.pi, np.tanh((Y - math.pi / 2) / delta), np.tanh((3 * math.pi / 2 - Y) / delta))
            v = 0.05 * np.sin(X) + 1e-3 * rng.standard_normal(X.shape)
            rho = np.ones_like(X)
            p = np.full_like(X, 1.0 / (g * self.mach ** 2))
        E = p / (g - 1.0) + 0.5 * rho * (u * u + v * v)
        return np.ascontiguousarray(np.stack([rho, rho * u, rho * v, E]).reshape(-1), dtype=np.float64)

    def time_step(self, u0, delta_p):
        """dt from the acoustic CFL on max(|v| + c) (builder choice)."""
        q = u0.reshape(4, -1)
        rho, mx, my, E = q
        p = (self.gamma - 1.0) * (E - 0.5 * (mx * mx + my * my) / rho)
        lam = float(np.max(np.sqrt(mx * mx + my * my) / rho + np.sqrt(self.gamma * p / rho)))
        h = self.length / self.nex
        return self.cfl * h / (2.0 * delta_p * lam)


CFG3 = Workload2D("cfg3_euler_vortex_128x128_P7", "vortex", 128, 128, 7, 3, 4, 2, 10.0, seed=3)
CFG4 = Workload2D("cfg4_ns_shear_256x256_P7", "shear", 256, 256, 7, 3, 5, 3, TWO_PI, seed=4, eta=1e-4)
CFG5 = Workload2D("cfg5_ns_shear_1024x1024_P7", "shear", 1024, 1024, 7, 3, 5, 3, TWO_PI, seed=5, eta=1e-4)
WORKLOADS.update({"cfg3": CFG3, "cfg4": CFG4, "cfg5": CFG5})


# ------------------------------------------------ Dirichlet front
def burgers_front_exact(nu):
    """u = 1 - tanh((x + 1/2 - t) / (2 nu)) (``problems.py:268-277``)."""
    def exact(x, t=0.0):
        return 1.0 - np.tanh((np.asarray(x) + 0.5 - t) / (2.0 * nu))
    return exact


def burgers_front_boundary(nu):
    """Trace data of the exact front at x = -1, 1 (``problems.py:280-291``)."""
    ex = burgers_front_exact(nu)
    return lambda t: (np.array([ex(-1.0, t)]), np.array([ex(1.0, t)]))


@dataclass(frozen=True)
class FrontWorkload:
    """The paper's Burgers moving front on [-1, 1] with time-dependent
    Dirichlet data (PAPER.md "Burgers moving front"); the parity workload of
    the Dirichlet faces (oracle/make_golden.py ``DIRICHLET`` / ``AV_CASE``)."""
    nu: float = 1e-2
    n_elem: int = 20
    p_fine: int = 8
    p_coarse: int = 4
    m_fine: int = 5
    m_coarse: int = 3
    cfl: float = 1.0
    n_cycles: int = 3
    av: tuple = None          # (kappa_s, c_s) or None


FRONT = FrontWorkload()
FRONT_AV = FrontWorkload(n_elem=16, p_fine=4, p_coarse=2, av=(0.5, 0.5))


# ------------------------------------------------- 1-D compressible flow (CNS)
@dataclass(frozen=True)
class AcousticWorkload:
    """1-D CompressibleFlow on the reference's right-running acoustic wave
    (``problems.py:294-316`` restated; CLI defaults ``cli.py:400-409``:
    gamma 1.4, R 287.28, Mach 0.1, p_inf 1000, T_inf 300, amp 1e-2) on a
    periodic [0, 1] mesh.  The single-level cases are the reference's own
    ``test_dgsem.py:553-600`` set-ups (eta 1e-5, 12 elements, P = 7)."""
    name: str
    n_elem: int = 12
    p_fine: int = 7
    p_coarse: int = 3
    m_fine: int = 5
    m_coarse: int = 3
    scheme: str = "si2"
    cfl: float = 0.8
    n_steps: int = 2
    n_sweeps: int = 4
    mlsdc: bool = False
    n_cycles: int = 3
    gamma: float = 1.4
    R_gas: float = 287.28
    eta: float = 1e-5
    prandtl: float = 0.75
    mach: float = 0.1
    p_inf: float = 1000.0
    T_inf: float = 300.0
    amp_frac: float = 1e-2
    x_left: float = 0.0
    x_right: float = 1.0

    @property
    def dx(self):
        return (self.x_right - self.x_left) / self.n_elem

    def initial_state(self, gll_nodes):
        """Conservative (rho, rho v, rho E), flat (3, ne, P+1), on the fine nodes."""
        e = self.x_left + self.dx * np.arange(self.n_elem)
        x = e[:, None] + 0.5 * self.dx * (np.asarray(gll_nodes) + 1.0)[None, :]
        g, R = self.gamma, self.R_gas
        a_inf = math.sqrt(g * R * self.T_inf)
        vp = self.amp_frac * a_inf * np.sin(2.0 * math.pi * x)
        T = (a_inf + 0.5 * (g - 1.0) * vp) ** 2 / (g * R)
        p = self.p_inf * (T / self.T_inf) ** (g / (g - 1.0))
        v = self.mach * a_inf + vp
        rho = p / (R * T)
        ener = p / (g - 1.0) + 0.5 * rho * v * v
        return np.ascontiguousarray(np.stack([rho, rho * v, ener]).reshape(-1), dtype=np.float64)

    def time_step(self, u0, delta_p):
        """dt_from_cfl(cfl, dx, max(|v| + c), P_fine) (dgsem.py:67-69)."""
        u3 = np.asarray(u0).reshape(3, self.n_elem, -1)
        rho, v = u3[0], u3[1] / u3[0]
        p = (self.gamma - 1.0) * (u3[2] - 0.5 * u3[1] * v)
        lam = float(np.max(np.abs(v) + np.sqrt(self.gamma * p / rho)))
        return self.cfl * self.dx / (2.0 * delta_p * lam)


CNS_CASES = (
    AcousticWorkload("cns_resolved", m_fine=3, scheme="si1", cfl=0.8),      # test_dgsem.py:575-600
    AcousticWorkload("cns_large", m_fine=5, scheme="si2", cfl=256.0, n_steps=1),  # test_dgsem.py:553-573
    AcousticWorkload("cns_mlsdc", m_fine=5, m_coarse=3, scheme="si2", cfl=0.8, mlsdc=True, n_cycles=2),
    AcousticWorkload("cns_mlsdc_visc", n_elem=16, p_fine=6, p_coarse=3, m_fine=4, m_coarse=2, scheme="si2",
                     cfl=1.0, eta=2e-4, mlsdc=True, n_steps=1),
)


# --------------------------------------- Burgers with a manufactured source term
@dataclass(frozen=True)
class ManufacturedWorkload:
    """Burgers with the source that makes u*(x, t) = 2 + a sin(k x + w t) an
    exact solution (the reference's ``manufactured_burgers_source``,
    ``problems.py:85-92``: src = u_t + u u_x - nu u_xx), Dirichlet trace data
    from u* on [-1, 1]: the parity workload of the host-evaluated source term
    (``dgsem.py:328-347``)."""
    nu: float = 0.05
    amp: float = 0.5
    k: float = math.pi
    w: float = 1.0
    n_elem: int = 12
    p_fine: int = 6
    p_coarse: int = 3
    m_fine: int = 4
    m_coarse: int = 2
    cfl: float = 1.0
    n_cycles: int = 2

    def exact(self, x, t=0.0):
        return 2.0 + self.amp * np.sin(self.k * np.asarray(x) + self.w * t)

    def source(self, x, t, u=None):
        ph = self.k * np.asarray(x) + self.w * t
        u_ = 2.0 + self.amp * np.sin(ph)
        ut = self.amp * self.w * np.cos(ph)
        ux = self.amp * self.k * np.cos(ph)
        uxx = -self.amp * self.k * self.k * np.sin(ph)
        return ut + u_ * ux - self.nu * uxx

    def boundary(self, t):
        return np.array([self.exact(-1.0, t)]), np.array([self.exact(1.0, t)])


MANUFACTURED = ManufacturedWorkload()


@dataclass(frozen=True)
class SodWorkload:
    """1-D CompressibleFlow on the reference CLI's Sod shock tube
    (``cli.py:766-772``, ``problems.sod_init`` ``problems.py:319-331``):
    (rho, v, p) = (1, 0, 1) left of the split, (0.125, 0, 0.1) right of it,
    Dirichlet faces holding the two end states, Persson-Peraire viscosity."""
    name: str
    n_elem: int = 20
    p_fine: int = 4
    p_coarse: int = 2
    m_fine: int = 3
    m_coarse: int = 2
    cfl: float = 0.5
    n_cycles: int = 2
    n_steps: int = 2
    eta: float = 0.0
    av: tuple = (0.5, 0.5)
    gamma: float = 1.4
    R_gas: float = 287.28
    prandtl: float = 0.75
    split: float = 0.5

    def states(self):
        g = self.gamma
        left = np.array([1.0, 0.0, 1.0 / (g - 1.0)])
        right = np.array([0.125, 0.0, 0.1 / (g - 1.0)])
        return left, right

    def initial(self, x):
        """Conservative (3, ...) field of the shock-tube data at x."""
        x = np.asarray(x, dtype=float)
        left, right = self.states()
        lt = x < self.split
        return np.stack([np.where(lt, left[c], right[c]) for c in range(3)])

    def boundary(self, t):
        return self.states()


SOD_CASES = (
    SodWorkload("sod_euler_av"),
    SodWorkload("sod_ns_av", n_elem=16, p_fine=5, p_coarse=3, eta=1e-3, av=(1.0, 1.0), cfl=0.4),
)
