// 2-D tensor-product DG-SEM building blocks (sm_100a, fp64).
//
// Uniform periodic Cartesian mesh, GLL collocation: the weak convection and
// the scalar-coefficient SIP operator are sums of the reference's 1-D
// operators (dgsem.py:205-225, 251-309) applied along x-lines and y-lines.
// State layout (ncomp, ney, nex, P+1 [y], P+1 [x]); one thread per node.
#pragma once
#include "sisdc_dev.cuh"

namespace sisdc {

struct Op2DDev {
  int nex, ney, p1, nc;  // ney: element rows this operator (partition) owns
  int nys, row0;         // storage rows and the storage row of owned row 0:
                         // (ney, 0) periodic single domain; (ney + 2, 1) for a
                         // partition whose ghost rows 0 / ney+1 hold the
                         // neighbour partitions' boundary rows (halo exchange)
  long long e0;          // global index of the first owned element (diagnostics)
  long long nn;          // field stride = nodes per field in storage = nys*nex*p1*p1
  long long n;           // nc * nn (one state vector of this partition)
  long long ns;          // node-array stride: u[m] = u + m * ns (n unless partitions are concatenated)
  int problem;
  double dx, dy, sx, sy, mux, muy;
  double gamma, nu, ax, ay;   // NS2D: nu = dynamic viscosity eta
  double pr, nsi;        // NS2D: Prandtl number, max(4/3, gamma / Pr) (SI coefficient bound)
  const double* tab;     // 1-D element tables (TabOff layout)
  const double* nu_art;  // per element, storage rows (nys*nex: ghost rows on a partition), or nullptr
  int fused_sub2;        // partition at P = 3 whose split solve iterates with the fused 2 x 2-tile pass (even nex, even rows on every rank)
};

constexpr int NC_MAX = 4;

// scalars of one partitioned (split) CG solve: every rank computes them from
// the same allreduced sums, so they are bitwise identical across ranks
struct CgPScal {
  double alpha, beta, rgam, ralpha, rho, thr;
  int k, done, ok, zero;
};
constexpr int MAXPART = 16;   // partitions one process can drive (in-process emulation)

// element / node addressing -------------------------------------------------
// ey is always a STORAGE row (owned rows are row0 .. row0+ney-1)
__device__ __forceinline__ long long nidx(const Op2DDev& op, int c, int ey, int ex, int j, int i) {
  return (((long long)c * op.nys + ey) * op.nex + ex) * (op.p1 * op.p1) + j * op.p1 + i;
}
__device__ __forceinline__ int wrapi(int a, int n) {
  a %= n;
  return a < 0 ? a + n : a;
}
// storage row of the y-neighbour (d = +1 above, -1 below) of storage row sy:
// periodic wrap on a single domain, the ghost row on a partition
__device__ __forceinline__ int ynb(const Op2DDev& op, int sy, int d) {
  return op.row0 ? sy + d : wrapi(sy + d, op.ney);
}

// physics (Euler / NS, scalar advection, scalar Burgers along x) -----------
__device__ __forceinline__ bool euler_like(const Op2DDev& op) {
  return op.problem == SISDC_EULER2D || op.problem == SISDC_NS2D;
}
__device__ __forceinline__ void flux2d(const Op2DDev& op, const double* s, int axis, double* f) {
  if (euler_like(op)) {
    const double ir = 1.0 / s[0], vx = s[1] * ir, vy = s[2] * ir;   // one division per state
    const double p = (op.gamma - 1.0) * (s[3] - 0.5 * (s[1] * vx + s[2] * vy));
    const double vn = axis == 0 ? vx : vy;
    f[0] = s[1 + axis];
    f[1] = s[1] * vn + (axis == 0 ? p : 0.0);
    f[2] = s[2] * vn + (axis == 1 ? p : 0.0);
    f[3] = vn * (s[3] + p);
  } else if (op.problem == SISDC_ADVECTION2D) {
    f[0] = (axis == 0 ? op.ax : op.ay) * s[0];
  } else {   // Burgers2D: x-flux only
    f[0] = axis == 0 ? 0.5 * s[0] * s[0] : 0.0;
  }
}
__device__ __forceinline__ double speed2d(const Op2DDev& op, const double* s, int axis) {
  if (euler_like(op)) {
    const double ir = 1.0 / s[0], vx = s[1] * ir, vy = s[2] * ir;
    const double p = (op.gamma - 1.0) * (s[3] - 0.5 * (s[1] * vx + s[2] * vy));
    return fabs(axis == 0 ? vx : vy) + sqrt(op.gamma * p * ir);
  }
  if (op.problem == SISDC_ADVECTION2D) return fabs(axis == 0 ? op.ax : op.ay);
  return axis == 0 ? fabs(s[0]) : 0.0;
}
__device__ __forceinline__ double lam_max2d(const Op2DDev& op, const double* s) {
  if (euler_like(op)) {
    const double ir = 1.0 / s[0], vx = s[1] * ir, vy = s[2] * ir;
    const double p = (op.gamma - 1.0) * (s[3] - 0.5 * (s[1] * vx + s[2] * vy));
    return sqrt(vx * vx + vy * vy) + sqrt(op.gamma * p * ir);
  }
  if (op.problem == SISDC_ADVECTION2D) return hypot(op.ax, op.ay);
  return fabs(s[0]);
}

// coefficient at a node (element eg = ey*nex+ex, in-field node index) --------
// (NS2D: the physical viscous term is the tensor operator of visc2d.cu, not a
// scalar coefficient, so its scalar physical coefficient is zero)
__device__ __forceinline__ bool phys2d(const Op2DDev& op, int eg, double& c) {
  if (op.problem == SISDC_NS2D) {   // the artificial viscosity (if any) is the only scalar-coefficient part
    c = op.nu_art ? op.nu_art[eg] : 0.0;
    return op.nu_art != nullptr;
  }
  if (op.nu_art) {
    c = (op.nu > 0.0 ? op.nu : 0.0) + op.nu_art[eg];
    return true;
  }
  c = op.nu;
  return op.nu > 0.0;
}
__device__ __forceinline__ double coef2d(const Op2DDev& op, const CoefDev& k, int ey, int ex, int j, int i) {
  const int eg = ey * op.nex + ex;
  switch (k.kind) {
    case SISDC_COEF_CONST: return k.value;
    case SISDC_COEF_FIELD: return k.ptr[(long long)eg * op.p1 * op.p1 + j * op.p1 + i];
    case SISDC_COEF_SI: {
      double s[NC_MAX];
#pragma unroll
      for (int c = 0; c < NC_MAX; ++c) s[c] = c < op.nc ? k.ptr[nidx(op, c, ey, ex, j, i)] : 1.0;
      const double lam = lam_max2d(op, s);
      const double half = 0.5 * k.value * (lam * lam);
      if (op.problem == SISDC_NS2D)   // oracle NS2D.nu_si (+ the frozen artificial viscosity, as dgsem.py:356-396)
        return half + (op.nu / s[0]) * op.nsi + (op.nu_art ? op.nu_art[eg] : 0.0);
      double ph;
      return phys2d(op, eg, ph) ? half + ph : half;
    }
    case SISDC_COEF_PHYS: {
      double ph;
      return phys2d(op, eg, ph) ? ph : 0.0;
    }
    default: return 0.0;
  }
}

// tensor-product transfer tables (same table layout as XferDev)
struct Xfer2Dev {
  int nslab, pc, pf, Mc, Mf;
  const double* tab;   // It (Mf*Mc) | Pt (Mc*Mf) | Isp (pf*pc) | Psp (pc*pf)
};

// ---------------------------------------------------------------- Rusanov
__device__ __forceinline__ void rusanov2d(const Op2DDev& op, const double* um, const double* up, int axis,
                                          double* fh) {
  double fm[NC_MAX], fp[NC_MAX];
  flux2d(op, um, axis, fm);
  flux2d(op, up, axis, fp);
  const double lam = fmax(speed2d(op, um, axis), speed2d(op, up, axis));
#pragma unroll
  for (int c = 0; c < NC_MAX; ++c)
    if (c < op.nc) fh[c] = 0.5 * (fm[c] + fp[c]) - 0.5 * lam * (up[c] - um[c]);
}

// ------------------------------------------------- NS2D viscous physics
// (shared by the line-formulated k2_visc of visc2d.cu and the warp-per-element
// tensor-core kernel k2_visc8 of ops2d.cu)
constexpr int NCV = 4;   // (rho, rho u, rho v, rho E)
struct Prim {
  double rho, vx, vy, Es, nu;
};
__device__ __forceinline__ Prim prim(const Op2DDev& op, const double* s) {
  const double rho = s[0], ir = 1.0 / rho;   // one division per state (the oracle divides four times: <= 1 ulp apart)
  return Prim{rho, s[1] * ir, s[2] * ir, s[3] * ir, op.nu * ir};
}

// viscous flux at a node from the state and its gradients (oracle NS2D.visc_flux)
__device__ __forceinline__ void visc_flux(const Op2DDev& op, double gpr, const double* s, const double* gx,
                                          const double* gy, double* Fx, double* Fy) {
  const Prim q = prim(op, s);
  const double k = q.nu * gpr;   // gpr = gamma / Pr
  const double dxm = gx[1] - q.vx * gx[0], dym = gy[1] - q.vx * gy[0];
  const double dxn = gx[2] - q.vy * gx[0], dyn = gy[2] - q.vy * gy[0];
  const double txx = q.nu * ((4.0 / 3.0) * dxm - (2.0 / 3.0) * dyn);
  const double tyy = q.nu * ((4.0 / 3.0) * dyn - (2.0 / 3.0) * dxm);
  const double txy = q.nu * (dym + dxn);
  const double ex = gx[3] - q.Es * gx[0] - q.vx * dxm - q.vy * dxn;
  const double ey = gy[3] - q.Es * gy[0] - q.vx * dym - q.vy * dyn;
  Fx[0] = 0.0; Fx[1] = txx; Fx[2] = txy; Fx[3] = q.vx * txx + q.vy * txy + k * ex;
  Fy[0] = 0.0; Fy[1] = txy; Fy[2] = tyy; Fy[3] = q.vx * txy + q.vy * tyy + k * ey;
}

// G_nn(s) v (oracle NS2D.apply_gnn); axis 0: x-faces, 1: y-faces
__device__ __forceinline__ void apply_gnn(const Op2DDev& op, double gpr, const double* s, const double* v, int axis,
                                          double* r) {
  const Prim q = prim(op, s);
  const double k = q.nu * gpr;   // gpr = gamma / Pr
  const double a = v[1] - q.vx * v[0], b = v[2] - q.vy * v[0];
  const double r1 = q.nu * (axis == 0 ? (4.0 / 3.0) * a : a);
  const double r2 = q.nu * (axis == 0 ? b : (4.0 / 3.0) * b);
  r[0] = 0.0;
  r[1] = r1;
  r[2] = r2;
  r[3] = q.vx * r1 + q.vy * r2 + k * (v[3] - q.Es * v[0] - q.vx * a - q.vy * b);
}

}  // namespace sisdc
