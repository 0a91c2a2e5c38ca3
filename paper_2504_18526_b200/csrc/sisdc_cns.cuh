// Pointwise physics of the 1-D compressible-flow problem (SISDC_CNS1D),
// restating CompressibleFlow (problems.py:160-240): conservative
// (rho, rho v, rho E), ideal gas, Stokes viscosity (4/3 factor), Prandtl
// heat flux.  Shared by cns1d.cu and the Persson sensor in ops1d.cu.
#pragma once
#include "sisdc_dev.cuh"

namespace sisdc {

// _primitive (problems.py:98-102)
__device__ __forceinline__ void cns_prim(const Op1DDev& op, double u0, double u1, double u2, double& rho,
                                         double& v, double& p) {
  rho = u0;
  v = u1 / rho;
  p = (op.gamma - 1.0) * (u2 - 0.5 * u1 * v);
}
// flux (problems.py:190-192)
__device__ __forceinline__ void cns_flux(const Op1DDev& op, const double* u, double* f) {
  double rho, v, p;
  cns_prim(op, u[0], u[1], u[2], rho, v, p);
  f[0] = u[1];
  f[1] = u[1] * v + p;
  f[2] = v * (u[2] + p);
}
// max_speed (problems.py:194-196)
__device__ __forceinline__ double cns_speed(const Op1DDev& op, double u0, double u1, double u2) {
  double rho, v, p;
  cns_prim(op, u0, u1, u2, rho, v, p);
  return fabs(v) + sqrt(op.gamma * p / rho);
}
// conv_jacobian (problems.py:204-219), row-major 3x3
__device__ __forceinline__ void cns_jac(const Op1DDev& op, const double* u, double* A) {
  const double g = op.gamma;
  double rho, v, p;
  cns_prim(op, u[0], u[1], u[2], rho, v, p);
  const double H = (u[2] + p) / rho;
  A[0] = 0.0; A[1] = 1.0; A[2] = 0.0;
  A[3] = 0.5 * (g - 3.0) * v * v; A[4] = (3.0 - g) * v; A[5] = g - 1.0;
  A[6] = (0.5 * (g - 1.0) * v * v - H) * v; A[7] = H - (g - 1.0) * v * v; A[8] = g * v;
}
// diffusion_coeff (problems.py:221-237); false when eta == 0 (Euler: None)
__device__ __forceinline__ bool cns_dcoef(const Op1DDev& op, const double* u, double* A) {
  if (!(op.eta > 0.0)) return false;
  const double g = op.gamma;
  double rho, v, p;
  cns_prim(op, u[0], u[1], u[2], rho, v, p);
  const double E = u[2] / rho;
  const double nu = op.eta / rho;
  const double gk = g * nu / op.Pr;
  const double mu = (4.0 / 3.0) * nu;
  A[0] = 0.0; A[1] = 0.0; A[2] = 0.0;
  A[3] = -mu * v; A[4] = mu; A[5] = 0.0;
  A[6] = -(mu - gk) * v * v - gk * E; A[7] = (mu - gk) * v; A[8] = gk;
  return true;
}
// physical coefficient (dgsem.py:313-326): A_d(u) + nu_art I (scalar nu_art
// field alone when A_d is None); false for None
__device__ __forceinline__ bool cns_phys(const Op1DDev& op, const double* u, int e, double* C) {
  bool has = cns_dcoef(op, u, C);
  if (op.nu_art) {
    if (!has)
      for (int j = 0; j < 9; ++j) C[j] = 0.0;
    const double eps = op.nu_art[e];
    C[0] += eps; C[4] += eps; C[8] += eps;
    has = true;
  }
  return has;
}

}  // namespace sisdc
