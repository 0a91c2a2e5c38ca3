// Device-side building blocks of the 1-D DG-SEM sweep path (sm_100a, fp64).
//
// Layout: flat (n_elem, P+1) float64, element-major (dgsem.py:12-13).  Every
// element kernel stages a tile of EB elements plus one periodic halo element
// on each side in shared memory; face terms read the halo.  The per-node
// arithmetic restates the reference operators:
//   convection   dgsem.py:205-225  (weak volume term + Rusanov face flux)
//   SIP diffusion dgsem.py:251-309 (avg flux, penalty mu0{C}[u], adjoint lift)
//   coefficients  dgsem.py:313-326, 356-396
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/sisdc_b200.h"

namespace sisdc {

constexpr int MAXP1 = 16;   // P <= 15
constexpr int MAXM = 16;    // collocation nodes per level

// element tables, one contiguous device block per operator
//   D[p1*p1] | DTW[p1*p1] (DTW[i][k] = D[k][i] w[k]) | w | m | minv | D2W[p1*p1] (D[k][i]^2 w[k]) | Vinv[p1*p1]
struct TabOff {
  __host__ __device__ static int D(int) { return 0; }
  __host__ __device__ static int DTW(int p1) { return p1 * p1; }
  __host__ __device__ static int w(int p1) { return 2 * p1 * p1; }
  __host__ __device__ static int m(int p1) { return 2 * p1 * p1 + p1; }
  __host__ __device__ static int minv(int p1) { return 2 * p1 * p1 + 2 * p1; }
  __host__ __device__ static int D2W(int p1) { return 2 * p1 * p1 + 3 * p1; }
  __host__ __device__ static int Vinv(int p1) { return 3 * p1 * p1 + 3 * p1; }
  __host__ __device__ static int size(int p1) { return 4 * p1 * p1 + 3 * p1; }
};

struct Op1DDev {
  int ne, p1, n, problem;
  double dx, s, mu0, speed, nu;
  const double* tab;      // device tables (TabOff layout)
  const double* nu_art;   // per element or nullptr
  int bc;                 // SISDC_PERIODIC / SISDC_DIRICHLET (Mesh1D.bc)
  double gl, gr;          // Dirichlet: outside states at the time of this evaluation
  int nc;                 // components (1; 3 for SISDC_CNS1D, n counts one component)
  double gamma, eta, Pr;  // SISDC_CNS1D gas (problems.py:171-187)
  double gl3[3], gr3[3];  // SISDC_CNS1D Dirichlet: outside states (all components)
};

struct CoefDev {
  int kind;
  double value;
  const double* ptr;
};

// ------------------------------------------------------------ physics
__device__ __forceinline__ double flux(const Op1DDev& op, double u) {
  return op.problem == SISDC_BURGERS ? 0.5 * u * u : op.speed * u;   // problems.py:39-40,68-69
}
__device__ __forceinline__ double wave_speed(const Op1DDev& op, double u) {
  return op.problem == SISDC_BURGERS ? fabs(u) : fabs(op.speed);    // problems.py:42-43,71-72
}
// physical coefficient A_d (+ nu_art), dgsem.py:313-326; returns false for "None"
__device__ __forceinline__ bool phys_coef(const Op1DDev& op, int e, double& c) {
  if (op.nu_art) {
    c = (op.nu > 0.0 ? op.nu : 0.0) + op.nu_art[e];
    return true;
  }
  c = op.nu;
  return op.nu > 0.0;
}
// coefficient value at element e, node i
__device__ __forceinline__ double coef_at(const Op1DDev& op, const CoefDev& k, int e, int i) {
  switch (k.kind) {
    case SISDC_COEF_CONST: return k.value;
    case SISDC_COEF_FIELD: return k.ptr[e * op.p1 + i];
    case SISDC_COEF_SI: {
      // (dt_m/2) A_c(u_b)^2 + A_d (+ nu_art): dgsem.py:382-387
      double j = op.problem == SISDC_BURGERS ? k.ptr[e * op.p1 + i] : op.speed;
      double half = 0.5 * k.value * (j * j);
      double ph;
      return phys_coef(op, e, ph) ? half + ph : half;
    }
    case SISDC_COEF_PHYS: {
      double ph;
      return phys_coef(op, e, ph) ? ph : 0.0;
    }
    default: return 0.0;
  }
}

// ----------------------------------------------------------- tiles
// periodic element index; tiles may be wider than the whole mesh, so fold fully
__device__ __forceinline__ int wrap(int e, int ne) {
  e %= ne;
  return e < 0 ? e + ne : e;
}

// tile[(el+1)*p1 + i] = u[(ebase+el) wrapped, i] for el = -1..EB.  Dirichlet:
// the ghost elements outside the mesh hold the outside state g_l / g_r
// (only their face node enters: dgsem.py:179-194, 212-216, 282-284)
template <bool DIR>
__device__ __forceinline__ void load_tile(const Op1DDev& op, double* tile, const double* __restrict__ u, int ebase,
                                          int EB) {
  const int p1 = op.p1, ne = op.ne;
  int tot = (EB + 2) * p1;
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    int el = t / p1 - 1, i = t - (t / p1) * p1;
    const int eg = ebase + el;
    if (DIR && (eg < 0 || eg >= ne)) tile[t] = eg < 0 ? op.gl : op.gr;
    else tile[t] = u[wrap(eg, ne) * p1 + i];
  }
}
__device__ __forceinline__ void load_tab(double* stab, const double* __restrict__ tab, int p1) {
  int sz = TabOff::size(p1);
  for (int t = threadIdx.x; t < sz; t += blockDim.x) stab[t] = tab[t];
}

// Rusanov flux at a face from minus/plus traces: dgsem.py:217-220
__device__ __forceinline__ double rusanov(const Op1DDev& op, double um, double up) {
  double lam = fmax(wave_speed(op, um), wave_speed(op, up));
  return 0.5 * (flux(op, um) + flux(op, up)) - 0.5 * lam * (up - um);
}

// convection at node (el,i) of a tile (tile index el+1 holds element el)
__device__ __forceinline__ double conv_node(const Op1DDev& op, const double* st, const double* ut, int el,
                                            int i) {
  const int p1 = op.p1;
  const double* DTW = st + TabOff::DTW(p1);
  const double* ue = ut + (el + 1) * p1;
  double v = 0.0;
#pragma unroll 4
  for (int k = 0; k < p1; ++k) v = fma(DTW[i * p1 + k], flux(op, ue[k]), v);
  if (i == p1 - 1) v -= rusanov(op, ue[p1 - 1], ue[p1]);          // face e+1/2, dgsem.py:221
  if (i == 0) v += rusanov(op, ue[-1], ue[0]);                    // face e-1/2, dgsem.py:222
  return v * st[TabOff::minv(p1) + i];
}

// q = C * (2/dx) D u for every node of the tile (incl. halo elements); C tile must be filled.
// Dirichlet ghosts carry the interior boundary node's q (one-sided flux, dgsem.py:285-286)
template <bool DIR>
__device__ __forceinline__ void flux_q_tile(const Op1DDev& op, const double* st, const double* ut,
                                            const double* ct, double* qt, int EB, int ebase) {
  const int p1 = op.p1;
  const double* D = st + TabOff::D(p1);
  int tot = (EB + 2) * p1;
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    int e = t / p1, i = t - e * p1;
    const double* ue = ut + e * p1;
    if (DIR) {
      const int eg = ebase + e - 1;
      if (eg < 0) { ue = ut + p1; i = 0; }                          // interior element 0, node 0
      else if (eg >= op.ne) { ue = ut + (e - 1) * p1; i = p1 - 1; }  // interior element ne-1, node P
    }
    double g = 0.0;
#pragma unroll 4
    for (int j = 0; j < p1; ++j) g = fma(D[i * p1 + j], ue[j], g);
    qt[t] = ct[t] * (op.s * g);
  }
}

// SIP accumulator B_i (apply_diffusion = -B/m) at node (el,i); dgsem.py:270-308.
// eg = global element; Dirichlet outer faces take adjoint-lift weight 1 (dgsem.py:196-201)
template <bool DIR>
__device__ __forceinline__ double sip_B_node(const Op1DDev& op, const double* st, const double* ut,
                                             const double* ct, const double* qt, int el, int i, int eg) {
  const int p1 = op.p1, P = p1 - 1;
  const double* D = st + TabOff::D(p1);
  const double* DTW = st + TabOff::DTW(p1);
  const int b = (el + 1) * p1;
  double B = 0.0;
#pragma unroll 4
  for (int k = 0; k < p1; ++k) B = fma(DTW[i * p1 + k], qt[b + k], B);
  // right face (e+1/2): minus = (el,P), plus = (el+1,0)
  double jr = ut[b + P] - ut[b + p1];
  // left face (e-1/2): minus = (el-1,P), plus = (el,0)
  double jl = ut[b - 1] - ut[b];
  if (i == P) {
    double G = -(0.5 * (qt[b + P] + qt[b + p1])) + (op.mu0 * (0.5 * (ct[b + P] + ct[b + p1]))) * jr;
    B += G;
  }
  if (i == 0) {
    double G = -(0.5 * (qt[b - 1] + qt[b])) + (op.mu0 * (0.5 * (ct[b - 1] + ct[b]))) * jl;
    B -= G;
  }
  const double wr = (DIR && eg == op.ne - 1) ? 1.0 : 0.5, wl = (DIR && eg == 0) ? 1.0 : 0.5;
  B -= (op.s * ((wr * ct[b + P]) * jr)) * D[P * p1 + i];
  B -= (op.s * ((wl * ct[b]) * jl)) * D[i];
  return B;
}

// fill a C tile from a coefficient descriptor (with halo); Dirichlet ghosts carry
// the interior boundary node's coefficient (one-sided C, dgsem.py:287-288)
template <bool DIR>
__device__ __forceinline__ void coef_tile(const Op1DDev& op, const CoefDev& k, double* ct, int ebase, int EB) {
  int tot = (EB + 2) * op.p1;
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    int el = t / op.p1 - 1, i = t - (t / op.p1) * op.p1;
    const int eg = ebase + el;
    if (DIR && eg < 0) ct[t] = coef_at(op, k, 0, 0);
    else if (DIR && eg >= op.ne) ct[t] = coef_at(op, k, op.ne - 1, op.p1 - 1);
    else ct[t] = coef_at(op, k, wrap(eg, op.ne), i);
  }
}

__device__ __forceinline__ void flag_nonfinite(int* status, double v, int e) {
  if (!isfinite(v)) atomicMin(status, e);
}

// space-time p-transfer tables
struct XferDev {
  int ne, pc, pf, Mc, Mf;
  const double* tab;   // It (Mf*Mc) | Pt (Mc*Mf) | Isp (pf*pc) | Psp (pc*pf) | Rsp (pc*pf)
};
__host__ __device__ inline int xo_It(const XferDev&) { return 0; }
__host__ __device__ inline int xo_Pt(const XferDev& x) { return x.Mf * x.Mc; }
__host__ __device__ inline int xo_Isp(const XferDev& x) { return 2 * x.Mf * x.Mc; }
__host__ __device__ inline int xo_Psp(const XferDev& x) { return 2 * x.Mf * x.Mc + x.pf * x.pc; }
__host__ __device__ inline int xo_Rsp(const XferDev& x) { return 2 * x.Mf * x.Mc + 2 * x.pf * x.pc; }
__host__ __device__ inline int xo_size(const XferDev& x) { return 2 * x.Mf * x.Mc + 3 * x.pf * x.pc; }


__global__ void k_reset_status(int* status, int reset_log);

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; it lets its own successor launch at once
// (launch_dependents) and waits for the predecessor's completion and memory
// flush (wait) before touching anything the predecessor wrote.  Both are
// no-ops without a programmatic dependency.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace sisdc
