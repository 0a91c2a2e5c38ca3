// 1-D compressible flow (SISDC_CNS1D: CompressibleFlow, problems.py:160-240)
// on the sm_100a sweep path: 3 conservative fields in the reference layout
// (3, n_elem, P+1), matrix-valued (3x3 per node) diffusion / SI coefficients.
//
//   kc_conv      apply_convection (dgsem.py:205-225): weak volume term + Rusanov
//   kc_sip       apply_diffusion with a matrix coefficient (dgsem.py:251-309)
//   kc_coef      coefficient materialisation (dgsem.py:229-239, 313-326, 356-396)
//   kc_eval      eval_rhs / node caches f, h1, h2 (dgsem.py:337-352, sdc.py:77-119)
//   kc_stage     stage rhs (sdc.py:218-237)
//   kc_pinv      element-block Jacobi: inverse of the diagonal element block of
//                M + a B[C] (the closed form of dgsem.py:414-490 restricted to
//                one element), Gauss-Jordan with partial pivoting
//   kc_bicgstab  the implicit solve (replaces splu, dgsem.py:503-533): the
//                pinned right-preconditioned BiCGStab of oracle/cg.py, ONE
//                launch per solve on a thread-block cluster (K <= 16 CTAs,
//                one thread per node holding the 3 fields), vectors in
//                registers / shared memory, face halo read through DSMEM,
//                cluster reductions in rank order (bitwise-identical scalars)
//
// The implicit system is non-symmetric (C = (dt_m/2) A_c^2 + A_d is not
// symmetric), so the CG of cg1d.cu does not apply.
#include <string>
#include <cooperative_groups.h>
#include "sisdc_cns.cuh"
#include "sisdc_host.h"

namespace cgx = cooperative_groups;

namespace sisdc {
namespace {

__host__ __device__ inline int cns_eb(int p1) { int eb = 96 / p1; return eb < 1 ? 1 : eb; }
struct W16c { double v[MAXM]; };

// coefficient matrix at node (e, i) from a descriptor; false for a zero coefficient
__device__ __forceinline__ bool cns_coef_node(const Op1DDev& op, const CoefDev& k, int e, int i, double* C) {
  const int gi = e * op.p1 + i;
  switch (k.kind) {
    case SISDC_COEF_CONST:
    case SISDC_COEF_FIELD: {
      const double v = k.kind == SISDC_COEF_CONST ? k.value : k.ptr[gi];
      for (int j = 0; j < 9; ++j) C[j] = 0.0;
      C[0] = v; C[4] = v; C[8] = v;
      return true;
    }
    case SISDC_COEF_MATRIX:
      for (int j = 0; j < 9; ++j) C[j] = k.ptr[(size_t)gi * 9 + j];
      return true;
    case SISDC_COEF_SI: {   // (dt_m/2) A_c(u_b)^2 (+ phys(u_b)), dgsem.py:356-396
      const double ub[3] = {k.ptr[gi], k.ptr[op.n + gi], k.ptr[2 * op.n + gi]};
      double J[9], Ph[9];
      cns_jac(op, ub, J);
      const double h = 0.5 * k.value;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          C[a * 3 + b] = h * ((J[a * 3] * J[b] + J[a * 3 + 1] * J[3 + b]) + J[a * 3 + 2] * J[6 + b]);
      if (cns_phys(op, ub, e, Ph))
        for (int j = 0; j < 9; ++j) C[j] = C[j] + Ph[j];
      return true;
    }
    case SISDC_COEF_PHYS: {
      const double ub[3] = {k.ptr[gi], k.ptr[op.n + gi], k.ptr[2 * op.n + gi]};
      if (cns_phys(op, ub, e, C)) return true;
      for (int j = 0; j < 9; ++j) C[j] = 0.0;
      return false;
    }
    default:
      for (int j = 0; j < 9; ++j) C[j] = 0.0;
      return false;
  }
}

// tile of EB elements + one periodic halo element per side, field-major:
// ut[c*T + (el+1)*p1 + i]
__device__ __forceinline__ void cns_load_tile(const Op1DDev& op, double* ut, const double* __restrict__ u, int ebase,
                                              int EB) {
  const int p1 = op.p1, T = (EB + 2) * p1;
  for (int t = threadIdx.x; t < 3 * T; t += blockDim.x) {
    const int c = t / T, r = t - c * T, el = r / p1 - 1, i = r - (r / p1) * p1;
    const int eg = ebase + el;
    if (op.bc == SISDC_DIRICHLET && (eg < 0 || eg >= op.ne))   // ghost element: the outside state g(t)
      ut[t] = eg < 0 ? op.gl3[c] : op.gr3[c];
    else
      ut[t] = u[(size_t)c * op.n + wrap(eg, op.ne) * p1 + i];
  }
}
// ct[t*9 + ab] for every tile node
__device__ __forceinline__ void cns_coef_tile(const Op1DDev& op, const CoefDev& k, double* ct, int ebase, int EB) {
  const int p1 = op.p1, T = (EB + 2) * p1;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int el = t / p1 - 1, i = t - (t / p1) * p1;
    const int eg = ebase + el;
    if (op.bc == SISDC_DIRICHLET && eg < 0) cns_coef_node(op, k, 0, 0, ct + t * 9);
    else if (op.bc == SISDC_DIRICHLET && eg >= op.ne) cns_coef_node(op, k, op.ne - 1, p1 - 1, ct + t * 9);
    else cns_coef_node(op, k, wrap(eg, op.ne), i, ct + t * 9);
  }
}
// ft[c*T + t] = flux(u) at every tile node
__device__ __forceinline__ void cns_flux_tile(const Op1DDev& op, const double* ut, double* ft, int T) {
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const double u[3] = {ut[t], ut[T + t], ut[2 * T + t]};
    double f[3];
    cns_flux(op, u, f);
    ft[t] = f[0]; ft[T + t] = f[1]; ft[2 * T + t] = f[2];
  }
}
// q_a = sum_b C_ab (2/dx) (D u_b) at every tile node
__device__ __forceinline__ void cns_q_tile(const Op1DDev& op, const double* st, const double* ut, const double* ct,
                                           double* qt, int T, int ebase) {
  const int p1 = op.p1;
  const double* D = st + TabOff::D(p1);
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int e = t / p1;
    int i = t - e * p1, es = e;
    if (op.bc == SISDC_DIRICHLET) {   // ghosts carry the interior boundary node's q (dgsem.py:285-286)
      const int eg = ebase + e - 1;
      if (eg < 0) { es = e + 1; i = 0; }
      else if (eg >= op.ne) { es = e - 1; i = p1 - 1; }
    }
    double g[3];
    for (int b = 0; b < 3; ++b) {
      const double* ue = ut + b * T + es * p1;
      double s = 0.0;
      for (int j = 0; j < p1; ++j) s = fma(D[i * p1 + j], ue[j], s);
      g[b] = op.s * s;
    }
    const double* C = ct + t * 9;
    for (int a = 0; a < 3; ++a) qt[a * T + t] = (C[a * 3] * g[0] + C[a * 3 + 1] * g[1]) + C[a * 3 + 2] * g[2];
  }
}
// Rusanov flux of the system (dgsem.py:217-220)
__device__ __forceinline__ void cns_rusanov(const Op1DDev& op, const double* um, const double* up, double* fh) {
  const double lam = fmax(cns_speed(op, um[0], um[1], um[2]), cns_speed(op, up[0], up[1], up[2]));
  double fm[3], fp[3];
  cns_flux(op, um, fm);
  cns_flux(op, up, fp);
  for (int c = 0; c < 3; ++c) fh[c] = 0.5 * (fm[c] + fp[c]) - 0.5 * lam * (up[c] - um[c]);
}
// convection at tile node (el, i) (dgsem.py:205-225)
__device__ __forceinline__ void cns_conv_node(const Op1DDev& op, const double* st, const double* ut,
                                              const double* ft, int T, int el, int i, double* out) {
  const int p1 = op.p1, P = p1 - 1, b = (el + 1) * p1;
  const double* DTW = st + TabOff::DTW(p1);
  double v[3];
  for (int c = 0; c < 3; ++c) {
    double s = 0.0;
    for (int k = 0; k < p1; ++k) s = fma(DTW[i * p1 + k], ft[c * T + b + k], s);
    v[c] = s;
  }
  if (i == P) {
    const double um[3] = {ut[b + P], ut[T + b + P], ut[2 * T + b + P]};
    const double up[3] = {ut[b + p1], ut[T + b + p1], ut[2 * T + b + p1]};
    double fh[3];
    cns_rusanov(op, um, up, fh);
    for (int c = 0; c < 3; ++c) v[c] -= fh[c];
  }
  if (i == 0) {
    const double um[3] = {ut[b - 1], ut[T + b - 1], ut[2 * T + b - 1]};
    const double up[3] = {ut[b], ut[T + b], ut[2 * T + b]};
    double fh[3];
    cns_rusanov(op, um, up, fh);
    for (int c = 0; c < 3; ++c) v[c] += fh[c];
  }
  const double mi = st[TabOff::minv(p1) + i];
  for (int c = 0; c < 3; ++c) out[c] = v[c] * mi;
}
// SIP accumulator B (apply_diffusion = -B/m) at tile node (el, i), matrix
// coefficient; face penalty mu0 {C}[u], average flux, adjoint lift with each
// side's own coefficient (dgsem.py:270-308)
__device__ __forceinline__ void cns_B_node(const Op1DDev& op, const double* st, const double* ut, const double* ct,
                                           const double* qt, int T, int el, int i, double* B, int eg) {
  // Dirichlet outer faces take adjoint-lift weight 1 (dgsem.py:196-201)
  const double wr = (op.bc == SISDC_DIRICHLET && eg == op.ne - 1) ? 1.0 : 0.5;
  const double wl = (op.bc == SISDC_DIRICHLET && eg == 0) ? 1.0 : 0.5;
  const int p1 = op.p1, P = p1 - 1, b = (el + 1) * p1;
  const double* D = st + TabOff::D(p1);
  const double* DTW = st + TabOff::DTW(p1);
  for (int c = 0; c < 3; ++c) {
    double s = 0.0;
    for (int k = 0; k < p1; ++k) s = fma(DTW[i * p1 + k], qt[c * T + b + k], s);
    B[c] = s;
  }
  double jr[3], jl[3];
  for (int c = 0; c < 3; ++c) {
    jr[c] = ut[c * T + b + P] - ut[c * T + b + p1];
    jl[c] = ut[c * T + b - 1] - ut[c * T + b];
  }
  const double* Cmr = ct + (b + P) * 9;    // right face: minus (el, P), plus (el+1, 0)
  const double* Cpr = ct + (b + p1) * 9;
  const double* Cml = ct + (b - 1) * 9;    // left face: minus (el-1, P), plus (el, 0)
  const double* Cpl = ct + b * 9;
  for (int a = 0; a < 3; ++a) {
    if (i == P) {
      double pen = 0.0;
      for (int c = 0; c < 3; ++c) pen += (0.5 * (Cmr[a * 3 + c] + Cpr[a * 3 + c])) * jr[c];
      B[a] += op.mu0 * pen - 0.5 * (qt[a * T + b + P] + qt[a * T + b + p1]);
    }
    if (i == 0) {
      double pen = 0.0;
      for (int c = 0; c < 3; ++c) pen += (0.5 * (Cml[a * 3 + c] + Cpl[a * 3 + c])) * jl[c];
      B[a] -= op.mu0 * pen - 0.5 * (qt[a * T + b - 1] + qt[a * T + b]);
    }
    const double lm = wr * ((Cmr[a * 3] * jr[0] + Cmr[a * 3 + 1] * jr[1]) + Cmr[a * 3 + 2] * jr[2]);
    const double lp = wl * ((Cpl[a * 3] * jl[0] + Cpl[a * 3 + 1] * jl[1]) + Cpl[a * 3 + 2] * jl[2]);
    B[a] -= (op.s * lm) * D[P * p1 + i];
    B[a] -= (op.s * lp) * D[i];
  }
}

// ----------------------------------------------------------------- kernels
__global__ void kc_conv(Op1DDev op, const double* __restrict__ u, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int p1 = op.p1, EB = cns_eb(p1), T = (EB + 2) * p1, ebase = blockIdx.x * EB;
  double* st = sm;
  double* ut = st + TabOff::size(p1);
  double* ft = ut + 3 * T;
  load_tab(st, op.tab, p1);
  cns_load_tile(op, ut, u, ebase, EB);
  __syncthreads();
  cns_flux_tile(op, ut, ft, T);
  __syncthreads();
  const int t = threadIdx.x, el = t / p1, i = t - el * p1;
  if (!(el < EB && ebase + el < op.ne)) return;
  double v[3];
  cns_conv_node(op, st, ut, ft, T, el, i, v);
  const size_t gi = (size_t)(ebase + el) * p1 + i;
  for (int c = 0; c < 3; ++c) out[c * op.n + gi] = v[c];
}

__global__ void kc_sip(Op1DDev op, CoefDev k, const double* __restrict__ u, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int p1 = op.p1, EB = cns_eb(p1), T = (EB + 2) * p1, ebase = blockIdx.x * EB;
  double* st = sm;
  double* ut = st + TabOff::size(p1);
  double* qt = ut + 3 * T;
  double* ct = qt + 3 * T;
  load_tab(st, op.tab, p1);
  cns_load_tile(op, ut, u, ebase, EB);
  cns_coef_tile(op, k, ct, ebase, EB);
  __syncthreads();
  cns_q_tile(op, st, ut, ct, qt, T, ebase);
  __syncthreads();
  const int t = threadIdx.x, el = t / p1, i = t - el * p1;
  if (!(el < EB && ebase + el < op.ne)) return;
  double B[3];
  cns_B_node(op, st, ut, ct, qt, T, el, i, B, ebase + el);
  const double mi = st[TabOff::minv(p1) + i];
  const size_t gi = (size_t)(ebase + el) * p1 + i;
  for (int c = 0; c < 3; ++c) out[c * op.n + gi] = -B[c] * mi;
}

__global__ void kc_coef(Op1DDev op, CoefDev k, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= op.n) return;
  double C[9];
  cns_coef_node(op, k, t / op.p1, t % op.p1, C);
  for (int j = 0; j < 9; ++j) out[(size_t)t * 9 + j] = C[j];
}

// node caches (sdc.py:77-98) / eval_rhs (dgsem.py:337-352); blockIdx.y = node
struct CnsCacheArgs {
  const double* u0;
  const double* u;          // (M, 3n)
  const double* conv_prev;  // nullable: m_count vectors, conv(u_{m-1}) of every evaluated node
  int scheme, m_first, mode;
  W16c dts;
  double* f;
  double* h1;
  double* h2;               // nullable
  int* status;
  int has_bnd;              // Dirichlet: outside states per node
  double bnd[MAXM][12];     // g_l(t_m), g_r(t_m), g_l(t_{m-1}), g_r(t_{m-1}) (3 fields each)
};

__global__ void kc_eval(Op1DDev op_in, CnsCacheArgs a) {
  extern __shared__ double sm[];
  Op1DDev op = op_in, opp = op_in;   // boundary data at t_m (u_m) and t_{m-1} (conv of u_{m-1})
  if (a.has_bnd) {
    const int mm = a.m_first + blockIdx.y;
    for (int c = 0; c < 3; ++c) {
      op.gl3[c] = a.bnd[mm][c]; op.gr3[c] = a.bnd[mm][3 + c];
      opp.gl3[c] = a.bnd[mm][6 + c]; opp.gr3[c] = a.bnd[mm][9 + c];
    }
  }
  const int p1 = op.p1, EB = cns_eb(p1), T = (EB + 2) * p1, ebase = blockIdx.x * EB;
  const size_t N = (size_t)3 * op.n;
  const int m = a.m_first + blockIdx.y;
  double* st = sm;
  double* ut = st + TabOff::size(p1);   // u_m
  double* ft = ut + 3 * T;              // flux tile, then u_{m-1} tile
  double* qt = ft + 3 * T;
  double* ct = qt + 3 * T;
  const double* um = a.u + (size_t)m * N;
  const double* up = m == 0 ? a.u0 : a.u + (size_t)(m - 1) * N;
  load_tab(st, op.tab, p1);
  cns_load_tile(op, ut, um, ebase, EB);
  CoefDev phys{SISDC_COEF_PHYS, 0.0, um};
  cns_coef_tile(op, phys, ct, ebase, EB);
  __syncthreads();
  cns_flux_tile(op, ut, ft, T);
  cns_q_tile(op, st, ut, ct, qt, T, ebase);
  __syncthreads();
  const int t = threadIdx.x, el = t / p1, i = t - el * p1;
  const bool own = el < EB && ebase + el < op.ne;
  const size_t gi = (size_t)(ebase + el) * p1 + i;
  const double mi = st[TabOff::minv(p1) + i];
  double cm[3] = {0.0, 0.0, 0.0}, f[3] = {0.0, 0.0, 0.0};
  if (own) {
    cns_conv_node(op, st, ut, ft, T, el, i, cm);
    double B[3];
    cns_B_node(op, st, ut, ct, qt, T, el, i, B, ebase + el);   // zero coefficient -> B = 0
    for (int c = 0; c < 3; ++c) {
      f[c] = cm[c] + (-B[c] * mi);
      flag_nonfinite(a.status, f[c], ebase + el);
      a.f[(size_t)m * N + c * op.n + gi] = f[c];
    }
  }
  if (a.mode == 0) return;
  const double dtm = a.dts.v[m];
  if (dtm == 0.0) {   // sdc.py:90-94
    if (own)
      for (int c = 0; c < 3; ++c) {
        a.h1[(size_t)m * N + c * op.n + gi] = 0.0;
        if (a.h2) a.h2[(size_t)m * N + c * op.n + gi] = 0.0;
      }
    return;
  }
  __syncthreads();
  // C_m frozen at u_{m-1}: SI for si1/si2, physical for euler (dgsem.py:365-366)
  CoefDev cmod = a.scheme == SISDC_EULER ? CoefDev{SISDC_COEF_PHYS, 0.0, up} : CoefDev{SISDC_COEF_SI, dtm, up};
  cns_coef_tile(op, cmod, ct, ebase, EB);
  if (a.conv_prev == nullptr) cns_load_tile(opp, ft, up, ebase, EB);   // u_{m-1} tile
  __syncthreads();
  cns_q_tile(op, st, ut, ct, qt, T, ebase);
  __syncthreads();
  double* fpt = qt;   // reused below only after B is formed
  double d[3] = {0.0, 0.0, 0.0}, cp[3] = {0.0, 0.0, 0.0};
  if (own) {
    double B[3];
    cns_B_node(op, st, ut, ct, qt, T, el, i, B, ebase + el);
    for (int c = 0; c < 3; ++c) d[c] = -B[c] * mi;
  }
  if (a.conv_prev) {
    if (own)
      for (int c = 0; c < 3; ++c) cp[c] = a.conv_prev[(size_t)(m - a.m_first) * 3 * op.n + c * op.n + gi];
  } else {
    __syncthreads();
    cns_flux_tile(opp, ft, fpt, T);
    __syncthreads();
    if (own) cns_conv_node(opp, st, ft, fpt, T, el, i, cp);
  }
  if (!own) return;
  for (int c = 0; c < 3; ++c) {
    a.h1[(size_t)m * N + c * op.n + gi] = dtm * (cp[c] + d[c]);
    if (a.h2) a.h2[(size_t)m * N + c * op.n + gi] = dtm * (cm[c] + d[c]);
  }
}

struct CnsStageArgs {
  const double* base;
  const double* conv_in;
  double dt_m;
  const double* f_old;
  int M;
  W16c w;
  double dt;
  const double* g;
  const double* h;
  double* rhs;
  double* conv_out;
};

// rhs = base + dt sum_j w_j f_old[j] (+ g) + dt_m conv(conv_in) - h   (sdc.py:218-237)
__global__ void kc_stage(Op1DDev op, CnsStageArgs a) {
  extern __shared__ double sm[];
  const int p1 = op.p1, EB = cns_eb(p1), T = (EB + 2) * p1, ebase = blockIdx.x * EB;
  const size_t N = (size_t)3 * op.n;
  double* st = sm;
  double* ut = st + TabOff::size(p1);
  double* ft = ut + 3 * T;
  load_tab(st, op.tab, p1);
  cns_load_tile(op, ut, a.conv_in, ebase, EB);
  __syncthreads();
  cns_flux_tile(op, ut, ft, T);
  __syncthreads();
  const int t = threadIdx.x, el = t / p1, i = t - el * p1;
  if (!(el < EB && ebase + el < op.ne)) return;
  double cv[3];
  cns_conv_node(op, st, ut, ft, T, el, i, cv);
  for (int c = 0; c < 3; ++c) {
    const size_t gi = (size_t)c * op.n + (size_t)(ebase + el) * p1 + i;
    if (a.conv_out) a.conv_out[gi] = cv[c];
    double q = 0.0;
    if (a.f_old) {
      double acc = 0.0;
      for (int j = 0; j < a.M; ++j) acc = fma(a.w.v[j], a.f_old[(size_t)j * N + gi], acc);
      q = a.dt * acc;
    }
    if (a.g) q = q + a.g[gi];
    double r = (a.base[gi] + q) + a.dt_m * cv[c];
    if (a.h) r = r - a.h[gi];
    a.rhs[gi] = r;
  }
}

// Element-block Jacobi: pinv[e] = inverse of the (3(P+1))^2 diagonal block of
// M + a B[C] for element e, rows/cols ordered (field, node).  Entries
// (dgsem.py:414-490 restricted to the element; C materialised, (n, 9)):
//   m_i d_ab d_ij + a [ s sum_k D_ki w_k C_ab(k) D_kj
//     - [i=P] s/2 CLr_ab D_Pj - [j=P] s/2 CLr_ab D_Pi + [i=j=P] mu0 (CLr+CRr)_ab / 2
//     + [i=0] s/2 CRl_ab D_0j + [j=0] s/2 CRl_ab D_0i + [i=j=0] mu0 (CLl+CRl)_ab / 2 ]
// with CLr = C(e,P), CRr = C(e+1,0), CLl = C(e-1,P), CRl = C(e,0).
__global__ void kc_pinv(Op1DDev op, const double* __restrict__ C9, double a, double* __restrict__ pinv) {
  extern __shared__ double sm[];
  const int p1 = op.p1, P = p1 - 1, nb = 3 * p1, w2 = 2 * nb, e = blockIdx.x;
  double* st = sm;
  double* Ag = st + TabOff::size(p1);   // [nb][2 nb]
  double* fr = Ag + nb * w2;            // [nb] elimination factors
  __shared__ int piv;
  __shared__ double pval;
  load_tab(st, op.tab, p1);
  __syncthreads();
  const double* D = st + TabOff::D(p1);
  const double* w = st + TabOff::w(p1);
  const double* CLr = C9 + ((size_t)e * p1 + P) * 9;
  const double* CRr = C9 + ((size_t)wrap(e + 1, op.ne) * p1) * 9;
  const double* CLl = C9 + ((size_t)wrap(e - 1, op.ne) * p1 + P) * 9;
  const double* CRl = C9 + ((size_t)e * p1) * 9;   // (re-pointed one-sided at Dirichlet outer faces below)
  const double s = op.s;
  const bool dR = op.bc == SISDC_DIRICHLET && e == op.ne - 1, dL = op.bc == SISDC_DIRICHLET && e == 0;
  const double hsR = dR ? op.s : 0.5 * op.s, hsL = dL ? op.s : 0.5 * op.s;   // outer faces: weight 1, one-sided C
  if (dR) CRr = CLr;
  if (dL) CLl = CRl;
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int r = idx / nb, col = idx - r * nb;
    const int ca = r / p1, i = r - ca * p1, cb = col / p1, j = col - cb * p1;
    const int ab = ca * 3 + cb;
    double v = 0.0;
    for (int k = 0; k < p1; ++k) v = fma(D[k * p1 + i] * w[k], C9[((size_t)e * p1 + k) * 9 + ab] * D[k * p1 + j], v);
    v = s * v;
    if (i == P) v -= hsR * CLr[ab] * D[P * p1 + j];
    if (j == P) v -= hsR * CLr[ab] * D[P * p1 + i];
    if (i == P && j == P) v += op.mu0 * (0.5 * (CLr[ab] + CRr[ab]));
    if (i == 0) v += hsL * CRl[ab] * D[j];
    if (j == 0) v += hsL * CRl[ab] * D[i];
    if (i == 0 && j == 0) v += op.mu0 * (0.5 * (CLl[ab] + CRl[ab]));
    double m = (r == col) ? st[TabOff::m(p1) + i] : 0.0;
    Ag[r * w2 + col] = m + a * v;
    Ag[r * w2 + nb + col] = r == col ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int c = 0; c < nb; ++c) {
    if (threadIdx.x < 32) {   // partial pivoting: first row of maximal |A[r][c]|, r >= c
      double best = -1.0;
      int br = c;
      for (int r = c + threadIdx.x; r < nb; r += 32) {
        const double v = fabs(Ag[r * w2 + c]);
        if (v > best) { best = v; br = r; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (ob > best || (ob == best && orr < br)) { best = ob; br = orr; }
      }
      if (threadIdx.x == 0) piv = br;
    }
    __syncthreads();
    const int pr = piv;
    if (pr != c)
      for (int col = threadIdx.x; col < w2; col += blockDim.x) {
        const double t0 = Ag[c * w2 + col];
        Ag[c * w2 + col] = Ag[pr * w2 + col];
        Ag[pr * w2 + col] = t0;
      }
    __syncthreads();
    if (threadIdx.x == 0) pval = Ag[c * w2 + c];
    __syncthreads();
    const double inv = 1.0 / pval;
    for (int col = threadIdx.x; col < w2; col += blockDim.x) Ag[c * w2 + col] *= inv;
    __syncthreads();
    for (int r = threadIdx.x; r < nb; r += blockDim.x) fr[r] = r == c ? 0.0 : Ag[r * w2 + c];
    __syncthreads();
    for (int idx = threadIdx.x; idx < nb * w2; idx += blockDim.x) {
      const int r = idx / w2, col = idx - r * w2;
      if (r != c) Ag[idx] = fma(-fr[r], Ag[c * w2 + col], Ag[idx]);
    }
    __syncthreads();
  }
  double* out = pinv + (size_t)e * nb * nb;
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int r = idx / nb, col = idx - r * nb;
    out[idx] = Ag[r * w2 + nb + col];
  }
}

// ------------------------------------------------------------- BiCGStab
struct BicgArgs {
  Op1DDev op;
  const double* C9;     // materialised coefficient (n, 9)
  const double* pinv;   // element-block inverses (ne, nb, nb)
  const double* dbc;    // Dirichlet: D(0; t) (affine part of the SIP), nullable
  double a;
  const double* rhs;
  double* x;
  double rtol2;
  int maxit, E, K;
  int* status;
  int* log_it;
  double* log_margin;
  int log_cap;
  // grid mode (levels beyond one cluster: K > 16 CTAs of a cooperative launch): the face-node halo
  // and the reduction slots go through global memory, grid barriers replace the cluster barriers.
  // Layout (doubles): halo [2 buf][K][2 sides][U0 U1 U2 Q0 Q1 Q2] | slots [2][K][BNV]
  double* gws;
};

constexpr int BNV = 4;   // reduction width

template <int P1>
__global__ void __launch_bounds__(256) kc_bicgstab(BicgArgs A) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = P1 - 1, NB = 3 * P1;
  const Op1DDev& op = A.op;
  cgx::cluster_group cl = cgx::this_cluster();
  cgx::grid_group grid = cgx::this_grid();
  const bool GM = A.gws != nullptr;
  const int rank = GM ? (int)blockIdx.x : (int)cl.block_rank();
  const int K = A.K, E = A.E, NL = E * P1;
  double* const gH = A.gws;                         // [2][K][12]
  double* const gS = A.gws + (size_t)2 * K * 12;    // [2][K][BNV]
  unsigned nsum = 0;                                // reductions done (slot parity)
  auto csync = [&]() {   // every CTA's shared data (cluster) / published halo and slots (grid) visible
    if (GM) {
      __threadfence();
      grid.sync();
    } else {
      cl.sync();
    }
  };
  const int e0 = rank * E, e1 = min(op.ne, e0 + E);
  const int nl = (e1 - e0) * P1;
  const int L = threadIdx.x, el = L / P1, i = L - el * P1;
  const bool own = L < nl;
  const bool first = el == 0, last = (el + 1) * P1 >= nl;
  const int nw = (blockDim.x + 31) >> 5, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // shared layout
  double* st = sm;                                   // tables
  double* U = st + TabOff::size(P1);                 // [2 buf][3][NL]
  double* Q = U + 2 * 3 * NL;                        // [2 buf][3][NL]
  double* Pv = Q + 2 * 3 * NL;                       // [3][NL] vector to precondition
  double* Cs = Pv + 3 * NL;                          // [NL][9]
  double* wsum = Cs + 9 * NL;                        // [nw][BNV]
  double* slot = wsum + nw * BNV;                    // [BNV]
  double* bc = slot + BNV;                           // [BNV]
  for (int t = threadIdx.x; t < TabOff::size(P1); t += blockDim.x) st[t] = op.tab[t];
  // neighbour ranks / elements (periodic)
  const int egL = wrap(e0 - 1, op.ne), egR = wrap(e1, op.ne);
  const int rL = egL / E, rR = egR / E;
  const int lastL = egL - rL * E;                    // local index of the left neighbour element in rank rL
  const double* D = st + TabOff::D(P1);
  const double* DTW = st + TabOff::DTW(P1);
  double Cn[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double a_shift = A.a;
  double xv[3] = {0.0, 0.0, 0.0}, bv[3] = {0.0, 0.0, 0.0};
  const size_t gi = (size_t)e0 * P1 + L;
  __syncthreads();
  const double mi = st[TabOff::m(P1) + i];
  if (own) {
    for (int j = 0; j < 9; ++j) { Cn[j] = A.C9[gi * 9 + j]; Cs[L * 9 + j] = Cn[j]; }
    for (int c = 0; c < 3; ++c) {   // b = M rhs (+ a M D(0; t), dgsem.py:517-529)
      xv[c] = A.rhs[c * op.n + gi];
      bv[c] = mi * xv[c];
      if (A.dbc) bv[c] = bv[c] + (a_shift * mi) * A.dbc[c * op.n + gi];
    }
  }
  // face coefficients of the element's two faces (global field: no exchange needed)
  const int eg = e0 + el;
  double CRr[9], CLl[9];
  {
    const size_t ir = (size_t)wrap(eg + 1, op.ne) * P1, il = (size_t)wrap(eg - 1, op.ne) * P1 + P;
    for (int j = 0; j < 9; ++j) { CRr[j] = own ? A.C9[ir * 9 + j] : 0.0; CLl[j] = own ? A.C9[il * 9 + j] : 0.0; }
  }
  const double* pinv_rows = A.pinv + (size_t)(own ? eg : 0) * NB * NB;
  const bool dL = op.bc == SISDC_DIRICHLET && eg == 0, dR = op.bc == SISDC_DIRICHLET && eg == op.ne - 1;
  const double wL = dL ? 1.0 : 0.5, wR = dR ? 1.0 : 0.5;   // adjoint-lift face weights (dgsem.py:196-201)
  const double sc = op.s, mu0 = op.mu0, a = A.a;
  __syncthreads();

  // y = Pinv_e v_e for this node's three rows; v staged in Pv
  auto precond = [&](const double* v, double* y) {
    if (L < NL)   // threads past the CTA's node range (warp rounding) own no slot
      for (int c = 0; c < 3; ++c) Pv[c * NL + L] = own ? v[c] : 0.0;
    __syncthreads();
    if (!own) { y[0] = y[1] = y[2] = 0.0; return; }
    for (int c = 0; c < 3; ++c) {
      const double* row = pinv_rows + (size_t)(c * P1 + i) * NB;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int j = 0; j < P1; ++j) {
        s0 = fma(row[j], Pv[el * P1 + j], s0);
        s1 = fma(row[P1 + j], Pv[NL + el * P1 + j], s1);
        s2 = fma(row[2 * P1 + j], Pv[2 * NL + el * P1 + j], s2);
      }
      y[c] = (s0 + s1) + s2;
    }
  };
  // w = (M + a B[C]) v on own nodes (buffer buf of U / Q)
  auto matvec = [&](const double* v, double* w, int buf) {
    double* Ub = U + buf * 3 * NL;
    double* Qb = Q + buf * 3 * NL;
    if (L < NL)
      for (int c = 0; c < 3; ++c) Ub[c * NL + L] = own ? v[c] : 0.0;
    __syncthreads();
    if (own) {
      double g[3];
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < P1; ++j) s = fma(D[i * P1 + j], Ub[b * NL + el * P1 + j], s);
        g[b] = sc * s;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) Qb[c * NL + L] = (Cn[c * 3] * g[0] + Cn[c * 3 + 1] * g[1]) + Cn[c * 3 + 2] * g[2];
    }
    if (GM && own) {   // publish this CTA's two outer face nodes (its first node, its last node)
      double* h = gH + ((size_t)buf * K + rank) * 12;
      if (L == 0)
        for (int c = 0; c < 3; ++c) { h[c] = Ub[c * NL]; h[3 + c] = Qb[c * NL]; }
      if (L == nl - 1)
        for (int c = 0; c < 3; ++c) { h[6 + c] = Ub[c * NL + L]; h[9 + c] = Qb[c * NL + L]; }
    }
    csync();   // U, Q of every CTA visible (DSMEM / the published face nodes)
    if (!own) { w[0] = w[1] = w[2] = 0.0; return; }
    // neighbour face node values: right (el+1, 0), left (el-1, P)
    double nuR[3], nqR[3], nuL[3], nqL[3];
    if (!last) {
      for (int c = 0; c < 3; ++c) { nuR[c] = Ub[c * NL + (el + 1) * P1]; nqR[c] = Qb[c * NL + (el + 1) * P1]; }
    } else if (GM) {
      const double* h = gH + ((size_t)buf * K + rR) * 12;
      for (int c = 0; c < 3; ++c) { nuR[c] = __ldcg(h + c); nqR[c] = __ldcg(h + 3 + c); }
    } else {
      const double* UR = cl.map_shared_rank(Ub, rR);
      const double* QR = cl.map_shared_rank(Qb, rR);
      for (int c = 0; c < 3; ++c) { nuR[c] = UR[c * NL]; nqR[c] = QR[c * NL]; }
    }
    if (!first) {
      for (int c = 0; c < 3; ++c) { nuL[c] = Ub[c * NL + (el - 1) * P1 + P]; nqL[c] = Qb[c * NL + (el - 1) * P1 + P]; }
    } else if (GM) {
      const double* h = gH + ((size_t)buf * K + rL) * 12;
      for (int c = 0; c < 3; ++c) { nuL[c] = __ldcg(h + 6 + c); nqL[c] = __ldcg(h + 9 + c); }
    } else {
      const double* UL = cl.map_shared_rank(Ub, rL);
      const double* QL = cl.map_shared_rank(Qb, rL);
      for (int c = 0; c < 3; ++c) { nuL[c] = UL[c * NL + lastL * P1 + P]; nqL[c] = QL[c * NL + lastL * P1 + P]; }
    }
    const int ob = el * P1;
    double jr[3], jl[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {   // Dirichlet outer faces: outside value 0 in the linear operator
      jr[c] = Ub[c * NL + ob + P] - (dR ? 0.0 : nuR[c]);
      jl[c] = (dL ? 0.0 : nuL[c]) - Ub[c * NL + ob];
    }
    const double* Cmr = Cs + (ob + P) * 9;
    const double* Cpl = Cs + ob * 9;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double B = 0.0;
#pragma unroll
      for (int k = 0; k < P1; ++k) B = fma(DTW[i * P1 + k], Qb[c * NL + ob + k], B);
      if (i == P) {   // Dirichlet: one-sided q and C (dgsem.py:285-288)
        double pen = 0.0;
        for (int b = 0; b < 3; ++b) pen += (0.5 * (Cmr[c * 3 + b] + (dR ? Cmr : CRr)[c * 3 + b])) * jr[b];
        const double qo = Qb[c * NL + ob + P];
        B += mu0 * pen - 0.5 * (qo + (dR ? qo : nqR[c]));
      }
      if (i == 0) {
        double pen = 0.0;
        for (int b = 0; b < 3; ++b) pen += (0.5 * ((dL ? Cpl : CLl)[c * 3 + b] + Cpl[c * 3 + b])) * jl[b];
        const double qo = Qb[c * NL + ob];
        B -= mu0 * pen - 0.5 * ((dL ? qo : nqL[c]) + qo);
      }
      const double lm = wR * ((Cmr[c * 3] * jr[0] + Cmr[c * 3 + 1] * jr[1]) + Cmr[c * 3 + 2] * jr[2]);
      const double lp = wL * ((Cpl[c * 3] * jl[0] + Cpl[c * 3 + 1] * jl[1]) + Cpl[c * 3 + 2] * jl[2]);
      B -= (sc * lm) * D[P * P1 + i];
      B -= (sc * lp) * D[i];
      w[c] = fma(a, B, mi * v[c]);
    }
  };
  // cluster sum of NV values, identical bits in every CTA (rank order)
  auto csum = [&](double* v, int nv) {
    for (int j = 0; j < nv; ++j) {
      double t = v[j];
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) wsum[wid * BNV + j] = t;
    }
    __syncthreads();
    if (threadIdx.x < nv) {
      double t = 0.0;
      for (int q = 0; q < nw; ++q) t += wsum[q * BNV + threadIdx.x];
      slot[threadIdx.x] = t;
      if (GM) gS[((size_t)(nsum & 1u) * K + rank) * BNV + threadIdx.x] = t;
    }
    csync();
    if (threadIdx.x < nv) {
      double t = 0.0;
      if (GM) {
        const double* gs = gS + (size_t)(nsum & 1u) * K * BNV + threadIdx.x;
        for (int q = 0; q < K; ++q) t += __ldcg(gs + (size_t)q * BNV);
      } else {
        for (int q = 0; q < K; ++q) t += cl.map_shared_rank(slot, q)[threadIdx.x];
      }
      bc[threadIdx.x] = t;
    }
    ++nsum;
    __syncthreads();
    for (int j = 0; j < nv; ++j) v[j] = bc[j];
  };
  auto dot3 = [&](const double* p, const double* q) -> double {
    return own ? (p[0] * q[0] + p[1] * q[1]) + p[2] * q[2] : 0.0;
  };

  // ---- setup: r0 = b - A x0, r^ = r0, p = r0
  double r[3], rh[3], p[3], v[3], y[3], sv[3], z[3], t[3], w[3];
  matvec(xv, w, 0);
  for (int c = 0; c < 3; ++c) { r[c] = bv[c] - w[c]; rh[c] = r[c]; p[c] = r[c]; v[c] = 0.0; }
  double red[BNV] = {dot3(bv, bv), (own && (bv[0] != 0.0 || bv[1] != 0.0 || bv[2] != 0.0)) ? 1.0 : 0.0,
                     dot3(r, r), 0.0};
  csum(red, 3);
  if (red[1] == 0.0) {   // b == 0 -> zeros (dgsem.py:510-511)
    if (own)
      for (int c = 0; c < 3; ++c) A.x[c * op.n + gi] = 0.0;
    if (!GM) cl.sync();   // no CTA leaves while a peer may still read its shared memory
    return;
  }
  const double thr = A.rtol2 * red[0];
  double rr = red[2], rho = red[2], rhrh = red[2], rho_new = rho, alpha = 1.0, omega = 1.0;
  int k = 0;
  bool ok = true, fresh = true, restarted = false;
  for (;;) {
    if (!fresh) {
      const double beta = (rho_new / rho) * (alpha / omega);
      for (int c = 0; c < 3; ++c) p[c] = r[c] + beta * (p[c] - omega * v[c]);
      rho = rho_new;
    }
    fresh = false;
    precond(p, y);
    matvec(y, v, 0);
    double r1[BNV] = {dot3(rh, v), dot3(r, r), 0.0, 0.0};
    csum(r1, 2);
    if (k > 0) rr = r1[1];
    if (!isfinite(rr)) { ok = false; break; }   // breakdown / overflow: a failure, never "converged"
    if (!(rr > thr)) break;
    if (k >= A.maxit) { ok = false; break; }
    // Lanczos breakdown (r^ _|_ r): restart with r^ = p = r at the same k.  The
    // oracle tests before forming y, v; here (r, r) arrives with them, so the
    // restart recomputes y, v once (identical iterates, one extra matvec)
    if (!restarted && fabs(rho) <= 1e-10 * sqrt(rhrh * rr)) {
      for (int c = 0; c < 3; ++c) { rh[c] = r[c]; p[c] = r[c]; }
      rhrh = rr;
      rho = rr;
      restarted = true;
      fresh = true;
      continue;
    }
    restarted = false;
    alpha = rho / r1[0];
    for (int c = 0; c < 3; ++c) sv[c] = r[c] - alpha * v[c];
    precond(sv, z);
    matvec(z, t, 1);
    double r2[BNV] = {dot3(t, sv), dot3(t, t), dot3(rh, sv), dot3(rh, t)};
    csum(r2, 4);
    omega = r2[1] != 0.0 ? r2[0] / r2[1] : 0.0;
    for (int c = 0; c < 3; ++c) {
      xv[c] = xv[c] + alpha * y[c] + omega * z[c];
      r[c] = sv[c] - omega * t[c];
    }
    rho_new = r2[2] - omega * r2[3];
    ++k;
  }
  if (own)
    for (int c = 0; c < 3; ++c) A.x[c * op.n + gi] = xv[c];
  if (!GM) cl.sync();   // no CTA leaves while a peer may still read its shared memory
  if (rank == 0 && threadIdx.x == 0) {
    const int idx = atomicAdd(&A.status[2], 1);
    if (idx < A.log_cap) {
      A.log_it[idx] = ok ? k : -1;
      A.log_margin[idx] = thr > 0.0 ? sqrt(rr / thr) : 0.0;
    }
    if (!ok) atomicAdd(&A.status[1], 1);
  }
}

size_t tile_smem3(int p1, int nvec) { return sizeof(double) * (TabOff::size(p1) + nvec * (cns_eb(p1) + 2) * p1); }
dim3 tile_grid3(int ne, int p1, int ny = 1) { int EB = cns_eb(p1); return dim3((ne + EB - 1) / EB, ny); }
dim3 tile_block3(int p1) { int t = cns_eb(p1) * p1; return dim3((t + 31) / 32 * 32); }

template <int P1>
int launch_bicg_t(Ctx* c, BicgArgs& A, int threads, size_t smem) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kc_bicgstab<P1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(kc_bicgstab<P1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(A.K);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  if (A.gws != nullptr) {   // grid mode: cooperative launch, every block resident
    int per_sm = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kc_bicgstab<P1>, threads, smem);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    if (e != cudaSuccess) return c->cuda(e, "cns bicgstab occupancy");
    if (A.K > per_sm * sms || A.K > CG1G_MAXK)
      return c->fail(SISDC_ERR_UNSUPPORTED, "implicit_solve: 1-D CNS level too large for the grid-mode BiCGStab (" +
                                                std::to_string(A.K) + " blocks of 256 nodes, " +
                                                std::to_string(per_sm * sms) + " resident)");
    cudaLaunchAttribute atc[1];
    atc[0].id = cudaLaunchAttributeCooperative;
    atc[0].val.cooperative = 1;
    cfg.attrs = atc;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kc_bicgstab<P1>, A);
    if (e != cudaSuccess) return c->cuda(e, "cns bicgstab grid-mode launch");
    return c->after_launch("cns_bicgstab (grid mode)");
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = A.K;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kc_bicgstab<P1>, A);
  if (e != cudaSuccess) return c->cuda(e, "cns bicgstab cluster launch");
  return c->after_launch("cns_bicgstab");
}

}  // namespace

// ----------------------------------------------------------------- launchers
int cns_conv(Ctx* c, const Op1DDev& op, const double* u, double* out) {
  kc_conv<<<tile_grid3(op.ne, op.p1), tile_block3(op.p1), tile_smem3(op.p1, 6), c->stream>>>(op, u, out);
  return c->after_launch("cns_conv");
}
int cns_sip(Ctx* c, const Op1DDev& op, CoefDev k, const double* u, double* out) {
  kc_sip<<<tile_grid3(op.ne, op.p1), tile_block3(op.p1), tile_smem3(op.p1, 15), c->stream>>>(op, k, u, out);
  return c->after_launch("cns_sip");
}
int cns_coef(Ctx* c, const Op1DDev& op, CoefDev k, double* out) {
  kc_coef<<<(op.n + 127) / 128, 128, 0, c->stream>>>(op, k, out);
  return c->after_launch("cns_coef");
}
int cns_node_eval(Ctx* c, const Op1DDev& op, int mode, int scheme, int M, int m_first, int m_count,
                  const double* u0, const double* u, const double* conv_prev, const double* dts, double* f,
                  double* h1, double* h2, const double* bnd) {
  if (M > MAXM || m_first + m_count > M) return c->fail(SISDC_ERR_ARG, "bad node range");
  CnsCacheArgs a{};
  if (bnd) {
    a.has_bnd = 1;
    for (int m = 0; m < M; ++m)
      for (int j = 0; j < 12; ++j) a.bnd[m][j] = bnd[m * 12 + j];
  }
  a.u0 = u0; a.u = u; a.conv_prev = conv_prev; a.scheme = scheme; a.m_first = m_first; a.mode = mode;
  for (int m = 0; m < M; ++m) a.dts.v[m] = dts ? dts[m] : 0.0;
  a.f = f; a.h1 = h1; a.h2 = h2; a.status = c->d_status;
  kc_eval<<<tile_grid3(op.ne, op.p1, m_count), tile_block3(op.p1), tile_smem3(op.p1, 18), c->stream>>>(op, a);
  return c->after_launch("cns_eval");
}
int cns_stage(Ctx* c, const Op1DDev& op, const double* base, const double* conv_in, double dt_m,
              const double* f_old, int M, const double* w_row, double dt, const double* g, const double* h,
              double* rhs, double* conv_out) {
  if (M > MAXM) return c->fail(SISDC_ERR_ARG, "too many collocation nodes");
  CnsStageArgs a{};
  a.base = base; a.conv_in = conv_in; a.dt_m = dt_m; a.f_old = f_old; a.M = M; a.dt = dt;
  for (int j = 0; j < M; ++j) a.w.v[j] = (f_old && w_row) ? w_row[j] : 0.0;
  a.g = g; a.h = h; a.rhs = rhs; a.conv_out = conv_out;
  kc_stage<<<tile_grid3(op.ne, op.p1), tile_block3(op.p1), tile_smem3(op.p1, 6), c->stream>>>(op, a);
  return c->after_launch("cns_stage");
}
int cns_solve(Ctx* c, const Op1DDev& op, CoefDev k, double a, const double* rhs, double* x, double* c9,
              double* pinv, const double* dbc) {
  const int p1 = op.p1, nb = 3 * p1;
  // partition: one thread per node, <= 256 nodes per CTA, <= 16 CTAs
  int E = 256 / p1;
  int K = (op.ne + E - 1) / E;
  const bool grid_mode = K > 16;   // beyond one cluster: the same kernel as a cooperative launch
  E = (op.ne + K - 1) / K;
  K = (op.ne + E - 1) / E;
  if (int rc = cns_coef(c, op, k, c9)) return rc;
  const size_t smp = sizeof(double) * (TabOff::size(p1) + (size_t)nb * 2 * nb + nb);   // <= 46 KB at P = 15
  kc_pinv<<<op.ne, 256, smp, c->stream>>>(op, c9, a, pinv);
  if (int rc = c->after_launch("cns_pinv")) return rc;
  int threads = ((E * p1 + 31) / 32) * 32;
  if (threads < 64) threads = 64;
  const int NL = E * p1, nw = threads / 32;
  const size_t smem = sizeof(double) * (TabOff::size(p1) + 2 * 3 * NL + 2 * 3 * NL + 3 * NL + 9 * NL +
                                        nw * BNV + 2 * BNV);
  BicgArgs A{};
  A.op = op; A.C9 = c9; A.pinv = pinv; A.dbc = dbc; A.a = a; A.rhs = rhs; A.x = x;
  A.rtol2 = c->rtol * c->rtol; A.maxit = c->maxit; A.E = E; A.K = K;
  A.status = c->d_status; A.log_it = c->d_log_it; A.log_margin = c->d_log_margin; A.log_cap = c->log_cap;
  A.gws = grid_mode ? c->d_cg1g : nullptr;
  switch (p1) {
    case 2: return launch_bicg_t<2>(c, A, threads, smem);
    case 3: return launch_bicg_t<3>(c, A, threads, smem);
    case 4: return launch_bicg_t<4>(c, A, threads, smem);
    case 5: return launch_bicg_t<5>(c, A, threads, smem);
    case 6: return launch_bicg_t<6>(c, A, threads, smem);
    case 7: return launch_bicg_t<7>(c, A, threads, smem);
    case 8: return launch_bicg_t<8>(c, A, threads, smem);
    case 9: return launch_bicg_t<9>(c, A, threads, smem);
    case 10: return launch_bicg_t<10>(c, A, threads, smem);
    case 11: return launch_bicg_t<11>(c, A, threads, smem);
    case 12: return launch_bicg_t<12>(c, A, threads, smem);
    case 13: return launch_bicg_t<13>(c, A, threads, smem);
    case 14: return launch_bicg_t<14>(c, A, threads, smem);
    case 15: return launch_bicg_t<15>(c, A, threads, smem);
    case 16: return launch_bicg_t<16>(c, A, threads, smem);
    default: return c->fail(SISDC_ERR_UNSUPPORTED, "degree outside 1..15");
  }
}

}  // namespace sisdc
