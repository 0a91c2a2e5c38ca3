// Element kernels of the 1-D SI-SDC sweep: operator applications, fused
// sweep stages, node caches and the space-time p-transfers (sm_100a, fp64).
#include "sisdc_dev.cuh"
#include "sisdc_cns.cuh"
#include "sisdc_host.h"

namespace sisdc {

// elements per block for element kernels
__host__ __device__ inline int eb_for(int p1) { int eb = 128 / p1; return eb < 1 ? 1 : eb; }

struct W16 { double v[MAXM]; };   // small host arrays passed by value

// ------------------------------------------------------------ operators
template <bool DIR>
__global__ void k_apply_convection(Op1DDev op, const double* __restrict__ u, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int p1 = op.p1, EB = eb_for(p1);
  double* st = sm;
  double* ut = st + TabOff::size(p1);
  int ebase = blockIdx.x * EB;
  load_tab(st, op.tab, p1);
  load_tile<DIR>(op, ut, u, ebase, EB);
  __syncthreads();
  int t = threadIdx.x, el = t / p1, i = t - el * p1;
  if (el < EB && ebase + el < op.ne) out[(ebase + el) * p1 + i] = conv_node(op, st, ut, el, i);
}

// out = -B[C]u / m  (apply_diffusion, dgsem.py:251-309)
template <bool DIR>
__global__ void k_apply_diffusion(Op1DDev op, CoefDev c, const double* __restrict__ u, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int p1 = op.p1, EB = eb_for(p1), T = (EB + 2) * p1;
  double* st = sm;
  double* ut = st + TabOff::size(p1);
  double* ct = ut + T;
  double* qt = ct + T;
  int ebase = blockIdx.x * EB;
  load_tab(st, op.tab, p1);
  load_tile<DIR>(op, ut, u, ebase, EB);
  coef_tile<DIR>(op, c, ct, ebase, EB);
  __syncthreads();
  flux_q_tile<DIR>(op, st, ut, ct, qt, EB, ebase);
  __syncthreads();
  int t = threadIdx.x, el = t / p1, i = t - el * p1;
  if (el < EB && ebase + el < op.ne)
    out[(ebase + el) * p1 + i] = -sip_B_node<DIR>(op, st, ut, ct, qt, el, i, ebase + el) * st[TabOff::minv(p1) + i];
}

__global__ void k_coef_field(Op1DDev op, CoefDev c, double* __restrict__ out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < op.ne * op.p1) out[t] = coef_at(op, c, t / op.p1, t % op.p1);
}

// Node-parallel multi-state evaluation: blockIdx.y = node m.
//   mode 0: f[m] = eval_rhs(u[m])                              (dgsem.py:337-352)
//   mode 1: node caches f, h1, h2 of sdc.py:77-98 (coefficient frozen at u_{m-1})
struct CacheArgs {
  const double* u0;
  const double* u;          // (M, N)
  const double* conv_prev;  // nullable: m_count vectors, conv(u_{m-1}) of every evaluated node
  int scheme, m_first, mode;
  W16 dts;
  W16 gl, gr, glp, grp;     // Dirichlet outside states at t_m and t_{m-1} per node
  double* f;
  double* h1;
  double* h2;               // nullable
  int* status;              // [0] first non-finite element
};

template <bool DIR>
__global__ void k_node_eval(Op1DDev op_in, CacheArgs a) {
  extern __shared__ double sm[];
  const int m = a.m_first + blockIdx.y;
  Op1DDev op = op_in, opp = op_in;   // boundary data at t_m (u_m) and t_{m-1} (conv of u_{m-1})
  op.gl = a.gl.v[m]; op.gr = a.gr.v[m];
  opp.gl = a.glp.v[m]; opp.gr = a.grp.v[m];
  const int p1 = op.p1, EB = eb_for(p1), T = (EB + 2) * p1, N = op.n;
  double* st = sm;
  double* ut = st + TabOff::size(p1);   // u_m tile
  double* ct = ut + T;                  // coefficient tile
  double* qt = ct + T;                  // flux tile
  double* pt = qt + T;                  // u_{m-1} tile
  const int ebase = blockIdx.x * EB;
  const double* um = a.u + (size_t)m * N;
  const double* up = m == 0 ? a.u0 : a.u + (size_t)(m - 1) * N;
  const int t = threadIdx.x, el = t / p1, i = t - el * p1;
  const bool own = el < EB && ebase + el < op.ne;
  const int gi = (ebase + el) * p1 + i;
  pdl_launch_dependents();
  load_tab(st, op.tab, p1);   // constant tables
  pdl_wait();                 // u, caches: the predecessor's output
  load_tile<DIR>(op, ut, um, ebase, EB);
  CoefDev phys{SISDC_COEF_PHYS, 0.0, nullptr};
  coef_tile<DIR>(op, phys, ct, ebase, EB);
  double dummy;
  const bool has_phys = op.nu_art != nullptr || phys_coef(op, 0, dummy);
  __syncthreads();
  // f = conv(u_m) + D[phys] u_m  (eval_rhs)
  double cm = own ? conv_node(op, st, ut, el, i) : 0.0;
  double f = cm;
  if (has_phys) {
    flux_q_tile<DIR>(op, st, ut, ct, qt, EB, ebase);
    __syncthreads();
    if (own) f = cm + (-sip_B_node<DIR>(op, st, ut, ct, qt, el, i, ebase + el) * st[TabOff::minv(p1) + i]);
    __syncthreads();
  }
  if (own) {
    flag_nonfinite(a.status, f, ebase + el);
    a.f[(size_t)m * N + gi] = f;
  }
  if (a.mode == 0) return;
  const double dtm = a.dts.v[m];
  if (dtm == 0.0) {                     // sdc.py:90-94
    if (own) {
      a.h1[(size_t)m * N + gi] = 0.0;
      if (a.h2) a.h2[(size_t)m * N + gi] = 0.0;
    }
    return;
  }
  // C_m frozen at u_{m-1}: SI for si1/si2, physical for euler (dgsem.py:365-366)
  CoefDev cmod = a.scheme == SISDC_EULER ? phys : CoefDev{SISDC_COEF_SI, dtm, up};
  coef_tile<DIR>(op, cmod, ct, ebase, EB);
  if (a.conv_prev == nullptr) load_tile<DIR>(opp, pt, up, ebase, EB);
  __syncthreads();
  flux_q_tile<DIR>(op, st, ut, ct, qt, EB, ebase);
  __syncthreads();
  if (!own) return;
  double d = -sip_B_node<DIR>(op, st, ut, ct, qt, el, i, ebase + el) * st[TabOff::minv(p1) + i];
  // conv_prev: one cached conv(u_{m-1}) vector per evaluated node (node stride N)
  double cp = a.conv_prev ? a.conv_prev[(size_t)(m - a.m_first) * N + gi] : conv_node(opp, st, pt, el, i);
  a.h1[(size_t)m * N + gi] = dtm * (cp + d);
  if (a.h2) a.h2[(size_t)m * N + gi] = dtm * (cm + d);
}

// rhs = base + dt*sum_i w_i f_old[i] (+ g) + dt_m conv(conv_in) - h_old   (sdc.py:218-237)
struct StageArgs {
  const double* base;
  const double* conv_in;
  double dt_m;
  const double* f_old;
  int M;
  W16 w;
  double dt;
  const double* g;
  const double* h;
  double* rhs;
  double* conv_out;
};

template <bool DIR>
__global__ void k_stage_rhs(Op1DDev op, StageArgs a) {
  extern __shared__ double sm[];
  const int p1 = op.p1, EB = eb_for(p1);
  double* st = sm;
  double* ut = st + TabOff::size(p1);
  const int ebase = blockIdx.x * EB;
  load_tab(st, op.tab, p1);
  load_tile<DIR>(op, ut, a.conv_in, ebase, EB);
  __syncthreads();
  const int t = threadIdx.x, el = t / p1, i = t - el * p1;
  if (!(el < EB && ebase + el < op.ne)) return;
  const int gi = (ebase + el) * p1 + i;
  double c = conv_node(op, st, ut, el, i);
  if (a.conv_out) a.conv_out[gi] = c;
  double q = 0.0;
  if (a.f_old) {
    double acc = 0.0;
    for (int j = 0; j < a.M; ++j) acc = fma(a.w.v[j], a.f_old[(size_t)j * op.n + gi], acc);
    q = a.dt * acc;
  }
  if (a.g) q = q + a.g[gi];
  double r = (a.base[gi] + q) + a.dt_m * c;
  if (a.h) r = r - a.h[gi];
  a.rhs[gi] = r;
}

// collocation defect (sdc.py:304-319): out = sign*(u - prev - dt W f) + add
struct DefectArgs {
  int M, incremental;
  W16 W[MAXM];
  double dt, sign;
  const double* u0;
  const double* u;
  const double* f;
  const double* add;
  double* out;
};
__global__ void k_defect(int N, DefectArgs a) {
  int gi = blockIdx.x * blockDim.x + threadIdx.x;
  int m = blockIdx.y;
  if (gi >= N) return;
  double acc = 0.0;
  for (int j = 0; j < a.M; ++j) acc = fma(a.W[m].v[j], a.f[(size_t)j * N + gi], acc);
  double prev = (a.incremental && m > 0) ? a.u[(size_t)(m - 1) * N + gi] : a.u0[gi];
  double F = (a.u[(size_t)m * N + gi] - prev) - a.dt * acc;
  double v = a.sign * F;
  if (a.add) v = v + a.add[(size_t)m * N + gi];
  a.out[(size_t)m * N + gi] = v;
}

// out = c0 v0 + c1 v1 + c2 v2 + c3 v3 (null vectors skipped), evaluated left to
// right as ((c0 v0 + c1 v1) + c2 v2) + c3 v3 -- the vector updates of the
// non-incremental sweep (sdc.py:245-284: running sum S, g differences)
struct LinArgs {
  double c[4];
  const double* v[4];
  double* out;
};
__global__ void k_lincomb(long long n, LinArgs a) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    double acc = a.v[0] ? a.c[0] * a.v[0][t] : 0.0;
#pragma unroll
    for (int k = 1; k < 4; ++k)
      if (a.v[k]) acc = acc + a.c[k] * a.v[k][t];
    a.out[t] = acc;
  }
}

// smooth_start (dgsem.py:574-589): every interior interface (and the periodic
// wrap) gets the mean of its two traces; blockIdx.y = node vector
__global__ void k_smooth_start(Op1DDev op, const double* __restrict__ u, double* __restrict__ out) {
  const int p1 = op.p1, P = p1 - 1, ne = op.ne;
  const int N = op.n * op.nc;   // op.n counts one component
  const size_t mo = (size_t)blockIdx.y * N;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N; t += gridDim.x * blockDim.x) {
    const int eg = t / p1, i = t - eg * p1;
    const int c = eg / ne, e = eg - c * ne;          // field-major (ncomp, ne, p1): every field on its own
    const size_t fo = mo + (size_t)c * ne * p1;
    double v = u[mo + t];
    if (i == P && (e + 1 < ne || op.bc == SISDC_PERIODIC)) {
      const int en = e + 1 < ne ? e + 1 : 0;
      v = 0.5 * (v + u[fo + (size_t)en * p1]);
    } else if (i == 0 && (e > 0 || op.bc == SISDC_PERIODIC)) {
      const int ep = e > 0 ? e - 1 : ne - 1;
      v = 0.5 * (u[fo + (size_t)ep * p1 + P] + v);
    }
    out[mo + t] = v;
  }
}

// ---------------------------------------------------------- transfers
// spatial single state: dir 0 interp c->f, 1 project f->c, 2 restrict f->c  (transfer.py:156-163)
__global__ void k_xfer_spatial(XferDev x, int dir, const double* __restrict__ in, double* __restrict__ out) {
  int nout = dir == 0 ? x.pf : x.pc, nin = dir == 0 ? x.pc : x.pf;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= x.ne * nout) return;
  int e = t / nout, i = t - e * nout;
  const double* Isp = x.tab + xo_Isp(x);
  const double* Psp = x.tab + xo_Psp(x);
  double acc = 0.0;
  for (int j = 0; j < nin; ++j) {
    const double* Rsp = x.tab + xo_Rsp(x);
    double a = dir == 0 ? Isp[i * x.pc + j] : (dir == 1 ? Psp[i * x.pf + j] : Rsp[i * x.pf + j]);
    acc = fma(a, in[e * nin + j], acc);
  }
  out[t] = acc;
}

// FAS restriction: r = g_f - F_f(u_f); v = P_t P_sp u_f; rr = R_t R_sp r  (mlsdc.py:84-101, transfer.py:335-342)
struct FasArgs {
  W16 Wf[MAXM];
  double dt;
  int incremental;
  const double* u0f;
  const double* uf;
  const double* ff;
  const double* gf;
  double* v;
  double* rr;
};
__global__ void k_fas_restrict(XferDev x, FasArgs a) {
  // one block per element; shared: r[Mf][pf], u[Mf][pf]
  extern __shared__ double sm[];
  const int e = blockIdx.x, pf = x.pf, pc = x.pc, Mf = x.Mf, Mc = x.Mc;
  const size_t Nf = (size_t)x.ne * pf, Nc = (size_t)x.ne * pc;
  double* su = sm;
  double* sr = su + Mf * pf;
  double* sps = sr + Mf * pf;        // spatially projected u   [Mf][pc]
  double* srs = sps + Mf * pc;       // spatially restricted r  [Mf][pc]
  for (int t = threadIdx.x; t < Mf * pf; t += blockDim.x) {
    int m = t / pf, i = t - m * pf;
    size_t gi = (size_t)e * pf + i;
    double acc = 0.0;
    for (int j = 0; j < Mf; ++j) acc = fma(a.Wf[m].v[j], a.ff[j * Nf + gi], acc);
    double um = a.uf[m * Nf + gi];
    double prev = (a.incremental && m > 0) ? a.uf[(m - 1) * Nf + gi] : a.u0f[gi];
    double F = (um - prev) - a.dt * acc;
    su[t] = um;
    sr[t] = a.gf ? a.gf[m * Nf + gi] - F : -F;
  }
  __syncthreads();
  const double* It = x.tab + xo_It(x);
  const double* Pt = x.tab + xo_Pt(x);
  const double* Isp = x.tab + xo_Isp(x);
  const double* Psp = x.tab + xo_Psp(x);
  const double* Rsp = x.tab + xo_Rsp(x);
  for (int t = threadIdx.x; t < Mf * pc; t += blockDim.x) {
    int m = t / pc, i = t - m * pc;
    double pu = 0.0, rr = 0.0;
    for (int j = 0; j < pf; ++j) {
      pu = fma(Psp[i * pf + j], su[m * pf + j], pu);
      rr = fma(Rsp[i * pf + j], sr[m * pf + j], rr);
    }
    sps[t] = pu;
    srs[t] = rr;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mc * pc; t += blockDim.x) {
    int mc = t / pc, i = t - mc * pc;
    double pv = 0.0, pr = 0.0;
    for (int mf = 0; mf < Mf; ++mf) {
      pv = fma(Pt[mc * Mf + mf], sps[mf * pc + i], pv);
      pr = fma(It[mf * Mc + mc], srs[mf * pc + i], pr);
    }
    size_t gi = (size_t)e * pc + i;
    a.v[mc * Nc + gi] = pv;
    a.rr[mc * Nc + gi] = pr;
  }
}

// out (Mc,Nc) = T S in (Mf,Nf): spatial first (transfer.py:335-342)
__global__ void k_xfer_down(XferDev x, int sdir, int tdir, const double* __restrict__ in, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int e = blockIdx.x, pf = x.pf, pc = x.pc, Mf = x.Mf, Mc = x.Mc;
  const size_t Nf = (size_t)x.ne * pf, Nc = (size_t)x.ne * pc;
  const double* It = x.tab + xo_It(x);
  const double* Pt = x.tab + xo_Pt(x);
  const double* Isp = x.tab + xo_Isp(x);
  const double* Psp = x.tab + xo_Psp(x);
  double* ss = sm;   // [Mf][pc]
  for (int t = threadIdx.x; t < Mf * pc; t += blockDim.x) {
    int m = t / pc, i = t - m * pc;
    double acc = 0.0;
    for (int j = 0; j < pf; ++j)
      acc = fma(sdir == 1 ? Psp[i * pf + j] : x.tab[xo_Rsp(x) + i * pf + j], in[m * Nf + (size_t)e * pf + j], acc);
    ss[t] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mc * pc; t += blockDim.x) {
    int mc = t / pc, i = t - mc * pc;
    double acc = 0.0;
    for (int mf = 0; mf < Mf; ++mf) acc = fma(tdir == 1 ? Pt[mc * Mf + mf] : It[mf * Mc + mc], ss[mf * pc + i], acc);
    out[mc * Nc + (size_t)e * pc + i] = acc;
  }
}

// uf (+)= I_sp I_t (uc - vc)   (transfer.py:344-352)
__global__ void k_xfer_interp(XferDev x, int accumulate, const double* __restrict__ uc,
                              const double* __restrict__ vc, double* __restrict__ uf) {
  extern __shared__ double sm[];
  const int e = blockIdx.x, pf = x.pf, pc = x.pc, Mf = x.Mf, Mc = x.Mc;
  const size_t Nf = (size_t)x.ne * pf, Nc = (size_t)x.ne * pc;
  double* sd = sm;              // [Mc][pc]
  double* stt = sd + Mc * pc;   // temporal interp [Mf][pc]
  const double* It = x.tab + xo_It(x);
  const double* Isp = x.tab + xo_Isp(x);
  for (int t = threadIdx.x; t < Mc * pc; t += blockDim.x) {
    int m = t / pc, i = t - m * pc;
    size_t gi = m * Nc + (size_t)e * pc + i;
    sd[t] = vc ? uc[gi] - vc[gi] : uc[gi];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mf * pc; t += blockDim.x) {
    int m = t / pc, i = t - m * pc;
    double acc = 0.0;
    for (int j = 0; j < Mc; ++j) acc = fma(It[m * Mc + j], sd[j * pc + i], acc);
    stt[t] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mf * pf; t += blockDim.x) {
    int m = t / pf, i = t - m * pf;
    double acc = 0.0;
    for (int j = 0; j < pc; ++j) acc = fma(Isp[i * pc + j], stt[m * pc + j], acc);
    size_t gi = m * Nf + (size_t)e * pf + i;
    uf[gi] = accumulate ? uf[gi] + acc : acc;
  }
}

// Persson-Peraire sensor (dgsem.py:537-559): one thread per element
__global__ void k_persson(Op1DDev op, const double* __restrict__ u, double kappa, double cs,
                          double* __restrict__ nu_art) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= op.ne) return;
  const int p1 = op.p1, P = p1 - 1;
  const double* Vinv = op.tab + TabOff::Vinv(p1);
  const double* ue = u + (size_t)e * p1;
  double tot = 0.0, top = 0.0, lam = 0.0;
  for (int k = 0; k < p1; ++k) {
    double mk = 0.0;
    for (int j = 0; j < p1; ++j) mk = fma(Vinv[k * p1 + j], ue[j], mk);
    double en = mk * mk * (2.0 / (2.0 * k + 1.0));
    tot += en;
    if (k == P) top = en;
    lam = fmax(lam, op.problem == SISDC_CNS1D   // sensor on rho, max_speed of the system (dgsem.py:551-553)
                        ? cns_speed(op, ue[k], u[op.n + (size_t)e * p1 + k], u[2 * (size_t)op.n + (size_t)e * p1 + k])
                        : wave_speed(op, ue[k]));
  }
  double s = tot > 0.0 ? log10(fmax(top, 1e-300) / tot) : -INFINITY;
  double s0 = -4.0 * log10((double)P);
  double eps0 = cs * op.dx * lam / P;
  double ramp = s < s0 - kappa ? 0.0 : (s > s0 + kappa ? 1.0 : 0.5 * (1.0 + sin(0.5 * M_PI * (s - s0) / kappa)));
  nu_art[e] = eps0 * ramp;
}

__global__ void k_reset_status(int* status, int reset_log) {
  if (threadIdx.x == 0) { status[0] = 0x7fffffff; status[1] = 0; if (reset_log) status[2] = 0; }
}

// ------------------------------------------------------------ launchers
static size_t tile_smem(int p1, int ntiles) { return sizeof(double) * (TabOff::size(p1) + ntiles * (eb_for(p1) + 2) * p1); }
static dim3 tile_grid(int ne, int p1, int ny = 1) { int EB = eb_for(p1); return dim3((ne + EB - 1) / EB, ny); }
static dim3 tile_block(int p1) { int t = eb_for(p1) * p1; return dim3((t + 31) / 32 * 32); }

int launch_apply_convection(Ctx* c, const Op1DDev& op, const double* u, double* out) {
  (op.bc == SISDC_DIRICHLET ? k_apply_convection<true> : k_apply_convection<false>)<<<tile_grid(op.ne, op.p1), tile_block(op.p1), tile_smem(op.p1, 1), c->stream>>>(op, u, out);
  return c->after_launch("apply_convection");
}
int launch_apply_diffusion(Ctx* c, const Op1DDev& op, CoefDev k, const double* u, double* out) {
  (op.bc == SISDC_DIRICHLET ? k_apply_diffusion<true> : k_apply_diffusion<false>)<<<tile_grid(op.ne, op.p1), tile_block(op.p1), tile_smem(op.p1, 3), c->stream>>>(op, k, u, out);
  return c->after_launch("apply_diffusion");
}
int launch_coef_field(Ctx* c, const Op1DDev& op, CoefDev k, double* out) {
  int n = op.ne * op.p1;
  k_coef_field<<<(n + 255) / 256, 256, 0, c->stream>>>(op, k, out);
  return c->after_launch("coef_field");
}
// bnd (nullable, Dirichlet): [4][M] outside states g_l(t_m), g_r(t_m), g_l(t_{m-1}), g_r(t_{m-1})
int launch_node_eval(Ctx* c, const Op1DDev& op, int mode, int scheme, int M, int m_first, int m_count,
                     const double* u0, const double* u, const double* conv_prev, const double* dts,
                     double* f, double* h1, double* h2, const double* bnd) {
  if (M > MAXM || m_first < 0 || m_count < 1 || m_first + m_count > M) return c->fail(SISDC_ERR_ARG, "bad node range");
  CacheArgs a{};
  a.u0 = u0; a.u = u; a.conv_prev = conv_prev; a.scheme = scheme; a.m_first = m_first; a.mode = mode;
  for (int j = 0; j < M; ++j) a.dts.v[j] = dts ? dts[j] : 0.0;
  for (int j = 0; j < M; ++j) {
    a.gl.v[j] = bnd ? bnd[j] : op.gl;
    a.gr.v[j] = bnd ? bnd[M + j] : op.gr;
    a.glp.v[j] = bnd ? bnd[2 * M + j] : op.gl;
    a.grp.v[j] = bnd ? bnd[3 * M + j] : op.gr;
  }
  a.f = f; a.h1 = h1; a.h2 = h2; a.status = c->d_status;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = tile_grid(op.ne, op.p1, m_count);
  cfg.blockDim = tile_block(op.p1);
  cfg.dynamicSmemBytes = tile_smem(op.p1, 4);
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = c->pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = op.bc == SISDC_DIRICHLET ? cudaLaunchKernelEx(&cfg, k_node_eval<true>, op, a)
                                           : cudaLaunchKernelEx(&cfg, k_node_eval<false>, op, a);
  if (e != cudaSuccess) return c->cuda(e, "node_eval launch");
  return c->after_launch("node_eval");
}
int launch_stage_rhs(Ctx* c, const Op1DDev& op, const double* base, const double* conv_in, double dt_m,
                     const double* f_old, int M, const double* w_row, double dt, const double* g,
                     const double* h, double* rhs, double* conv_out) {
  if (M > MAXM) return c->fail(SISDC_ERR_ARG, "too many collocation nodes");
  StageArgs a{};
  a.base = base; a.conv_in = conv_in; a.dt_m = dt_m; a.f_old = f_old; a.M = M; a.dt = dt;
  for (int j = 0; j < M; ++j) a.w.v[j] = (f_old && w_row) ? w_row[j] : 0.0;
  a.g = g; a.h = h; a.rhs = rhs; a.conv_out = conv_out;
  (op.bc == SISDC_DIRICHLET ? k_stage_rhs<true> : k_stage_rhs<false>)<<<tile_grid(op.ne, op.p1), tile_block(op.p1), tile_smem(op.p1, 1), c->stream>>>(op, a);
  return c->after_launch("stage_rhs");
}
int launch_defect(Ctx* c, int N, int M, const double* W, double dt, int incremental, const double* u0,
                  const double* u, const double* f, double sign, const double* add, double* out) {
  if (M > MAXM) return c->fail(SISDC_ERR_ARG, "too many collocation nodes");
  DefectArgs a{};
  a.M = M; a.incremental = incremental; a.dt = dt; a.sign = sign;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) a.W[i].v[j] = W[i * M + j];
  a.u0 = u0; a.u = u; a.f = f; a.add = add; a.out = out;
  k_defect<<<dim3((N + 255) / 256, M), 256, 0, c->stream>>>(N, a);
  return c->after_launch("collocation_defect");
}
int launch_lincomb(Ctx* c, long long n, const double* coef, const double* const* v, double* out) {
  LinArgs a{};
  for (int k = 0; k < 4; ++k) { a.c[k] = coef[k]; a.v[k] = v[k]; }
  a.out = out;
  long long nb = (n + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  if (nb < 1) nb = 1;
  k_lincomb<<<(unsigned)nb, 256, 0, c->stream>>>(n, a);
  return c->after_launch("lincomb");
}
int launch_smooth_start(Ctx* c, const Op1DDev& op, int M, const double* u, double* out) {
  if (u == out) return c->fail(SISDC_ERR_ARG, "smooth_start needs distinct input and output");
  k_smooth_start<<<dim3((op.n * op.nc + 255) / 256, M), 256, 0, c->stream>>>(op, u, out);
  return c->after_launch("smooth_start");
}
int launch_xfer_spatial(Ctx* c, const XferDev& x, int dir, const double* in, double* out) {
  int n = x.ne * (dir == 0 ? x.pf : x.pc);
  k_xfer_spatial<<<(n + 127) / 128, 128, 0, c->stream>>>(x, dir, in, out);
  return c->after_launch("xfer_spatial");
}
int launch_fas_restrict(Ctx* c, const XferDev& x, const double* Wf, double dt, int incremental, const double* u0f,
                        const double* uf, const double* ff, const double* gf, double* v, double* rr) {
  FasArgs a{};
  for (int i = 0; i < x.Mf; ++i)
    for (int j = 0; j < x.Mf; ++j) a.Wf[i].v[j] = Wf[i * x.Mf + j];
  a.dt = dt; a.incremental = incremental; a.u0f = u0f; a.uf = uf; a.ff = ff; a.gf = gf; a.v = v; a.rr = rr;
  size_t sm = sizeof(double) * (2 * x.Mf * x.pf + 2 * x.Mf * x.pc);
  k_fas_restrict<<<x.ne, 64, sm, c->stream>>>(x, a);
  return c->after_launch("fas_restrict");
}
int launch_xfer_down(Ctx* c, const XferDev& x, int sdir, int tdir, const double* in, double* out) {
  size_t sm = sizeof(double) * x.Mf * x.pc;
  k_xfer_down<<<x.ne, 64, sm, c->stream>>>(x, sdir, tdir, in, out);
  return c->after_launch("xfer_down");
}
int launch_xfer_interp(Ctx* c, const XferDev& x, int accumulate, const double* uc, const double* vc, double* uf) {
  size_t sm = sizeof(double) * (x.Mc * x.pc + x.Mf * x.pc);
  k_xfer_interp<<<x.ne, 64, sm, c->stream>>>(x, accumulate, uc, vc, uf);
  return c->after_launch("xfer_interp");
}
int launch_persson(Ctx* c, const Op1DDev& op, const double* u, double kappa, double cs, double* nu_art) {
  k_persson<<<(op.ne + 127) / 128, 128, 0, c->stream>>>(op, u, kappa, cs, nu_art);
  return c->after_launch("persson_viscosity");
}

}  // namespace sisdc
