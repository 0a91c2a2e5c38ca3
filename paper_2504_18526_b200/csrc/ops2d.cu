// 2-D sweep-path kernels (BASELINE configs 3-5): operators, fused sweep
// stages, tensor-product space-time transfers and the grid-persistent
// Chronopoulos-Gear PCG over HBM-resident vectors.
#include <cooperative_groups.h>
#include "sisdc_dev2d.cuh"
#include "sisdc_host.h"

namespace cg = cooperative_groups;

namespace sisdc {

template <int P1>
struct Blk {
  static constexpr int NN = P1 * P1;
  static constexpr int EB = NN >= 256 ? 1 : 256 / NN;   // elements per CTA
  static constexpr int NT = ((EB * NN + 31) / 32) * 32;  // threads per CTA
};

// shared-memory carve (doubles) for the element routines
template <int P1>
struct Sm2 {
  static constexpr int NN = P1 * P1, EB = Blk<P1>::EB;
  static constexpr int TAB = 4 * P1 * P1 + 3 * P1;
  static constexpr int FX = 0, FY = FX + EB * NC_MAX * NN;            // convection fluxes
  static constexpr int U = FY + EB * NC_MAX * NN, CS = U + EB * NN;    // SIP field / coefficient
  static constexpr int QX = CS + EB * NN, QY = QX + EB * NN;
  static constexpr int FC = QY + EB * NN;                              // face coeffs [EB][4][P1]
  static constexpr int FU = FC + EB * 4 * P1, FQ = FU + EB * 4 * P1;   // face u, q [EB][4][P1]
  static constexpr int ST = FQ + EB * 4 * P1;
  static constexpr int SIZE = ST + TAB;
};
enum { FR = 0, FL = 1, FT = 2, FB = 3 };   // right, left, top, bottom neighbour faces

struct Node2 {
  int el, nd, i, j, eg, ey, ex;
  bool valid;
};
template <int P1>
__device__ __forceinline__ Node2 node2(const Op2DDev& op, int tile) {
  Node2 n;
  const int t = threadIdx.x;
  n.el = t / Blk<P1>::NN;
  n.nd = t - n.el * Blk<P1>::NN;
  n.j = n.nd / P1;
  n.i = n.nd - n.j * P1;
  n.eg = tile * Blk<P1>::EB + n.el;
  n.valid = n.el < Blk<P1>::EB && n.eg < op.nex * op.ney;
  const int eg = n.valid ? n.eg : 0;
  n.ey = eg / op.nex;
  n.ex = eg - n.ey * op.nex;
  return n;
}

template <int P1>
__device__ __forceinline__ void load_tab2(double* st, const double* tab) {
  for (int t = threadIdx.x; t < Sm2<P1>::TAB; t += blockDim.x) st[t] = tab[t];
}

// ---------------------------------------------------------------- convection
// r[c] = conv(u) at this thread's node, all fields (dgsem.py:205-225 per direction)
template <int P1>
__device__ __forceinline__ void conv_block(const Op2DDev& op, double* sm, const double* __restrict__ u,
                                           const Node2& n, double* r) {
  constexpr int P = P1 - 1, NN = P1 * P1;
  const double* st = sm + Sm2<P1>::ST;
  const double* DTW = st + TabOff::DTW(P1);
  const double* w = st + TabOff::w(P1);
  double* FXs = sm + Sm2<P1>::FX + n.el * NC_MAX * NN;
  double* FYs = sm + Sm2<P1>::FY + n.el * NC_MAX * NN;
  double s[NC_MAX], f[NC_MAX];
  if (n.valid) {
    for (int c = 0; c < op.nc; ++c) s[c] = u[nidx(op, c, n.ey, n.ex, n.j, n.i)];
    flux2d(op, s, 0, f);
    for (int c = 0; c < op.nc; ++c) FXs[c * NN + n.nd] = f[c];
    flux2d(op, s, 1, f);
    for (int c = 0; c < op.nc; ++c) FYs[c * NN + n.nd] = f[c];
  }
  __syncthreads();
  if (n.valid) {
    double vx[NC_MAX], vy[NC_MAX];
    for (int c = 0; c < op.nc; ++c) {
      double ax = 0.0, ay = 0.0;
#pragma unroll
      for (int k = 0; k < P1; ++k) {
        ax = fma(DTW[n.i * P1 + k], FXs[c * NN + n.j * P1 + k], ax);
        ay = fma(DTW[n.j * P1 + k], FYs[c * NN + k * P1 + n.i], ay);
      }
      vx[c] = ax;
      vy[c] = ay;
    }
    double nb[NC_MAX], fh[NC_MAX];
    if (n.i == P) {   // right x-face: own (P,j) | right neighbour (0,j)
      const int exr = wrapi(n.ex + 1, op.nex);
      for (int c = 0; c < op.nc; ++c) nb[c] = u[nidx(op, c, n.ey, exr, n.j, 0)];
      rusanov2d(op, s, nb, 0, fh);
      for (int c = 0; c < op.nc; ++c) vx[c] -= fh[c];
    }
    if (n.i == 0) {   // left x-face: left neighbour (P,j) | own (0,j)
      const int exl = wrapi(n.ex - 1, op.nex);
      for (int c = 0; c < op.nc; ++c) nb[c] = u[nidx(op, c, n.ey, exl, n.j, P)];
      rusanov2d(op, nb, s, 0, fh);
      for (int c = 0; c < op.nc; ++c) vx[c] += fh[c];
    }
    if (n.j == P) {   // top y-face
      const int eyt = wrapi(n.ey + 1, op.ney);
      for (int c = 0; c < op.nc; ++c) nb[c] = u[nidx(op, c, eyt, n.ex, 0, n.i)];
      rusanov2d(op, s, nb, 1, fh);
      for (int c = 0; c < op.nc; ++c) vy[c] -= fh[c];
    }
    if (n.j == 0) {   // bottom y-face
      const int eyb = wrapi(n.ey - 1, op.ney);
      for (int c = 0; c < op.nc; ++c) nb[c] = u[nidx(op, c, eyb, n.ex, P, n.i)];
      rusanov2d(op, nb, s, 1, fh);
      for (int c = 0; c < op.nc; ++c) vy[c] += fh[c];
    }
    for (int c = 0; c < op.nc; ++c) r[c] = vx[c] * op.sx / w[n.i] + vy[c] * op.sy / w[n.j];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------- SIP
// Per field c of the state u (or a scalar-valued getter), the line SIP
// accumulators Bx, By at this node (dgsem.py:251-309 along x-lines and
// y-lines).  MODE 0: r[c] = apply_diffusion = -(Bx/(dx/2 w_i) + By/(dy/2 w_j));
// MODE 1: r[c] = (M + a B2) v with B2 = (dy/2 w_j) Bx + (dx/2 w_i) By.
// Source values: v(c, ey, ex, j, i) = src[nidx] * (scale ? scale[in-field node] : 1).
template <int P1, int MODE>
__device__ __forceinline__ void sip_block(const Op2DDev& op, double* sm, const CoefDev& k, const double* __restrict__ src,
                                          const double* __restrict__ scale, int nfields, double a, const Node2& n,
                                          double* r) {
  constexpr int P = P1 - 1, NN = P1 * P1;
  const double* st = sm + Sm2<P1>::ST;
  const double* D = st + TabOff::D(P1);
  const double* DTW = st + TabOff::DTW(P1);
  const double* w = st + TabOff::w(P1);
  double* U = sm + Sm2<P1>::U + n.el * NN;
  double* CS = sm + Sm2<P1>::CS + n.el * NN;
  double* QX = sm + Sm2<P1>::QX + n.el * NN;
  double* QY = sm + Sm2<P1>::QY + n.el * NN;
  double* FCo = sm + Sm2<P1>::FC + n.el * 4 * P1;
  double* FUo = sm + Sm2<P1>::FU + n.el * 4 * P1;
  double* FQo = sm + Sm2<P1>::FQ + n.el * 4 * P1;
  const int exr = wrapi(n.ex + 1, op.nex), exl = wrapi(n.ex - 1, op.nex);
  const int eyt = wrapi(n.ey + 1, op.ney), eyb = wrapi(n.ey - 1, op.ney);
  const long long fld = op.nn;
  auto in_field = [&](int ey, int ex, int j, int i) -> long long {
    return ((long long)ey * op.nex + ex) * NN + j * P1 + i;
  };
  auto val = [&](int c, int ey, int ex, int j, int i) -> double {
    const long long f = in_field(ey, ex, j, i);
    const double v = src[c * fld + f];
    return scale ? v * scale[f] : v;
  };
  double ci = 0.0;
  if (n.valid) {
    ci = coef2d(op, k, n.ey, n.ex, n.j, n.i);
    CS[n.nd] = ci;
    if (n.i == P) FCo[FR * P1 + n.j] = coef2d(op, k, n.ey, exr, n.j, 0);
    if (n.i == 0) FCo[FL * P1 + n.j] = coef2d(op, k, n.ey, exl, n.j, P);
    if (n.j == P) FCo[FT * P1 + n.i] = coef2d(op, k, eyt, n.ex, 0, n.i);
    if (n.j == 0) FCo[FB * P1 + n.i] = coef2d(op, k, eyb, n.ex, P, n.i);
  }
  for (int c = 0; c < nfields; ++c) {
    if (n.valid) U[n.nd] = val(c, n.ey, n.ex, n.j, n.i);
    __syncthreads();
    if (n.valid) {
      double gx = 0.0, gy = 0.0;
#pragma unroll
      for (int q = 0; q < P1; ++q) {
        gx = fma(D[n.i * P1 + q], U[n.j * P1 + q], gx);
        gy = fma(D[n.j * P1 + q], U[q * P1 + n.i], gy);
      }
      QX[n.nd] = ci * (op.sx * gx);
      QY[n.nd] = ci * (op.sy * gy);
      // neighbour face values and face fluxes (normal derivative of the neighbour)
      if (n.i == P) {
        double g = 0.0;
        for (int q = 0; q < P1; ++q) g = fma(D[q], val(c, n.ey, exr, n.j, q), g);
        FUo[FR * P1 + n.j] = val(c, n.ey, exr, n.j, 0);
        FQo[FR * P1 + n.j] = FCo[FR * P1 + n.j] * (op.sx * g);
      }
      if (n.i == 0) {
        double g = 0.0;
        for (int q = 0; q < P1; ++q) g = fma(D[P * P1 + q], val(c, n.ey, exl, n.j, q), g);
        FUo[FL * P1 + n.j] = val(c, n.ey, exl, n.j, P);
        FQo[FL * P1 + n.j] = FCo[FL * P1 + n.j] * (op.sx * g);
      }
      if (n.j == P) {
        double g = 0.0;
        for (int q = 0; q < P1; ++q) g = fma(D[q], val(c, eyt, n.ex, q, n.i), g);
        FUo[FT * P1 + n.i] = val(c, eyt, n.ex, 0, n.i);
        FQo[FT * P1 + n.i] = FCo[FT * P1 + n.i] * (op.sy * g);
      }
      if (n.j == 0) {
        double g = 0.0;
        for (int q = 0; q < P1; ++q) g = fma(D[P * P1 + q], val(c, eyb, n.ex, q, n.i), g);
        FUo[FB * P1 + n.i] = val(c, eyb, n.ex, P, n.i);
        FQo[FB * P1 + n.i] = FCo[FB * P1 + n.i] * (op.sy * g);
      }
    }
    __syncthreads();
    if (n.valid) {
      const int i = n.i, j = n.j;
      double Bx = 0.0, By = 0.0;
#pragma unroll
      for (int q = 0; q < P1; ++q) {
        Bx = fma(DTW[i * P1 + q], QX[j * P1 + q], Bx);
        By = fma(DTW[j * P1 + q], QY[q * P1 + i], By);
      }
      const double jr = U[j * P1 + P] - FUo[FR * P1 + j];
      const double jl = FUo[FL * P1 + j] - U[j * P1];
      const double cPx = CS[j * P1 + P], c0x = CS[j * P1];
      if (i == P) Bx += -(0.5 * (QX[j * P1 + P] + FQo[FR * P1 + j])) + (op.mux * (0.5 * (cPx + FCo[FR * P1 + j]))) * jr;
      if (i == 0) Bx -= -(0.5 * (FQo[FL * P1 + j] + QX[j * P1])) + (op.mux * (0.5 * (FCo[FL * P1 + j] + c0x))) * jl;
      Bx -= (op.sx * ((0.5 * cPx) * jr)) * D[P * P1 + i];
      Bx -= (op.sx * ((0.5 * c0x) * jl)) * D[i];
      const double jt = U[P * P1 + i] - FUo[FT * P1 + i];
      const double jb = FUo[FB * P1 + i] - U[i];
      const double cPy = CS[P * P1 + i], c0y = CS[i];
      if (j == P) By += -(0.5 * (QY[P * P1 + i] + FQo[FT * P1 + i])) + (op.muy * (0.5 * (cPy + FCo[FT * P1 + i]))) * jt;
      if (j == 0) By -= -(0.5 * (FQo[FB * P1 + i] + QY[i])) + (op.muy * (0.5 * (FCo[FB * P1 + i] + c0y))) * jb;
      By -= (op.sy * ((0.5 * cPy) * jt)) * D[P * P1 + j];
      By -= (op.sy * ((0.5 * c0y) * jb)) * D[j];
      const double hwx = 0.5 * op.dx * w[i], hwy = 0.5 * op.dy * w[j];
      if (MODE == 0) r[c] = -(Bx / hwx) - By / hwy;
      else r[c] = fma(a, fma(hwy, Bx, hwx * By), (hwx * hwy) * U[n.nd]);
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------- operator kernels
template <int P1>
__global__ void __launch_bounds__(256) k2_conv(Op2DDev op, const double* __restrict__ u, double* __restrict__ out) {
  extern __shared__ double sm[];
  load_tab2<P1>(sm + Sm2<P1>::ST, op.tab);
  __syncthreads();
  const Node2 n = node2<P1>(op, blockIdx.x);
  double r[NC_MAX];
  conv_block<P1>(op, sm, u, n, r);
  if (n.valid)
    for (int c = 0; c < op.nc; ++c) out[nidx(op, c, n.ey, n.ex, n.j, n.i)] = r[c];
}

template <int P1>
__global__ void __launch_bounds__(256) k2_sip(Op2DDev op, CoefDev k, const double* __restrict__ u, double* __restrict__ out) {
  extern __shared__ double sm[];
  load_tab2<P1>(sm + Sm2<P1>::ST, op.tab);
  __syncthreads();
  const Node2 n = node2<P1>(op, blockIdx.x);
  double r[NC_MAX];
  sip_block<P1, 0>(op, sm, k, u, nullptr, op.nc, 0.0, n, r);
  if (n.valid)
    for (int c = 0; c < op.nc; ++c) out[nidx(op, c, n.ey, n.ex, n.j, n.i)] = r[c];
}

template <int P1>
__global__ void k2_coef(Op2DDev op, CoefDev k, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= op.nn) return;
  const int NN = P1 * P1;
  const long long eg = t / NN;
  const int nd = (int)(t - eg * NN);
  out[t] = coef2d(op, k, (int)(eg / op.nex), (int)(eg % op.nex), nd / P1, nd % P1);
}

// node caches / eval_rhs for nodes m (blockIdx.y): mode 0 f only; mode 1 f, h1, h2
struct Cache2Args {
  const double* u0;
  const double* u;
  const double* conv_prev;
  int scheme, m_first, mode;
  double dts[16];
  double* f;
  double* h1;
  double* h2;
  int* status;
};
template <int P1>
__global__ void __launch_bounds__(256) k2_node_eval(Op2DDev op, Cache2Args a) {
  extern __shared__ double sm[];
  load_tab2<P1>(sm + Sm2<P1>::ST, op.tab);
  __syncthreads();
  const Node2 n = node2<P1>(op, blockIdx.x);
  const int m = a.m_first + blockIdx.y;
  const double* um = a.u + (size_t)m * op.n;
  const double* up = m == 0 ? a.u0 : a.u + (size_t)(m - 1) * op.n;
  double cm[NC_MAX], d[NC_MAX];
  conv_block<P1>(op, sm, um, n, cm);
  double ph;
  const bool has_phys = op.nu_art != nullptr || phys2d(op, 0, ph);
  const CoefDev phys{SISDC_COEF_PHYS, 0.0, nullptr};
  if (has_phys) sip_block<P1, 0>(op, sm, phys, um, nullptr, op.nc, 0.0, n, d);
  if (n.valid)
    for (int c = 0; c < op.nc; ++c) {
      const double f = has_phys ? cm[c] + d[c] : cm[c];
      if (!isfinite(f)) atomicMin(a.status, n.eg);
      a.f[(size_t)m * op.n + nidx(op, c, n.ey, n.ex, n.j, n.i)] = f;
    }
  if (a.mode == 0) return;
  const double dtm = a.dts[m];
  if (dtm == 0.0) {
    if (n.valid)
      for (int c = 0; c < op.nc; ++c) {
        const long long g = (size_t)m * op.n + nidx(op, c, n.ey, n.ex, n.j, n.i);
        a.h1[g] = 0.0;
        if (a.h2) a.h2[g] = 0.0;
      }
    return;
  }
  const CoefDev cmod = a.scheme == SISDC_EULER ? phys : CoefDev{SISDC_COEF_SI, dtm, up};
  sip_block<P1, 0>(op, sm, cmod, um, nullptr, op.nc, 0.0, n, d);
  double cp[NC_MAX];
  if (a.conv_prev) {
    if (n.valid)
      for (int c = 0; c < op.nc; ++c) cp[c] = a.conv_prev[nidx(op, c, n.ey, n.ex, n.j, n.i)];
  } else {
    conv_block<P1>(op, sm, up, n, cp);
  }
  if (n.valid)
    for (int c = 0; c < op.nc; ++c) {
      const long long g = (size_t)m * op.n + nidx(op, c, n.ey, n.ex, n.j, n.i);
      a.h1[g] = dtm * (cp[c] + d[c]);
      if (a.h2) a.h2[g] = dtm * (cm[c] + d[c]);
    }
}

struct Stage2Args {
  const double* base;
  const double* conv_in;
  double dt_m;
  const double* f_old;
  int M;
  double w[16];
  double dt;
  const double* g;
  const double* h;
  double* rhs;
  double* conv_out;
};
template <int P1>
__global__ void __launch_bounds__(256) k2_stage(Op2DDev op, Stage2Args a) {
  extern __shared__ double sm[];
  load_tab2<P1>(sm + Sm2<P1>::ST, op.tab);
  __syncthreads();
  const Node2 n = node2<P1>(op, blockIdx.x);
  double cv[NC_MAX];
  conv_block<P1>(op, sm, a.conv_in, n, cv);
  if (!n.valid) return;
  for (int c = 0; c < op.nc; ++c) {
    const long long gi = nidx(op, c, n.ey, n.ex, n.j, n.i);
    if (a.conv_out) a.conv_out[gi] = cv[c];
    double q = 0.0;
    if (a.f_old) {
      double acc = 0.0;
      for (int jj = 0; jj < a.M; ++jj) acc = fma(a.w[jj], a.f_old[(size_t)jj * op.n + gi], acc);
      q = a.dt * acc;
    }
    if (a.g) q = q + a.g[gi];
    double rr = (a.base[gi] + q) + a.dt_m * cv[c];
    if (a.h) rr = rr - a.h[gi];
    a.rhs[gi] = rr;
  }
}

// ---------------------------------------------------------------- transfers
// element slabs (nex*ney*ncomp) of p x p nodes; 1-D matrices applied in x and y
__device__ __forceinline__ double xf_spatial_coef(const Xfer2Dev& x, int dir, int a, int b) {
  const double* Isp = x.tab + 2 * x.Mf * x.Mc;
  const double* Psp = Isp + x.pf * x.pc;
  const double* Rsp = Psp + x.pf * x.pc;
  // dir 0: interp (pf x pc) = Isp[a][b]; 1: project (pc x pf) = Psp[a][b]; 2: restrict (pc x pf) = Rsp[a][b]
  return dir == 0 ? Isp[a * x.pc + b] : (dir == 1 ? Psp[a * x.pf + b] : Rsp[a * x.pf + b]);
}
// out_slab = S (x) S applied to one slab: out[ja][ia] = sum S[ja][jb] S[ia][ib] in[jb][ib]
__device__ __forceinline__ double sp2(const Xfer2Dev& x, int dir, const double* in, int nin, int ja, int ia) {
  double acc = 0.0;
  for (int jb = 0; jb < nin; ++jb) {
    double row = 0.0;
    for (int ib = 0; ib < nin; ++ib) row = fma(xf_spatial_coef(x, dir, ia, ib), in[jb * nin + ib], row);
    acc = fma(xf_spatial_coef(x, dir, ja, jb), row, acc);
  }
  return acc;
}

__global__ void k2x_spatial(Xfer2Dev x, int dir, const double* __restrict__ in, double* __restrict__ out) {
  const int nout = dir == 0 ? x.pf : x.pc, nin = dir == 0 ? x.pc : x.pf;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nsl = nout * nout;
  if (t >= (long long)x.nslab * nsl) return;
  const long long s = t / nsl;
  const int nd = (int)(t - s * nsl), ja = nd / nout, ia = nd % nout;
  out[t] = sp2(x, dir, in + s * nin * nin, nin, ja, ia);
}

// out (Mc, Nc) = T S in (Mf, Nf): spatial first; tdir 1 project (Pt), 2 restrict (It^T);
// sdir 1 project / 2 restrict.  Optionally in = g - F(u) built on the fly (FAS).
struct Fas2Args {
  double Wf[16 * 16];
  double dt;
  int incremental, build_residual;
  const double* u0f;
  const double* uf;
  const double* ff;
  const double* gf;
};
__global__ void k2x_down(Xfer2Dev x, int sdir, int tdir, const double* __restrict__ in, double* __restrict__ out,
                         long long Nf, long long Nc, int with_res, Fas2Args fa, double* __restrict__ out2) {
  // one block per slab; smem: fine slab values for all Mf nodes (two sets when with_res)
  extern __shared__ double sm[];
  const int s = blockIdx.x, pf = x.pf, pc = x.pc, Mf = x.Mf, Mc = x.Mc;
  const int nfs = pf * pf, ncs = pc * pc;
  double* su = sm;                 // [Mf][nfs]  (u or input)
  double* sr = su + Mf * nfs;      // [Mf][nfs]  residual (with_res)
  double* spu = sr + Mf * nfs;     // [Mf][ncs]  spatially transferred u
  double* spr = spu + Mf * ncs;    // [Mf][ncs]
  for (int t = threadIdx.x; t < Mf * nfs; t += blockDim.x) {
    const int m = t / nfs, nd = t - m * nfs;
    const long long gi = (long long)s * nfs + nd;
    if (with_res) {
      double acc = 0.0;
      for (int jj = 0; jj < Mf; ++jj) acc = fma(fa.Wf[m * Mf + jj], fa.ff[jj * Nf + gi], acc);
      const double um = fa.uf[m * Nf + gi];
      const double prev = (fa.incremental && m > 0) ? fa.uf[(m - 1) * Nf + gi] : fa.u0f[gi];
      const double F = (um - prev) - fa.dt * acc;
      su[t] = um;
      sr[t] = fa.gf ? fa.gf[m * Nf + gi] - F : -F;
    } else {
      su[t] = in[m * Nf + gi];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mf * ncs; t += blockDim.x) {
    const int m = t / ncs, nd = t - m * ncs, ja = nd / pc, ia = nd % pc;
    spu[t] = sp2(x, with_res ? 1 : sdir, su + m * nfs, pf, ja, ia);
    if (with_res) spr[t] = sp2(x, 2, sr + m * nfs, pf, ja, ia);
  }
  __syncthreads();
  const double* It = x.tab;
  const double* Pt = x.tab + Mf * Mc;
  for (int t = threadIdx.x; t < Mc * ncs; t += blockDim.x) {
    const int mc = t / ncs, nd = t - mc * ncs;
    double a1 = 0.0, a2 = 0.0;
    const int td1 = with_res ? 1 : tdir;
    for (int mf = 0; mf < Mf; ++mf) {
      a1 = fma(td1 == 1 ? Pt[mc * Mf + mf] : It[mf * Mc + mc], spu[mf * ncs + nd], a1);
      if (with_res) a2 = fma(It[mf * Mc + mc], spr[mf * ncs + nd], a2);
    }
    const long long go = mc * Nc + (long long)s * ncs + nd;
    out[go] = a1;
    if (with_res) out2[go] = a2;
  }
}

// uf (+)= I_sp(x) I_sp I_t (uc - vc)
__global__ void k2x_interp(Xfer2Dev x, int accumulate, const double* __restrict__ uc, const double* __restrict__ vc,
                           double* __restrict__ uf, long long Nf, long long Nc) {
  extern __shared__ double sm[];
  const int s = blockIdx.x, pf = x.pf, pc = x.pc, Mf = x.Mf, Mc = x.Mc;
  const int nfs = pf * pf, ncs = pc * pc;
  double* sd = sm;              // [Mc][ncs]
  double* stt = sd + Mc * ncs;  // [Mf][ncs]
  for (int t = threadIdx.x; t < Mc * ncs; t += blockDim.x) {
    const int m = t / ncs, nd = t - m * ncs;
    const long long gi = m * Nc + (long long)s * ncs + nd;
    sd[t] = vc ? uc[gi] - vc[gi] : uc[gi];
  }
  __syncthreads();
  const double* It = x.tab;
  for (int t = threadIdx.x; t < Mf * ncs; t += blockDim.x) {
    const int m = t / ncs, nd = t - m * ncs;
    double acc = 0.0;
    for (int jj = 0; jj < Mc; ++jj) acc = fma(It[m * Mc + jj], sd[jj * ncs + nd], acc);
    stt[t] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mf * nfs; t += blockDim.x) {
    const int m = t / nfs, nd = t - m * nfs, ja = nd / pf, ia = nd % pf;
    const double v = sp2(x, 0, stt + m * ncs, pc, ja, ia);
    const long long gi = m * Nf + (long long)s * nfs + nd;
    uf[gi] = accumulate ? uf[gi] + v : v;
  }
}

// ------------------------------------------------- grid-persistent 2-D PCG
// Chronopoulos-Gear Jacobi-PCG (oracle/cg.py) on HBM-resident vectors.  u is
// never stored: u = r * dinv on the fly.  Per iteration three grid-wide
// phases: A (stream p, s, x, r; partial (r,u), (r,r)), B (w = A u element
// matvec; partial (w,u)), R (block 0 reduces the partials in a fixed order ->
// alpha, beta, convergence), each followed by a grid barrier.
struct Cg2Args {
  Op2DDev op;
  CoefDev coef;
  double a;
  const double* rhs;
  double* x;
  double rtol2;
  int maxit;
  double* R;
  double* W;
  double* Pv;
  double* S;
  double* DINV;   // per in-field node
  double* Cf;     // per in-field node
  double* part;   // [gridDim][4]
  double* scal;   // [16]
  int* status;
  int* log_it;
  double* log_margin;
  int log_cap;
};

template <int P1>
__global__ void __launch_bounds__(256) k2_cg(Cg2Args A) {
  extern __shared__ double sm[];
  cg::grid_group grid = cg::this_grid();
  const Op2DDev& op = A.op;
  constexpr int NN = P1 * P1, P = P1 - 1;
  load_tab2<P1>(sm + Sm2<P1>::ST, op.tab);
  __syncthreads();
  const double* st = sm + Sm2<P1>::ST;
  const double* D2W = st + TabOff::D2W(P1);
  const double* D = st + TabOff::D(P1);
  const double* w = st + TabOff::w(P1);
  const int ntiles = (op.nex * op.ney + Blk<P1>::EB - 1) / Blk<P1>::EB;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double* red = sm;   // block reduction scratch (aliases FX, unused here) [32][4]
  auto block_sum = [&](double (&v)[3]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = 0; q < 3; ++q)
      for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    if (lane == 0)
      for (int q = 0; q < 3; ++q) red[wid * 4 + q] = v[q];
    __syncthreads();
    if (threadIdx.x == 0) {
      double t[3] = {0.0, 0.0, 0.0};
      for (int ww = 0; ww < nw; ++ww)
        for (int q = 0; q < 3; ++q) t[q] += red[ww * 4 + q];
      for (int q = 0; q < 3; ++q) A.part[blockIdx.x * 4 + q] = t[q];
    }
    __syncthreads();
  };
  auto mass = [&](long long f) -> double {   // lumped mass of in-field node f
    const int nd = (int)(f % NN);
    return (0.5 * op.dx * w[nd % P1]) * (0.5 * op.dy * w[nd / P1]);
  };
  // ---- setup 1: C, dinv per in-field node (closed-form diag of M + a B2), x0 = rhs, p = s = 0
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const Node2 n = node2<P1>(op, tile);
    double* CS = sm + Sm2<P1>::CS + n.el * NN;
    double* FCo = sm + Sm2<P1>::FC + n.el * 4 * P1;
    const int exr = wrapi(n.ex + 1, op.nex), exl = wrapi(n.ex - 1, op.nex);
    const int eyt = wrapi(n.ey + 1, op.ney), eyb = wrapi(n.ey - 1, op.ney);
    if (n.valid) {
      CS[n.nd] = coef2d(op, A.coef, n.ey, n.ex, n.j, n.i);
      if (n.i == P) FCo[FR * P1 + n.j] = coef2d(op, A.coef, n.ey, exr, n.j, 0);
      if (n.i == 0) FCo[FL * P1 + n.j] = coef2d(op, A.coef, n.ey, exl, n.j, P);
      if (n.j == P) FCo[FT * P1 + n.i] = coef2d(op, A.coef, eyt, n.ex, 0, n.i);
      if (n.j == 0) FCo[FB * P1 + n.i] = coef2d(op, A.coef, eyb, n.ex, P, n.i);
    }
    __syncthreads();
    if (n.valid) {
      const int i = n.i, j = n.j;
      double dx_ = 0.0, dy_ = 0.0;
      for (int q = 0; q < P1; ++q) {
        dx_ = fma(D2W[i * P1 + q], CS[j * P1 + q], dx_);
        dy_ = fma(D2W[j * P1 + q], CS[q * P1 + i], dy_);
      }
      dx_ *= op.sx;
      dy_ *= op.sy;
      if (i == P) dx_ += op.mux * (0.5 * (CS[j * P1 + P] + FCo[FR * P1 + j])) - op.sx * CS[j * P1 + P] * D[P * P1 + P];
      if (i == 0) dx_ += op.mux * (0.5 * (FCo[FL * P1 + j] + CS[j * P1])) + op.sx * CS[j * P1] * D[0];
      if (j == P) dy_ += op.muy * (0.5 * (CS[P * P1 + i] + FCo[FT * P1 + i])) - op.sy * CS[P * P1 + i] * D[P * P1 + P];
      if (j == 0) dy_ += op.muy * (0.5 * (FCo[FB * P1 + i] + CS[i])) + op.sy * CS[i] * D[0];
      const double hwx = 0.5 * op.dx * w[i], hwy = 0.5 * op.dy * w[j];
      const long long f = (long long)n.eg * NN + n.nd;
      A.Cf[f] = CS[n.nd];
      A.DINV[f] = 1.0 / (hwx * hwy + A.a * (hwy * dx_ + hwx * dy_));
    }
    __syncthreads();
  }
  for (long long t = gtid; t < op.n; t += nthr) {
    A.x[t] = A.rhs[t];
    A.Pv[t] = 0.0;
    A.S[t] = 0.0;
  }
  grid.sync();
  const CoefDev cfield{SISDC_COEF_FIELD, 0.0, A.Cf};
  // ---- setup 2: r0 = b - A x0 (b = M rhs), partial (b,b), #nonzero
  {
    double v[3] = {0.0, 0.0, 0.0};
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const Node2 n = node2<P1>(op, tile);
      double ax[NC_MAX];
      sip_block<P1, 1>(op, sm, cfield, A.x, nullptr, op.nc, A.a, n, ax);
      if (n.valid) {
        const double mi = (0.5 * op.dx * w[n.i]) * (0.5 * op.dy * w[n.j]);
        for (int c = 0; c < op.nc; ++c) {
          const long long g = nidx(op, c, n.ey, n.ex, n.j, n.i);
          const double b = mi * A.rhs[g];
          A.R[g] = b - ax[c];
          v[0] = fma(b, b, v[0]);
          v[1] += b != 0.0 ? 1.0 : 0.0;
        }
      }
    }
    block_sum(v);
  }
  grid.sync();
  // ---- setup 3: w0 = A u0, u0 = r0 dinv; partials gamma, delta, rho
  double bb = 0.0, nnz = 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) { t0 += A.part[b * 4]; t1 += A.part[b * 4 + 1]; }
    A.scal[8] = t0;
    A.scal[9] = t1;
  }
  grid.sync();   // the partial slots are reused below
  auto phase_B = [&]() {   // w = A u, u = r dinv; partial (w,u) into slot 1 (slots 0, 2 from phase A)
    double v[3] = {0.0, 0.0, 0.0};
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const Node2 n = node2<P1>(op, tile);
      double wv[NC_MAX];
      sip_block<P1, 1>(op, sm, cfield, A.R, A.DINV, op.nc, A.a, n, wv);
      if (n.valid) {
        const long long f = (long long)n.eg * NN + n.nd;
        const double di = A.DINV[f];
        for (int c = 0; c < op.nc; ++c) {
          const long long g = nidx(op, c, n.ey, n.ex, n.j, n.i);
          A.W[g] = wv[c];
          v[1] = fma(wv[c], A.R[g] * di, v[1]);
        }
      }
    }
    return v[1];
  };
  double v3[3] = {0.0, 0.0, 0.0};
  v3[1] = phase_B();
  for (long long t = gtid; t < op.n; t += nthr) {
    const double r = A.R[t], u = r * A.DINV[t % op.nn];
    v3[0] = fma(r, u, v3[0]);
    v3[2] = fma(r, r, v3[2]);
  }
  block_sum(v3);
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double t[3] = {0.0, 0.0, 0.0};
    for (int b = 0; b < (int)gridDim.x; ++b)
      for (int q = 0; q < 3; ++q) t[q] += A.part[b * 4 + q];
    A.scal[0] = t[0];              // gamma
    A.scal[1] = t[1];              // delta
    A.scal[2] = t[2];              // rho
    A.scal[3] = t[0] / t[1];       // alpha
    A.scal[4] = 0.0;               // beta
    A.scal[5] = 1.0 / t[0];        // 1/gamma
    A.scal[6] = 1.0 / A.scal[3];   // 1/alpha
  }
  grid.sync();
  bb = A.scal[8];
  nnz = A.scal[9];
  const double thr = A.rtol2 * bb;
  if (nnz == 0.0) {   // b == 0 -> zeros (dgsem.py:510-511)
    for (long long t = gtid; t < op.n; t += nthr) A.x[t] = 0.0;
    return;
  }
  int k = 0;
  bool ok = true;
  double rho = A.scal[2];
  while (rho > thr) {
    if (k >= A.maxit) { ok = false; break; }
    const double alpha = A.scal[3], beta = A.scal[4];
    // phase A: p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s
    double v[3] = {0.0, 0.0, 0.0};
    for (long long t = gtid; t < op.n; t += nthr) {
      const double di = A.DINV[t % op.nn];
      double r = A.R[t];
      const double p = fma(beta, A.Pv[t], r * di);
      const double s = fma(beta, A.S[t], A.W[t]);
      A.Pv[t] = p;
      A.S[t] = s;
      A.x[t] = fma(alpha, p, A.x[t]);
      r = fma(-alpha, s, r);
      A.R[t] = r;
      v[0] = fma(r, r * di, v[0]);
      v[2] = fma(r, r, v[2]);
    }
    grid.sync();
    v[1] = phase_B();
    block_sum(v);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double t[3] = {0.0, 0.0, 0.0};
      for (int b = 0; b < (int)gridDim.x; ++b)
        for (int q = 0; q < 3; ++q) t[q] += A.part[b * 4 + q];
      const double gn = t[0];
      const double be = gn * A.scal[5];
      const double al = gn / (t[1] - be * (gn * A.scal[6]));
      A.scal[0] = gn;
      A.scal[1] = t[1];
      A.scal[2] = t[2];
      A.scal[3] = al;
      A.scal[4] = be;
      A.scal[5] = 1.0 / gn;
      A.scal[6] = 1.0 / al;
    }
    grid.sync();
    ++k;
    rho = A.scal[2];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int idx = atomicAdd(&A.status[2], 1);
    if (idx < A.log_cap) {
      A.log_it[idx] = ok ? k : -1;
      A.log_margin[idx] = thr > 0.0 ? sqrt(rho / thr) : 0.0;
    }
    if (!ok) atomicAdd(&A.status[1], 1);
  }
}

// ------------------------------------------------------------- launchers
template <int P1>
static size_t smem2() { return sizeof(double) * Sm2<P1>::SIZE; }

#define SISDC_P1_SWITCH(p1, ...)                                 \
  switch (p1) {                                                  \
    case 2: { constexpr int P1 = 2; __VA_ARGS__; } break;        \
    case 3: { constexpr int P1 = 3; __VA_ARGS__; } break;        \
    case 4: { constexpr int P1 = 4; __VA_ARGS__; } break;        \
    case 5: { constexpr int P1 = 5; __VA_ARGS__; } break;        \
    case 6: { constexpr int P1 = 6; __VA_ARGS__; } break;        \
    case 7: { constexpr int P1 = 7; __VA_ARGS__; } break;        \
    case 8: { constexpr int P1 = 8; __VA_ARGS__; } break;        \
    case 9: { constexpr int P1 = 9; __VA_ARGS__; } break;        \
    default: return c->fail(SISDC_ERR_UNSUPPORTED, "2-D degree outside 1..8"); \
  }

template <int P1, typename K>
static void set_smem(K kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2<P1>());
}
template <int P1>
static dim3 grid2(const Op2DDev& op, int ny = 1) {
  return dim3((op.nex * op.ney + Blk<P1>::EB - 1) / Blk<P1>::EB, ny);
}

int launch2_conv(Ctx* c, const Op2DDev& op, const double* u, double* out) {
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_conv<P1>);
    k2_conv<P1><<<grid2<P1>(op), Blk<P1>::NT, smem2<P1>(), c->stream>>>(op, u, out);
  });
  return c->after_launch("k2_conv");
}
int launch2_sip(Ctx* c, const Op2DDev& op, CoefDev k, const double* u, double* out) {
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_sip<P1>);
    k2_sip<P1><<<grid2<P1>(op), Blk<P1>::NT, smem2<P1>(), c->stream>>>(op, k, u, out);
  });
  return c->after_launch("k2_sip");
}
int launch2_coef(Ctx* c, const Op2DDev& op, CoefDev k, double* out) {
  SISDC_P1_SWITCH(op.p1, {
    k2_coef<P1><<<(unsigned)((op.nn + 255) / 256), 256, 0, c->stream>>>(op, k, out);
  });
  return c->after_launch("k2_coef");
}
int launch2_node_eval(Ctx* c, const Op2DDev& op, int mode, int scheme, int M, int m_first, int m_count,
                      const double* u0, const double* u, const double* conv_prev, const double* dts,
                      double* f, double* h1, double* h2) {
  if (M > 16 || m_first < 0 || m_count < 1 || m_first + m_count > M) return c->fail(SISDC_ERR_ARG, "bad node range");
  Cache2Args a{};
  a.u0 = u0; a.u = u; a.conv_prev = conv_prev; a.scheme = scheme; a.m_first = m_first; a.mode = mode;
  for (int j = 0; j < M; ++j) a.dts[j] = dts ? dts[j] : 0.0;
  a.f = f; a.h1 = h1; a.h2 = h2; a.status = c->d_status;
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_node_eval<P1>);
    k2_node_eval<P1><<<grid2<P1>(op, m_count), Blk<P1>::NT, smem2<P1>(), c->stream>>>(op, a);
  });
  return c->after_launch("k2_node_eval");
}
int launch2_stage(Ctx* c, const Op2DDev& op, const double* base, const double* conv_in, double dt_m,
                  const double* f_old, int M, const double* w_row, double dt, const double* g,
                  const double* h, double* rhs, double* conv_out) {
  if (M > 16) return c->fail(SISDC_ERR_ARG, "too many collocation nodes");
  Stage2Args a{};
  a.base = base; a.conv_in = conv_in; a.dt_m = dt_m; a.f_old = f_old; a.M = M; a.dt = dt;
  for (int j = 0; j < M; ++j) a.w[j] = (f_old && w_row) ? w_row[j] : 0.0;
  a.g = g; a.h = h; a.rhs = rhs; a.conv_out = conv_out;
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_stage<P1>);
    k2_stage<P1><<<grid2<P1>(op), Blk<P1>::NT, smem2<P1>(), c->stream>>>(op, a);
  });
  return c->after_launch("k2_stage");
}

int launch2x_spatial(Ctx* c, const Xfer2Dev& x, int dir, const double* in, double* out) {
  const int nout = dir == 0 ? x.pf : x.pc;
  const long long tot = (long long)x.nslab * nout * nout;
  k2x_spatial<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(x, dir, in, out);
  return c->after_launch("k2x_spatial");
}
int launch2x_down(Ctx* c, const Xfer2Dev& x, int sdir, int tdir, const double* in, double* out) {
  const size_t sm = sizeof(double) * (2 * x.Mf * x.pf * x.pf + 2 * x.Mf * x.pc * x.pc);
  Fas2Args fa{};
  k2x_down<<<x.nslab, 128, sm, c->stream>>>(x, sdir, tdir, in, out, (long long)x.nslab * x.pf * x.pf,
                                            (long long)x.nslab * x.pc * x.pc, 0, fa, nullptr);
  return c->after_launch("k2x_down");
}
int launch2x_fas(Ctx* c, const Xfer2Dev& x, const double* Wf, double dt, int incremental, const double* u0f,
                 const double* uf, const double* ff, const double* gf, double* v, double* rr) {
  Fas2Args fa{};
  for (int i = 0; i < x.Mf * x.Mf; ++i) fa.Wf[i] = Wf[i];
  fa.dt = dt; fa.incremental = incremental; fa.u0f = u0f; fa.uf = uf; fa.ff = ff; fa.gf = gf;
  const size_t sm = sizeof(double) * (2 * x.Mf * x.pf * x.pf + 2 * x.Mf * x.pc * x.pc);
  k2x_down<<<x.nslab, 128, sm, c->stream>>>(x, 1, 1, nullptr, v, (long long)x.nslab * x.pf * x.pf,
                                            (long long)x.nslab * x.pc * x.pc, 1, fa, rr);
  return c->after_launch("k2x_fas");
}
int launch2x_interp(Ctx* c, const Xfer2Dev& x, int accumulate, const double* uc, const double* vc, double* uf) {
  const size_t sm = sizeof(double) * (x.Mc * x.pc * x.pc + x.Mf * x.pc * x.pc);
  k2x_interp<<<x.nslab, 128, sm, c->stream>>>(x, accumulate, uc, vc, uf, (long long)x.nslab * x.pf * x.pf,
                                              (long long)x.nslab * x.pc * x.pc);
  return c->after_launch("k2x_interp");
}

// CG workspace lives in the context, grown on demand (outside graph capture)
int launch2_cg(Ctx* c, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws,
               int nblocks) {
  Cg2Args A{};
  A.op = op; A.coef = k; A.a = a; A.rhs = rhs; A.x = x;
  A.rtol2 = c->rtol * c->rtol; A.maxit = c->maxit;
  double* p = ws;
  A.R = p; p += op.n;
  A.W = p; p += op.n;
  A.Pv = p; p += op.n;
  A.S = p; p += op.n;
  A.DINV = p; p += op.nn;
  A.Cf = p; p += op.nn;
  A.scal = p; p += 16;
  A.part = p;
  A.status = c->d_status; A.log_it = c->d_log_it; A.log_margin = c->d_log_margin; A.log_cap = c->log_cap;
  void* args[] = {&A};
  cudaError_t e = cudaSuccess;
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_cg<P1>);
    e = cudaLaunchCooperativeKernel((void*)k2_cg<P1>, dim3(nblocks), dim3(Blk<P1>::NT), args, smem2<P1>(), c->stream);
  });
  if (e != cudaSuccess) return c->cuda(e, "k2_cg cooperative launch");
  return c->after_launch("k2_cg");
}
// blocks for the cooperative CG: resident blocks x SMs, capped by the element tiles
int cg2_blocks(Ctx* c, const Op2DDev& op, int* nblocks) {
  int per_sm = 0, sms = 0;
  cudaError_t e = cudaSuccess;
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_cg<P1>);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_cg<P1>, Blk<P1>::NT, smem2<P1>());
    const int ntiles = (op.nex * op.ney + Blk<P1>::EB - 1) / Blk<P1>::EB;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    long long nb = (long long)per_sm * sms;
    if (nb > ntiles) nb = ntiles;
    if (nb < 1) nb = 1;
    *nblocks = (int)nb;
  });
  if (e != cudaSuccess) return c->cuda(e, "k2_cg occupancy");
  return SISDC_OK;
}

}  // namespace sisdc
