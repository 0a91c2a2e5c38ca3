// 2-D sweep-path kernels (BASELINE configs 3-5): operators, fused sweep
// stages, tensor-product space-time transfers and the grid-persistent
// Chronopoulos-Gear PCG over HBM-resident vectors.
#include <type_traits>
#include <cooperative_groups.h>
#include <vector>
#include <cstdlib>
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
  int el, nd, i, j, eg, ey, ex;   // eg: owned element index; ey: STORAGE row
  int es;                          // storage element index ey * nex + ex
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
  const int oy = eg / op.nex;
  n.ex = eg - oy * op.nex;
  n.ey = oy + op.row0;
  n.es = n.ey * op.nex + n.ex;
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
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) s[c] = u[nidx(op, c, n.ey, n.ex, n.j, n.i)];
    flux2d(op, s, 0, f);
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) FXs[c * NN + n.nd] = f[c];
    flux2d(op, s, 1, f);
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) FYs[c * NN + n.nd] = f[c];
  }
  __syncthreads();
  if (n.valid) {
    double vx[NC_MAX], vy[NC_MAX];
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) {
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
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) nb[c] = u[nidx(op, c, n.ey, exr, n.j, 0)];
      rusanov2d(op, s, nb, 0, fh);
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) vx[c] -= fh[c];
    }
    if (n.i == 0) {   // left x-face: left neighbour (P,j) | own (0,j)
      const int exl = wrapi(n.ex - 1, op.nex);
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) nb[c] = u[nidx(op, c, n.ey, exl, n.j, P)];
      rusanov2d(op, nb, s, 0, fh);
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) vx[c] += fh[c];
    }
    if (n.j == P) {   // top y-face
      const int eyt = ynb(op, n.ey, 1);
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) nb[c] = u[nidx(op, c, eyt, n.ex, 0, n.i)];
      rusanov2d(op, s, nb, 1, fh);
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) vy[c] -= fh[c];
    }
    if (n.j == 0) {   // bottom y-face
      const int eyb = ynb(op, n.ey, -1);
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) nb[c] = u[nidx(op, c, eyb, n.ex, P, n.i)];
      rusanov2d(op, nb, s, 1, fh);
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) vy[c] += fh[c];
    }
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) r[c] = vx[c] * op.sx / w[n.i] + vy[c] * op.sy / w[n.j];
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
  const int eyt = ynb(op, n.ey, 1), eyb = ynb(op, n.ey, -1);
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
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) out[nidx(op, c, n.ey, n.ex, n.j, n.i)] = r[c];
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
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) out[nidx(op, c, n.ey, n.ex, n.j, n.i)] = r[c];
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
__global__ void __launch_bounds__(256, 3) k2_node_eval(Op2DDev op, Cache2Args a) {
  extern __shared__ double sm[];
  load_tab2<P1>(sm + Sm2<P1>::ST, op.tab);
  __syncthreads();
  const Node2 n = node2<P1>(op, blockIdx.x);
  const int m = a.m_first + blockIdx.y;
  const double* um = a.u + (size_t)m * op.ns;
  const double* up = m == 0 ? a.u0 : a.u + (size_t)(m - 1) * op.ns;
  double cm[NC_MAX], d[NC_MAX];
  conv_block<P1>(op, sm, um, n, cm);
  double ph;
  const bool has_phys = op.nu_art != nullptr || phys2d(op, 0, ph);
  const CoefDev phys{SISDC_COEF_PHYS, 0.0, nullptr};
  if (has_phys) sip_block<P1, 0>(op, sm, phys, um, nullptr, op.nc, 0.0, n, d);
  if (n.valid)
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) {
      const double f = has_phys ? cm[c] + d[c] : cm[c];
      if (!isfinite(f)) atomicMin(a.status, (int)(op.e0 + n.eg));
      a.f[(size_t)m * op.ns + nidx(op, c, n.ey, n.ex, n.j, n.i)] = f;
    }
  if (a.mode == 0) return;
  double dtm = 0.0;   // static-index select (a dynamic index copies the parameter block to local memory)
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j == m) dtm = a.dts[j];
  if (dtm == 0.0) {
    if (n.valid)
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c) {
        const long long g = (size_t)m * op.ns + nidx(op, c, n.ey, n.ex, n.j, n.i);
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
#pragma unroll
      for (int c = 0; c < NC_MAX && c < op.nc; ++c)   // one cached vector per evaluated node (node stride op.ns)
        cp[c] = a.conv_prev[(size_t)(m - a.m_first) * op.ns + nidx(op, c, n.ey, n.ex, n.j, n.i)];
  } else {
    conv_block<P1>(op, sm, up, n, cp);
  }
  if (n.valid)
#pragma unroll
    for (int c = 0; c < NC_MAX && c < op.nc; ++c) {
      const long long g = (size_t)m * op.ns + nidx(op, c, n.ey, n.ex, n.j, n.i);
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
__global__ void __launch_bounds__(256, 3) k2_stage(Op2DDev op, Stage2Args a) {
  extern __shared__ double sm[];
  load_tab2<P1>(sm + Sm2<P1>::ST, op.tab);
  __syncthreads();
  const Node2 n = node2<P1>(op, blockIdx.x);
  double cv[NC_MAX];
  conv_block<P1>(op, sm, a.conv_in, n, cv);
  if (!n.valid) return;
#pragma unroll
  for (int c = 0; c < NC_MAX && c < op.nc; ++c) {
    const long long gi = nidx(op, c, n.ey, n.ex, n.j, n.i);
    if (a.conv_out) a.conv_out[gi] = cv[c];
    double q = 0.0;
    if (a.f_old) {
      double acc = 0.0;
      for (int jj = 0; jj < a.M; ++jj) acc = fma(a.w[jj], a.f_old[(size_t)jj * op.ns + gi], acc);
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
  double* tu = spr + Mf * ncs;     // [Mf][pf][pc] first (x) pass of the transfer
  double* tr = tu + Mf * pf * pc;
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
  // sum-factorised sp2 (two passes, the same operations in the same order):
  // T[jb][ia] = sum_ib S[ia][ib] in[jb][ib], out[ja][ia] = sum_jb S[ja][jb] T[jb][ia]
  const int sdu = with_res ? 1 : sdir;
  for (int t = threadIdx.x; t < Mf * pf * pc; t += blockDim.x) {
    const int m = t / (pf * pc), r = t - m * pf * pc, jb = r / pc, ia = r - jb * pc;
    double a1 = 0.0, a2 = 0.0;
    for (int ib = 0; ib < pf; ++ib) {
      a1 = fma(xf_spatial_coef(x, sdu, ia, ib), su[m * nfs + jb * pf + ib], a1);
      if (with_res) a2 = fma(xf_spatial_coef(x, 2, ia, ib), sr[m * nfs + jb * pf + ib], a2);
    }
    tu[t] = a1;
    if (with_res) tr[t] = a2;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mf * ncs; t += blockDim.x) {
    const int m = t / ncs, nd = t - m * ncs, ja = nd / pc, ia = nd % pc;
    double a1 = 0.0, a2 = 0.0;
    for (int jb = 0; jb < pf; ++jb) {
      a1 = fma(xf_spatial_coef(x, sdu, ja, jb), tu[(m * pf + jb) * pc + ia], a1);
      if (with_res) a2 = fma(xf_spatial_coef(x, 2, ja, jb), tr[(m * pf + jb) * pc + ia], a2);
    }
    spu[t] = a1;
    if (with_res) spr[t] = a2;
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
  double* tt = stt + Mf * ncs;  // [Mf][pc][pf] first (x) pass of the interpolation
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
  // sum-factorised sp2 (same operations, same order as the direct form)
  for (int t = threadIdx.x; t < Mf * pc * pf; t += blockDim.x) {
    const int m = t / (pc * pf), r = t - m * pc * pf, jb = r / pf, ia = r - jb * pf;
    double row = 0.0;
    for (int ib = 0; ib < pc; ++ib) row = fma(xf_spatial_coef(x, 0, ia, ib), stt[m * ncs + jb * pc + ib], row);
    tt[t] = row;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < Mf * nfs; t += blockDim.x) {
    const int m = t / nfs, nd = t - m * nfs, ja = nd / pf, ia = nd % pf;
    double v = 0.0;
    for (int jb = 0; jb < pc; ++jb) v = fma(xf_spatial_coef(x, 0, ja, jb), tt[(m * pc + jb) * pf + ia], v);
    const long long gi = m * Nf + (long long)s * nfs + nd;
    uf[gi] = accumulate ? uf[gi] + v : v;
  }
}

// ------------------------------------------------- grid-persistent 2-D PCG
// Chronopoulos-Gear Jacobi-PCG (oracle/cg.py) on HBM-resident vectors.  u is
// never stored: u = r * dinv on the fly.  Each iteration is two grid-wide
// phases, each closed by one grid barrier:
//   A  streaming update of p, s, x, r over (in-field node, field) with
//      16-byte accesses, partials (r,u) and (r,r);
//   B  w = A u over strip tiles (EB consecutive elements of one row) staged in
//      shared memory with their x/y neighbours by coalesced loads.  The
//      element contractions run per grid LINE (one thread = one x-row or
//      y-column of one element and field) with the reference-element
//      matrices in the constant bank, so the only shared-memory traffic is
//      the line itself (padded rows: conflict-free); partial (w,u).
// After the barrier every block reduces the per-block partials itself in one
// fixed order, so all blocks hold bitwise-identical alpha/beta and there is no
// separate reduction phase; partial slots alternate between iterations.
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
  double* U;      // u = r dinv, written by phase A (split solve: this iteration's u)
  double* U2;     // the other u buffer (split solve: the previous iteration's u, for p / x)
  double* Pv;
  double* S;
  double* DINV;   // per in-field node
  double* Cf;     // per in-field node
  double* part;   // [2][gridDim][4]
  double* scal;   // [16]
  int* status;
  int* log_it;
  double* log_margin;
  int log_cap;
  long long* timing;   // diagnostics: globaltimer stamps of blocks 0 and G-1 (nullable)
  int dbg;             // diagnostics only (SISDC_CG_DBG): 1 skip staging, 2 skip unit compute
  // partitioned (split) solve only: phase-B partial slots and the solve scalars
  double* part2;       // [gridDim][4]
  const struct CgPScal* sc;
  int px;              // split matvec: also advance p, x (p = u_prev + beta p, x += alpha p)
  int defer;           // split solve: p / x deferred to the matvec (P = 7), else in the update
  // fused single-pass iteration (k2_cgf): the second (r, s, w) buffers and the
  // setup-only mode of k2_cg (1: stop after setup 3 and leave the scalars in scal[2..7])
  double* R2;
  double* S2;
  double* W2;
  int mode;
  int bsel;            // single-pass mode on a partition: 0 every band, 1 interior bands (no ghost row
                       // touched: runs while the halo is in flight), 2 the first and last band
};

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// reference-element matrices per P1 in the constant bank: D | DTW | D2W | w
__host__ __device__ constexpr int ctab_off(int p1) {
  int o = 0;
  for (int p = 2; p < p1; ++p) o += 3 * p * p + p;
  return o;
}
__constant__ double c_tab2[ctab_off(10)];
template <int P1>
struct CT {
  static constexpr int D = ctab_off(P1), DTW = D + P1 * P1, D2W = DTW + P1 * P1, W = D2W + P1 * P1;
};

// shared-memory carve (doubles) of the CG strip tiles; element rows padded to
// P1+1 so line accesses are bank-conflict free
template <int P1, int NC>
struct CgSm {
  static constexpr int NN = P1 * P1, EB = Blk<P1>::EB, RP = P1 + 1, NP = P1 * RP;
  static constexpr int NS = 3 * EB + 2;   // slots: 0 left, 1..cnt own, cnt+1 right, EB+2.. above, 2EB+2.. below
  static constexpr int U = 0;                                   // [NC][NS][NP]
  static constexpr int C = U + NC * NS * NP;                    // [NS][NP] coefficient
  static constexpr int QX = C + NS * NP, QY = QX + NC * EB * NP;   // [NC][EB][NP]
  static constexpr int BX = QY + NC * EB * NP, BY = BX + NC * EB * NP;
  static constexpr int FQ = BY + NC * EB * NP;                  // [NC][EB][4][P1] neighbour face fluxes
  static constexpr int END0 = FQ + NC * EB * 4 * P1;
  // P1 = 8 runs phase B warp-per-element: 8 warps x Wpe<NC>::WARP (defined below)
  static constexpr int WPE = 8 * (2 * 80 + 2 * 4 * 64 + 2 * 80 + 64 + 160 + 32 + 64);
  static constexpr int END1 = P1 == 8 ? WPE : END0;
  static constexpr int RED = END1 > Sm2<P1>::FU ? END1 : Sm2<P1>::FU;   // [32][4]; setup scratch below
  static constexpr int SIZE = RED + 128;
};

// asynchronous 8-byte global->shared copy (LDGSTS) and its completion wait
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// One strip tile of w = (M + a B2) v (B2 as in sip_block MODE 1, same operation
// order), v = src * scale (scale per in-field node, or null).  epi(g, w, v) per
// own node and field, g the global index.
template <int P1, int NC, typename Epi>
__device__ __forceinline__ void cg_tile(const Op2DDev& op, double* sm, int tile, int tpr, const double* src,
                                        const double* scale, const double* Cf, double a, Epi&& epi) {
  using L = CgSm<P1, NC>;
  using T = CT<P1>;
  constexpr int NN = P1 * P1, EB = Blk<P1>::EB, P = P1 - 1, RP = L::RP, NP = L::NP, NS = L::NS;
  constexpr int nc = NC;
  const long long fld = op.nn;
  const int oy = tile / tpr, ex0 = (tile - oy * tpr) * EB, ey = oy + op.row0;
  const int cnt = min(EB, op.nex - ex0);
  // tile-variant zero (tile < 2^30): keeps the constant-bank matrix loads inside the
  // tile loop (uniform-register operands) instead of hoisted into the register file
  const double* ct = c_tab2 + (tile >> 30);
  const long long rowm = (long long)ey * op.nex;
  const long long rowt = (long long)ynb(op, ey, 1) * op.nex;
  const long long rowb = (long long)ynb(op, ey, -1) * op.nex;
  const int exl = wrapi(ex0 - 1, op.nex), exr = wrapi(ex0 + cnt, op.nex);
  __syncthreads();   // the previous tile's readers are done with the buffers
  // ---- stage: strip + x-halo (slots 0..cnt+1), rows above / below (contiguous
  // runs) by asynchronous global->shared copies, all in flight at once; the
  // scale (dinv) is applied in place by the thread that copied the entry
  {
    constexpr int NT = Blk<P1>::NT, KMAX = ((3 * EB + 2) * NN + NT - 1) / NT;
    const int n1 = (cnt + 2) * NN, ntot = n1 + 2 * cnt * NN;
    double sv[KMAX];
    int ov[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      const int t = threadIdx.x + k * NT;
      ov[k] = -1;
      if (t < ntot) {
        long long f;
        int slot, nd;
        if (t < n1) {
          const int s = t / NN;
          nd = t - s * NN;
          slot = s;
          f = (rowm + (s == 0 ? exl : (s == cnt + 1 ? exr : ex0 + s - 1))) * NN + nd;
        } else {
          const int tt = t - n1;
          const bool up = tt < cnt * NN;
          const int t2 = up ? tt : tt - cnt * NN;
          const int el = t2 / NN;
          nd = t2 - el * NN;
          slot = (up ? EB + 2 : 2 * EB + 2) + el;
          f = ((up ? rowt : rowb) + ex0) * NN + t2;
        }
        const int jj = nd / P1;
        const int o = slot * NP + jj * RP + (nd - jj * P1);
        ov[k] = o;
        cp_async8(sm + L::C + o, Cf + f);
#pragma unroll
        for (int c = 0; c < NC; ++c) cp_async8(sm + L::U + c * NS * NP + o, src + c * fld + f);
        if (scale) sv[k] = scale[f];
      }
    }
    cp_async_wait_all();
    if (scale) {
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (ov[k] >= 0) {
#pragma unroll
          for (int c = 0; c < NC; ++c) sm[L::U + c * NS * NP + ov[k]] *= sv[k];
        }
    }
  }
  __syncthreads();
  const int nl = nc * cnt * P1;   // element lines per direction
  // ---- fluxes q = C s D v along every own x-row / y-column; neighbour face fluxes
  for (int it = threadIdx.x; it < 2 * nl; it += blockDim.x) {
    const bool yd = it >= nl;
    const int r = yd ? it - nl : it;
    const int c = r / (cnt * P1), rem = r - c * cnt * P1, el = rem / P1, l = rem - el * P1;
    const int base = yd ? l : l * RP, stride = yd ? RP : 1;
    const double* U = sm + L::U + (c * NS + el + 1) * NP + base;
    const double* Cc = sm + L::C + (el + 1) * NP + base;
    double* Q = sm + (yd ? L::QY : L::QX) + (c * EB + el) * NP + base;
    const double s = yd ? op.sy : op.sx;
    double u[P1];
#pragma unroll
    for (int q = 0; q < P1; ++q) u[q] = U[q * stride];
#pragma unroll
    for (int i = 0; i < P1; ++i) {
      double g = 0.0;
#pragma unroll
      for (int q = 0; q < P1; ++q) g = fma(ct[T::D + i * P1 + q], u[q], g);
      Q[i * stride] = Cc[i * stride] * (s * g);
    }
  }
  for (int it = threadIdx.x; it < 4 * nl; it += blockDim.x) {
    const int c = it / (cnt * 4 * P1), rem = it - c * cnt * 4 * P1, el = rem / (4 * P1), r2 = rem - el * 4 * P1;
    const int face = r2 / P1, k = r2 - face * P1;
    const double* Un = sm + L::U + c * NS * NP;
    double g = 0.0, cf, s;
    if (face == FR) {          // right neighbour, row k, derivative at its node (k,0)
      const double* row = Un + (el + 2) * NP + k * RP;
#pragma unroll
      for (int q = 0; q < P1; ++q) g = fma(ct[T::D + q], row[q], g);
      cf = sm[L::C + (el + 2) * NP + k * RP];
      s = op.sx;
    } else if (face == FL) {   // left neighbour, row k, at its node (k,P)
      const double* row = Un + el * NP + k * RP;
#pragma unroll
      for (int q = 0; q < P1; ++q) g = fma(ct[T::D + P * P1 + q], row[q], g);
      cf = sm[L::C + el * NP + k * RP + P];
      s = op.sx;
    } else if (face == FT) {   // element above, column k, at its node (0,k)
      const double* col = Un + (EB + 2 + el) * NP + k;
#pragma unroll
      for (int q = 0; q < P1; ++q) g = fma(ct[T::D + q], col[q * RP], g);
      cf = sm[L::C + (EB + 2 + el) * NP + k];
      s = op.sy;
    } else {                   // element below, column k, at its node (P,k)
      const double* col = Un + (2 * EB + 2 + el) * NP + k;
#pragma unroll
      for (int q = 0; q < P1; ++q) g = fma(ct[T::D + P * P1 + q], col[q * RP], g);
      cf = sm[L::C + (2 * EB + 2 + el) * NP + P * RP + k];
      s = op.sy;
    }
    sm[L::FQ + ((c * EB + el) * 4 + face) * P1 + k] = cf * (s * g);
  }
  __syncthreads();
  // ---- SIP accumulators per line: volume DTW q, face terms, adjoint lifting
  for (int it = threadIdx.x; it < 2 * nl; it += blockDim.x) {
    const bool yd = it >= nl;
    const int r = yd ? it - nl : it;
    const int c = r / (cnt * P1), rem = r - c * cnt * P1, el = rem / P1, l = rem - el * P1;
    const int base = yd ? l : l * RP, stride = yd ? RP : 1;
    const double* Q = sm + (yd ? L::QY : L::QX) + (c * EB + el) * NP + base;
    const double* U = sm + L::U + (c * NS + el + 1) * NP + base;
    const double* Cc = sm + L::C + (el + 1) * NP + base;
    const double* fq = sm + L::FQ + (c * EB + el) * 4 * P1;
    double q[P1];
#pragma unroll
    for (int k = 0; k < P1; ++k) q[k] = Q[k * stride];
    const double cP = Cc[P * stride], c0 = Cc[0];
    double jp, jm, fcp, fcm, qp, qm, mu, s;
    if (!yd) {   // row l: right face at (l,P), left face at (l,0)
      const int ub = (c * NS) * NP + l * RP;
      jp = U[P] - sm[L::U + ub + (el + 2) * NP];
      jm = sm[L::U + ub + el * NP + P] - U[0];
      fcp = sm[L::C + (el + 2) * NP + l * RP];
      fcm = sm[L::C + el * NP + l * RP + P];
      qp = fq[FR * P1 + l];
      qm = fq[FL * P1 + l];
      mu = op.mux;
      s = op.sx;
    } else {     // column l: top face at (P,l), bottom face at (0,l)
      const int ub = (c * NS) * NP + l;
      jp = U[P * RP] - sm[L::U + ub + (EB + 2 + el) * NP];
      jm = sm[L::U + ub + (2 * EB + 2 + el) * NP + P * RP] - U[0];
      fcp = sm[L::C + (EB + 2 + el) * NP + l];
      fcm = sm[L::C + (2 * EB + 2 + el) * NP + P * RP + l];
      qp = fq[FT * P1 + l];
      qm = fq[FB * P1 + l];
      mu = op.muy;
      s = op.sy;
    }
    const double fp = -(0.5 * (q[P] + qp)) + (mu * (0.5 * (cP + fcp))) * jp;
    const double fm = -(0.5 * (qm + q[0])) + (mu * (0.5 * (fcm + c0))) * jm;
    const double lp = s * ((0.5 * cP) * jp), lm = s * ((0.5 * c0) * jm);
    double* Bo = sm + (yd ? L::BY : L::BX) + (c * EB + el) * NP + base;
#pragma unroll
    for (int i = 0; i < P1; ++i) {
      double b = 0.0;
#pragma unroll
      for (int k = 0; k < P1; ++k) b = fma(ct[T::DTW + i * P1 + k], q[k], b);
      if (i == P) b += fp;
      if (i == 0) b -= fm;
      b -= lp * ct[T::D + P * P1 + i];
      Bo[i * stride] = b - lm * ct[T::D + i];
    }
  }
  __syncthreads();
  // ---- combine per node: w = a (hwy Bx + hwx By) + hwx hwy v
  const int el = threadIdx.x / NN;
  if (el >= cnt) return;
  const int nd = threadIdx.x - el * NN, j = nd / P1, i = nd - j * P1, o = el * NP + j * RP + i;
  const double hwx = 0.5 * op.dx * ct[T::W + i], hwy = 0.5 * op.dy * ct[T::W + j];
  const long long g0 = (rowm + ex0 + el) * NN + nd;
  for (int c = 0; c < nc; ++c) {
    const double Bx = sm[L::BX + c * EB * NP + o], By = sm[L::BY + c * EB * NP + o];
    const double v = sm[L::U + (c * NS + 1) * NP + o];
    epi(c * fld + g0, fma(a, fma(hwy, Bx, hwx * By), (hwx * hwy) * v), v);
  }
}

// P = 3 (P1 = 4) CG matvec, register-resident: a half-warp owns an element
// (lane = node, j = t/4, i = t%4), all fields.  The element, its four face
// neighbours and the coefficient are read straight from global memory (one
// coalesced 128-byte run per element and field); every line contraction
// reaches its operands by warp shuffles, so there is no shared memory and no
// block barrier (cg_tile staged 3 EB + 2 elements per tile behind
// __syncthreads and was latency bound).  Same operations in the same order as
// cg_tile, so the results are bitwise identical.  epi(g, w, v) per own node.
__device__ __forceinline__ double pick4(const double* v, int c) {   // register select, no local memory
  return c == 0 ? v[0] : c == 1 ? v[1] : c == 2 ? v[2] : v[3];
}
template <int NC, typename Epi>
__device__ __forceinline__ void wph_phase(const Op2DDev& op, const double* src, const double* Cf, double a, Epi&& epi) {
  constexpr int P1 = 4, P = 3, NN = 16;
  using T = CT<P1>;
  // D | DTW in shared memory (lane-varying rows; registers are the limit here)
  __shared__ double sT[32];
  if (threadIdx.x < 32) sT[threadIdx.x] = op.tab[threadIdx.x];   // TabOff: D (16) then DTW (16)
  __syncthreads();
  const int lane = threadIdx.x & 31, t = lane & 15, j = t >> 2, i = t & 3, hb = lane & 16;
  const double hwx = 0.5 * op.dx * op.tab[TabOff::w(P1) + i], hwy = 0.5 * op.dy * op.tab[TabOff::w(P1) + j];
  auto sh = [&](double v, int src_t) { return __shfl_sync(0xffffffffu, v, hb | src_t); };
  const int ne = op.nex * op.ney;
  const int nw = (blockDim.x >> 5) * gridDim.x, w0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nn = op.nn;
  for (int pr = w0; 2 * pr < ne; pr += nw) {
    const int e = 2 * pr + (hb ? 1 : 0);
    const bool valid = e < ne;
    const int ee = valid ? e : ne - 1;
    const int oy = ee / op.nex, ex = ee - oy * op.nex, ey = oy + op.row0;
    const int exr = ex + 1 == op.nex ? 0 : ex + 1, exl = ex == 0 ? op.nex - 1 : ex - 1;
    const int eyt = ynb(op, ey, 1), eyb = ynb(op, ey, -1);
    const long long eo = ((long long)ey * op.nex + ex) * NN;
    const long long oR = ((long long)ey * op.nex + exr) * NN, oL = ((long long)ey * op.nex + exl) * NN;
    const long long oT = ((long long)eyt * op.nex + ex) * NN, oB = ((long long)eyb * op.nex + ex) * NN;
    // coefficient: own node, and the neighbours' face nodes of this lane's row / column
    const double cc = Cf[eo + t];
    const double fcp_x = Cf[oR + j * P1], fcm_x = Cf[oL + j * P1 + P];
    const double fcp_y = Cf[oT + i], fcm_y = Cf[oB + P * P1 + i];
    const double cPx = sh(cc, j * 4 + P), c0x = sh(cc, j * 4), cPy = sh(cc, P * 4 + i), c0y = sh(cc, i);
    // the next field's five loads are issued before this field's shuffle / FMA chain (the chain
    // consumed its own loads at once: 60% of the samples waited on them at 25% occupancy)
    double pv = src[eo + t], pR = src[oR + t], pL = src[oL + t], pT = src[oT + t], pB = src[oB + t];
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const double v = pv, nR = pR, nL = pL, nT = pT, nB = pB;
      if (c + 1 < NC) {
        const double* sn = src + (c + 1) * nn;
        pv = sn[eo + t]; pR = sn[oR + t]; pL = sn[oL + t]; pT = sn[oT + t]; pB = sn[oB + t];
      }
      // q = C s D u along the row (x) and the column (y) of this node
      double gx = 0.0, gy = 0.0, row0, rowP, col0, colP;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double r_ = sh(v, j * 4 + q), c_ = sh(v, q * 4 + i);
        gx = fma(sT[i * P1 + q], r_, gx);
        gy = fma(sT[j * P1 + q], c_, gy);
        if (q == 0) { row0 = r_; col0 = c_; }
        if (q == P) { rowP = r_; colP = c_; }
      }
      const double qx = cc * (op.sx * gx), qy = cc * (op.sy * gy);
      // neighbour face fluxes of this row / column and the neighbour face values
      double gR = 0.0, gL = 0.0, gT = 0.0, gB = 0.0, uRf = 0.0, uLf = 0.0, uTf = 0.0, uBf = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double r_ = sh(nR, j * 4 + q), l_ = sh(nL, j * 4 + q);
        const double t_ = sh(nT, q * 4 + i), b_ = sh(nB, q * 4 + i);
        gR = fma(c_tab2[T::D + q], r_, gR);
        gL = fma(c_tab2[T::D + P * P1 + q], l_, gL);
        gT = fma(c_tab2[T::D + q], t_, gT);
        gB = fma(c_tab2[T::D + P * P1 + q], b_, gB);
        if (q == 0) { uRf = r_; uTf = t_; }
        if (q == P) { uLf = l_; uBf = b_; }
      }
      const double qp_x = fcp_x * (op.sx * gR), qm_x = fcm_x * (op.sx * gL);
      const double qp_y = fcp_y * (op.sy * gT), qm_y = fcm_y * (op.sy * gB);
      double bx = 0.0, by = 0.0, qx0, qxP, qy0, qyP;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double a_ = sh(qx, j * 4 + k), b_ = sh(qy, k * 4 + i);
        bx = fma(sT[16 + i * P1 + k], a_, bx);
        by = fma(sT[16 + j * P1 + k], b_, by);
        if (k == 0) { qx0 = a_; qy0 = b_; }
        if (k == P) { qxP = a_; qyP = b_; }
      }
      // x-line (row j) and y-line (column i) face and adjoint-lift terms
      const double jpx = rowP - uRf, jmx = uLf - row0;
      const double fpx = -(0.5 * (qxP + qp_x)) + (op.mux * (0.5 * (cPx + fcp_x))) * jpx;
      const double fmx = -(0.5 * (qm_x + qx0)) + (op.mux * (0.5 * (fcm_x + c0x))) * jmx;
      const double lpx = op.sx * ((0.5 * cPx) * jpx), lmx = op.sx * ((0.5 * c0x) * jmx);
      const double jpy = colP - uTf, jmy = uBf - col0;
      const double fpy = -(0.5 * (qyP + qp_y)) + (op.muy * (0.5 * (cPy + fcp_y))) * jpy;
      const double fmy = -(0.5 * (qm_y + qy0)) + (op.muy * (0.5 * (fcm_y + c0y))) * jmy;
      const double lpy = op.sy * ((0.5 * cPy) * jpy), lmy = op.sy * ((0.5 * c0y) * jmy);
      if (i == P) bx += fpx;
      if (i == 0) bx -= fmx;
      bx -= lpx * c_tab2[T::D + P * P1 + i];
      bx = bx - lmx * c_tab2[T::D + i];
      if (j == P) by += fpy;
      if (j == 0) by -= fmy;
      by -= lpy * c_tab2[T::D + P * P1 + j];
      by = by - lmy * c_tab2[T::D + j];
      if (valid) epi(c * nn + eo + t, fma(a, fma(hwy, bx, hwx * by), (hwx * hwy) * v), v);
    }
  }
}

// phase A over in-field nodes [2h, 2h+2) of all fields: every load first, then
// the updates and stores; accumulates the partials (r,u), (r,r)
// first: the first iteration reads p = s = 0 and x = x0 = rhs instead of
// initialised vectors (same operations as with zero-filled p, s and x = rhs)
template <int NC>
__device__ __forceinline__ void cg_update2(const Cg2Args& A, double* Un, long long h, long long nh, double alpha,
                                           double beta, double& ru, double& rr, bool first) {
  const double2 di = reinterpret_cast<const double2*>(A.DINV)[h];
  double2 r[NC], pv[NC], sv[NC], wv[NC], xv[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const long long t = c * nh + h;
    r[c] = reinterpret_cast<const double2*>(A.R)[t];
    pv[c] = reinterpret_cast<const double2*>(A.Pv)[t];
    sv[c] = first ? make_double2(0.0, 0.0) : reinterpret_cast<const double2*>(A.S)[t];
    wv[c] = reinterpret_cast<const double2*>(A.W)[t];
    xv[c] = reinterpret_cast<const double2*>(A.x)[t];
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const long long t = c * nh + h;
    double2 p, s, x, rn;
    p.x = fma(beta, pv[c].x, r[c].x * di.x);
    p.y = fma(beta, pv[c].y, r[c].y * di.y);
    s.x = fma(beta, sv[c].x, wv[c].x);
    s.y = fma(beta, sv[c].y, wv[c].y);
    x.x = fma(alpha, p.x, xv[c].x);
    x.y = fma(alpha, p.y, xv[c].y);
    rn.x = fma(-alpha, s.x, r[c].x);
    rn.y = fma(-alpha, s.y, r[c].y);
    reinterpret_cast<double2*>(A.Pv)[t] = p;
    reinterpret_cast<double2*>(A.S)[t] = s;
    reinterpret_cast<double2*>(A.x)[t] = x;
    reinterpret_cast<double2*>(A.R)[t] = rn;
    const double2 un = make_double2(rn.x * di.x, rn.y * di.y);
    reinterpret_cast<double2*>(Un)[t] = un;
    ru = fma(rn.x, un.x, ru);
    rr = fma(rn.x, rn.x, rr);
    ru = fma(rn.y, un.y, ru);
    rr = fma(rn.y, rn.y, rr);
  }
}

// phase A' (p / x deferred to phase B): s = w + beta s, r -= alpha s,
// u_new = r dinv over in-field pairs; partials (r,u), (r,r).  p and x only feed
// the final x, so their update p = u_prev + beta p, x += alpha p (the same
// operations as cg_update2, u_prev = r_old dinv bitwise) rides in the
// issue-bound phase B, which has HBM bandwidth to spare; u is double-buffered.
template <int NC>
__device__ __forceinline__ void cg_update2s(const Cg2Args& A, double* Un, long long h, long long nh, double alpha,
                                            double beta, double& ru, double& rr, bool first) {
  const double2 di = reinterpret_cast<const double2*>(A.DINV)[h];
  double2 r[NC], sv[NC], wv[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const long long t = c * nh + h;
    r[c] = reinterpret_cast<const double2*>(A.R)[t];
    sv[c] = first ? make_double2(0.0, 0.0) : reinterpret_cast<const double2*>(A.S)[t];
    wv[c] = reinterpret_cast<const double2*>(A.W)[t];
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const long long t = c * nh + h;
    double2 s, rn;
    s.x = fma(beta, sv[c].x, wv[c].x);
    s.y = fma(beta, sv[c].y, wv[c].y);
    rn.x = fma(-alpha, s.x, r[c].x);
    rn.y = fma(-alpha, s.y, r[c].y);
    reinterpret_cast<double2*>(A.S)[t] = s;
    reinterpret_cast<double2*>(A.R)[t] = rn;
    const double2 un = make_double2(rn.x * di.x, rn.y * di.y);
    reinterpret_cast<double2*>(Un)[t] = un;
    ru = fma(rn.x, un.x, ru);
    rr = fma(rn.x, rn.x, rr);
    ru = fma(rn.y, un.y, ru);
    rr = fma(rn.y, rn.y, rr);
  }
}
// scalar form (odd sizes / misaligned x)
template <int NC>
__device__ __forceinline__ void cg_update1s(const Cg2Args& A, double* Un, long long f, long long nn, double alpha,
                                            double beta, double& ru, double& rr, bool first) {
  const double di = A.DINV[f];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const long long t = c * nn + f;
    const double s = fma(beta, first ? 0.0 : A.S[t], A.W[t]);
    A.S[t] = s;
    const double r = fma(-alpha, s, A.R[t]);
    A.R[t] = r;
    const double u = r * di;
    Un[t] = u;
    ru = fma(r, u, ru);
    rr = fma(r, r, rr);
  }
}
// full scalar update (p, x in phase A: the P != 7 levels, see k2_cg)
template <int NC>
__device__ __forceinline__ void cg_update1(const Cg2Args& A, double* Un, long long f, long long nn, double alpha,
                                           double beta, double& ru, double& rr, bool first) {
  const double di = A.DINV[f];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const long long t = c * nn + f;
    double r = A.R[t];
    const double p = fma(beta, A.Pv[t], r * di);
    const double s = fma(beta, first ? 0.0 : A.S[t], A.W[t]);
    A.Pv[t] = p;
    A.S[t] = s;
    A.x[t] = fma(alpha, p, A.x[t]);
    r = fma(-alpha, s, r);
    A.R[t] = r;
    const double u = r * di;
    Un[t] = u;
    ru = fma(r, u, ru);
    rr = fma(r, r, rr);
  }
}
// deferred p / x update at global index g (pair when two)
__device__ __forceinline__ void cg_px2(const Cg2Args& A, const double* Up, long long g, double alpha, double beta) {
  const double2 u = *reinterpret_cast<const double2*>(Up + g);
  double2 p = *reinterpret_cast<const double2*>(A.Pv + g);
  double2 x = *reinterpret_cast<const double2*>(A.x + g);
  p.x = fma(beta, p.x, u.x);
  p.y = fma(beta, p.y, u.y);
  x.x = fma(alpha, p.x, x.x);
  x.y = fma(alpha, p.y, x.y);
  *reinterpret_cast<double2*>(A.Pv + g) = p;
  *reinterpret_cast<double2*>(A.x + g) = x;
}
__device__ __forceinline__ void cg_px1(const Cg2Args& A, const double* Up, long long g, double alpha, double beta) {
  const double p = fma(beta, A.Pv[g], Up[g]);
  A.Pv[g] = p;
  A.x[g] = fma(alpha, p, A.x[g]);
}

// ------------------------------------------------------------------------
// P = 7 (P1 = 8) phase B: one warp per element, fp64 tensor cores.
// A warp owns element e (all fields).  It copies the element and its four face
// neighbours (whole elements, contiguous 512-byte runs per field) global ->
// shared with 16-byte cp.async, then per field runs the 8x8 contractions as
// mma.m8n8k4.f64:  QX = U D^T, QY = D U (times C s), BX = QX DTW^T,
// BY = DTW QY, with the D / DTW fragments in registers.  Everything a unit
// needs lives in the warp's own shared region, so phase B has no block
// barrier at all: warps stream through elements independently and latency is
// hidden across the warps of the SM.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

template <int NC>
struct Wpe {                 // per-warp shared region (doubles): a two-stage pipeline of (element, field) tasks
  static constexpr int RP = 10, NP = 80, NN = 64;   // own element rows padded to 10 (16-byte aligned)
  static constexpr int OWN = 0;                     // [2 stages][NP] one field of the own element
  static constexpr int NBR = OWN + 2 * NP;          // [2 stages][4 faces][64] that field's neighbour elements
  static constexpr int COEF = NBR + 2 * 4 * NN;     // [2 element parities][NP] own coefficient
  static constexpr int CFN = COEF + 2 * NP;         // [2 element parities][32] neighbour face coefficients
  static constexpr int QX = CFN + 64, QY = QX + NP, DOT = QY + NP;   // [NP] [NP] [32]
  static constexpr int FCON = DOT + 32;             // [16][4] face constants per x-row / y-column
  static constexpr int WARP = FCON + 64;
  static_assert(8 * WARP == CgSm<8, NC>::WPE, "keep CgSm::WPE in sync");
};

// neighbour element node (row, col) in the swizzled layout: chunk (col/2) ^ (row/2)
__device__ __forceinline__ int nsw(int row, int col) { return row * 8 + ((((col >> 1) ^ (row >> 1))) << 1) + (col & 1); }

struct MmaLane {            // per-lane constants, g = lane/4, t = lane%4, n0 = 2t
  double d0, d1, w0, w1;    // D[g][t], D[g][4+t], DTW[g][t], DTW[g][4+t]
  double drow[8];           // D row 0 (faces R, T) or row P (faces L, B) for this lane's face dot
  double dPn[2], d0n[2];    // D[P][n0+i], D[0][n0+i]
  double dPg, d0g;          // D[P][g], D[0][g]
  double hwy, hwx[2], hh[2];
  double wn[2], wg;         // GLL weights w[n0+i], w[g]
  double cfn;               // this lane's neighbour face coefficient (per element)
};
// lane-varying constants come from the global operator table (TabOff layout):
// lane-divergent constant-bank loads would serialise, and the compiler would
// rematerialise them inside the element loop
__device__ __forceinline__ void mma_lane_init(const Op2DDev& op, MmaLane& K) {
  const double* D = op.tab + TabOff::D(8);
  const double* DTW = op.tab + TabOff::DTW(8);
  const double* w = op.tab + TabOff::w(8);
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, f = lane >> 3, n0 = 2 * t;
  K.d0 = D[g * 8 + t];
  K.d1 = D[g * 8 + 4 + t];
  K.w0 = DTW[g * 8 + t];
  K.w1 = DTW[g * 8 + 4 + t];
  const int rr = (f == FL || f == FB) ? 7 : 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) K.drow[q] = D[rr * 8 + q];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    K.dPn[i] = D[7 * 8 + n0 + i];
    K.d0n[i] = D[n0 + i];
    K.hwx[i] = 0.5 * op.dx * w[n0 + i];
  }
  K.dPg = D[7 * 8 + g];
  K.d0g = D[g];
  K.hwy = 0.5 * op.dy * w[g];
  K.hh[0] = K.hwx[0] * K.hwy;
  K.hh[1] = K.hwx[1] * K.hwy;
  K.wn[0] = w[n0];
  K.wn[1] = w[n0 + 1];
  K.wg = w[g];
}

// SIP accumulators of one field of a staged element for the lane's node pair
// (row g, columns n0, n0+1): bx = Bx, by = By incl. face and adjoint terms
// (sip_block).  Ue: own element (padded rows), Nb: neighbour face lines of this
// field, Ce / cfn: coefficient at the own nodes (padded rows) / at the
// neighbour face nodes (lane = face*8 + k).  Scratch: QX, QY, DT, FC.
template <int NC, int FS = NC * 64>   // FS: stride between the four faces' lines in Nb
__device__ __forceinline__ void wpe_sip(const Op2DDev& op, const MmaLane& K, const double* Ue, const double* Nb,
                                        const double* Ce, const double* cfn, double* QX, double* QY, double* DT,
                                        double* FC, double& bx0, double& bx1, double& by0, double& by1) {
  constexpr int RP = 10, P = 7;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, n0 = 2 * t;
  // Q = C s (D u) along x and y
  double qx0 = 0.0, qx1 = 0.0, qy0 = 0.0, qy1 = 0.0;
  dmma(qx0, qx1, Ue[g * RP + t], K.d0);
  dmma(qx0, qx1, Ue[g * RP + 4 + t], K.d1);
  dmma(qy0, qy1, K.d0, Ue[t * RP + g]);
  dmma(qy0, qy1, K.d1, Ue[(4 + t) * RP + g]);
  {
    const double2 cg = *reinterpret_cast<const double2*>(Ce + g * RP + n0);
    *reinterpret_cast<double2*>(QX + g * RP + n0) = make_double2(cg.x * (op.sx * qx0), cg.y * (op.sx * qx1));
    *reinterpret_cast<double2*>(QY + g * RP + n0) = make_double2(cg.x * (op.sy * qy0), cg.y * (op.sy * qy1));
  }
  // neighbour face fluxes: lane = face*8 + k, line k of face f
  {
    const int f = lane >> 3, k = lane & 7;
    const double* ln = Nb + f * FS + k * 8;
    double gd = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(ln + 2 * (j ^ (k >> 1)));
      gd = fma(K.drow[2 * j], v.x, gd);
      gd = fma(K.drow[2 * j + 1], v.y, gd);
    }
    DT[lane] = cfn[lane] * ((f < FT ? op.sx : op.sy) * gd);
  }
  __syncwarp();
  bx0 = bx1 = by0 = by1 = 0.0;
  dmma(bx0, bx1, QX[g * RP + t], K.w0);
  dmma(bx0, bx1, QX[g * RP + 4 + t], K.w1);
  dmma(by0, by1, K.w0, QY[t * RP + g]);
  dmma(by0, by1, K.w1, QY[(4 + t) * RP + g]);
  // face constants, once per line: lanes 0-7 x-row r, lanes 8-15 y-column r
  if (lane < 16) {
    const bool yd = lane >= 8;
    const int r = lane & 7;
    const int up = yd ? P * RP + r : r * RP + P, u0 = yd ? r : r * RP;
    const double jp = Ue[up] - Nb[(yd ? FT : FR) * FS + nsw(r, 0)];
    const double jm = Nb[(yd ? FB : FL) * FS + nsw(r, P)] - Ue[u0];
    const double cP = Ce[up], c0 = Ce[u0];
    const double fcp = cfn[(yd ? 16 : 0) + r], fcm = cfn[(yd ? 24 : 8) + r];
    const double qP = (yd ? QY : QX)[up], q0 = (yd ? QY : QX)[u0];
    const double qnp = DT[(yd ? 16 : 0) + r], qnm = DT[(yd ? 24 : 8) + r];
    const double mu = yd ? op.muy : op.mux, sc = yd ? op.sy : op.sx;
    const double fp = -(0.5 * (qP + qnp)) + (mu * (0.5 * (cP + fcp))) * jp;
    const double fm = -(0.5 * (qnm + q0)) + (mu * (0.5 * (fcm + c0))) * jm;
    *reinterpret_cast<double4*>(FC + lane * 4) = make_double4(fp, fm, sc * ((0.5 * cP) * jp), sc * ((0.5 * c0) * jm));
  }
  __syncwarp();
  {
    const double4 rx = *reinterpret_cast<const double4*>(FC + g * 4);
    if (n0 + 1 == P) bx1 += rx.x;
    if (n0 == 0) bx0 -= rx.y;
    bx0 -= rx.z * K.dPn[0];
    bx1 -= rx.z * K.dPn[1];
    bx0 -= rx.w * K.d0n[0];
    bx1 -= rx.w * K.d0n[1];
    const double4 ca = *reinterpret_cast<const double4*>(FC + (8 + n0) * 4);
    const double4 cb = *reinterpret_cast<const double4*>(FC + (9 + n0) * 4);
    if (g == P) { by0 += ca.x; by1 += cb.x; }
    if (g == 0) { by0 -= ca.y; by1 -= cb.y; }
    by0 -= ca.z * K.dPg;
    by1 -= cb.z * K.dPg;
    by0 -= ca.w * K.d0g;
    by1 -= cb.w * K.d0g;
  }
  __syncwarp();   // QX / QY / DT / FC are rewritten by the next call
}

// deferred CG p / x update riding in phase B (see cg_update2s); up == nullptr: none
struct PxArgs {
  const double* up;
  double* p;
  double* x;
  double al, be;
};

// one field of a staged element: w = a (hwy Bx + hwx By) + hwx hwy v;
// epi(g, w0, w1, v0, v1) for the lane's node pair.  With px.up, the field's
// p / x operands are loaded before the contractions (their latency hides
// behind the tensor-core work) and updated after.  sb: stage buffer of the
// field, ep: element parity of the coefficient buffers.
template <int NC, typename Epi>
__device__ __forceinline__ void wpe_field(const Op2DDev& op, double* ws, int sb, int ep, const MmaLane& K, int c,
                                          double a, long long gi, Epi&& epi, const PxArgs& px) {
  using W = Wpe<NC>;
  const int lane = threadIdx.x & 31, g = lane >> 2, n0 = 2 * (lane & 3);
  const double* Ue = ws + W::OWN + sb * W::NP;
  const long long gc = gi + c * op.nn;
  double2 pu, pp, px_;
  if (px.up) {
    pu = __ldcs(reinterpret_cast<const double2*>(px.up + gc));
    pp = __ldcs(reinterpret_cast<const double2*>(px.p + gc));
    px_ = __ldcs(reinterpret_cast<const double2*>(px.x + gc));
  }
  double bx0, bx1, by0, by1;
  wpe_sip<NC, 64>(op, K, Ue, ws + W::NBR + sb * 4 * W::NN, ws + W::COEF + ep * W::NP, ws + W::CFN + ep * 32,
                  ws + W::QX, ws + W::QY, ws + W::DOT, ws + W::FCON, bx0, bx1, by0, by1);
  const double2 v = *reinterpret_cast<const double2*>(Ue + g * W::RP + n0);
  epi(gc, fma(a, fma(K.hwy, bx0, K.hwx[0] * by0), K.hh[0] * v.x),
      fma(a, fma(K.hwy, bx1, K.hwx[1] * by1), K.hh[1] * v.y), v.x, v.y);
  if (px.up) {
    pp.x = fma(px.be, pp.x, pu.x);
    pp.y = fma(px.be, pp.y, pu.y);
    px_.x = fma(px.al, pp.x, px_.x);
    px_.y = fma(px.al, pp.y, px_.y);
    __stcs(reinterpret_cast<double2*>(px.p + gc), pp);
    __stcs(reinterpret_cast<double2*>(px.x + gc), px_);
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// the block's share of phase B: warps stride over elements; each warp runs a
// two-stage cp.async pipeline over its (element, field) tasks -- the staging
// of the next task (one field of the element and of its four face
// neighbours; the coefficient with field 0) is in flight while the current
// task's contractions run.  Same tasks, same order, same arithmetic as the
// unpipelined version (bitwise).
template <int NC, typename Epi>
__device__ __forceinline__ void wpe_phase(const Op2DDev& op, double* sm, const double* src, const double* Cf,
                                          double a, Epi&& epi, long long* tacc = nullptr,
                                          const PxArgs& px = PxArgs{nullptr, nullptr, nullptr, 0.0, 0.0}) {
  using W = Wpe<NC>;
  MmaLane K;
  mma_lane_init(op, K);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  double* ws = sm + warp * W::WARP;
  const int ne = op.nex * op.ney;
  const long long nn = op.nn;
  const int r = lane >> 2, cc = (lane & 3) * 2;
  const int f = lane >> 3, k = lane & 7;
  const int fnode = f == FR ? k * 8 : f == FL ? k * 8 + 7 : f == FT ? k : 56 + k;   // neighbour's face node
  const int swz = r * 8 + 2 * ((lane & 3) ^ (r >> 1));            // row r, chunk lane&3 (swizzled)
  const int tr0 = nsw(lane & 7, lane >> 3), tr1 = nsw(lane & 7, 4 + (lane >> 3));   // transposed: node v -> line v%8, pos v/8
  const int stride = gridDim.x * nwb;
  auto eoff = [&](int e) -> unsigned {
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    return ((unsigned)ey * op.nex + ex) * 64u;
  };
  // stage field c of element e (and its neighbours' field c) into buffer sb;
  // field 0 also stages the element's coefficients into parity ep
  auto issue = [&](int e, int c, int sb, int ep) {
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    const int exr = ex + 1 == op.nex ? 0 : ex + 1, exl = ex == 0 ? op.nex - 1 : ex - 1;
    const int eyt = ynb(op, ey, 1), eyb = ynb(op, ey, -1);
    const unsigned eo = ((unsigned)ey * op.nex + ex) * 64u;
    const unsigned nbR = ((unsigned)ey * op.nex + exr) * 64u, nbL = ((unsigned)ey * op.nex + exl) * 64u;
    const unsigned nbT = ((unsigned)eyt * op.nex + ex) * 64u, nbB = ((unsigned)eyb * op.nex + ex) * 64u;
    const double* sc = src + c * nn;
    double* nbr = ws + W::NBR + sb * 4 * W::NN;
    cp_async16(ws + W::OWN + sb * W::NP + r * W::RP + cc, sc + eo + 2 * lane);
    // face lines in swizzled rows: R/L neighbours row-wise (16-byte copies), T/B
    // neighbours transposed (8-byte copies) so every face line is a row
    cp_async16(nbr + FR * 64 + swz, sc + nbR + 2 * lane);
    cp_async16(nbr + FL * 64 + swz, sc + nbL + 2 * lane);
    cp_async8(nbr + FT * 64 + tr0, sc + nbT + lane);
    cp_async8(nbr + FT * 64 + tr1, sc + nbT + 32 + lane);
    cp_async8(nbr + FB * 64 + tr0, sc + nbB + lane);
    cp_async8(nbr + FB * 64 + tr1, sc + nbB + 32 + lane);
    if (c == 0) {
      cp_async16(ws + W::COEF + ep * W::NP + r * W::RP + cc, Cf + eo + 2 * lane);
      cp_async8(ws + W::CFN + ep * 32 + lane, Cf + (f == FR ? nbR : f == FL ? nbL : f == FT ? nbT : nbB) + fnode);
    }
  };
  int e = blockIdx.x * nwb + warp;
  if (e >= ne) return;
  issue(e, 0, 0, 0);
  cp_async_commit();
  int sb = 0, ep = 0;
  const int g = lane >> 2, n0 = 2 * (lane & 3);
  for (; e < ne; e += stride, ep ^= 1) {
    const long long gi = (long long)eoff(e) + g * 8 + n0;
    const long long c0 = tacc ? clock64() : 0;
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const bool last = c + 1 == NC;
      const int en = last ? e + stride : e;
      if (en < ne) issue(en, last ? 0 : c + 1, sb ^ 1, last ? ep ^ 1 : ep);
      cp_async_commit();    // one group per task (possibly empty)
      cp_async_wait_1();    // this task's group has landed
      __syncwarp();
      wpe_field<NC>(op, ws, sb, ep, K, c, a, gi, epi, px);
      __syncwarp();         // buffer sb is refilled by the next task's prefetch
      sb ^= 1;
    }
    if (tacc) { tacc[1] += clock64() - c0; tacc[2] += 1; }
  }
  cp_async_wait_all();
}

// ------------------------------------------------------------------------
// P = 7 (P1 = 8) node evaluation / cache refresh (k2_node_eval semantics), one
// warp per element: u_m and its face neighbours staged as in the CG phase B,
// the convective volume terms and the SIP operators (physical and SI
// coefficient) on the fp64 tensor cores, Rusanov face fluxes per face node.
template <int NC>
struct Ev {                 // per-warp shared region (doubles)
  static constexpr int RP = 10, NP = 80;
  static constexpr int OWN = 0;                     // [NC][NP] u_m
  static constexpr int NBR = OWN + NC * NP;         // [4][NC][64] u_m face neighbours (lines)
  static constexpr int UPO = NBR + 4 * NC * 64;     // [NC][NP] u_{m-1}
  static constexpr int CSI = UPO + NC * NP, CFS = CSI + NP;   // SI coefficient own / face
  static constexpr int CPH = CFS + 32, CFP = CPH + NP;        // physical coefficient own / face
  static constexpr int QX = CFP + 32, QY = QX + NP, DOT = QY + NP, FCON = DOT + 32;
  static constexpr int FX = FCON + 64, FY = FX + NC * NP;     // fluxes of all fields [NC][NP]
  static constexpr int FHM = FY + NC * NP, FHP = FHM + 32 * NC;   // Rusanov fluxes [lane][NC]
  static constexpr int CPV = FHP + 32 * NC;         // [NC][NP] cached conv(u_{m-1}) (a.conv_prev), staged with the element
  static constexpr int WARP = CPV + NC * NP;
};
constexpr int EV_WARPS = 4;

// fluxes F^x, F^y of ALL fields at the lane's node pair of a staged element (state rows in
// `own`, padded) -> FX4 / FY4 [NC][80]: one flux evaluation per node and axis (the per-field
// version re-evaluated the full flux, divisions included, for every field it picked)
template <int NC>
__device__ __forceinline__ void wpe_flux_all(const Op2DDev& op, const double* own, double* FX4, double* FY4) {
  constexpr int RP = 10;
  const int lane = threadIdx.x & 31, g = lane >> 2, n0 = 2 * (lane & 3);
  double fx[2][NC_MAX], fy[2][NC_MAX];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    double st[NC_MAX];
#pragma unroll
    for (int q = 0; q < NC_MAX; ++q) st[q] = q < NC ? own[q * 80 + g * RP + n0 + i] : 1.0;
    flux2d(op, st, 0, fx[i]);
    flux2d(op, st, 1, fy[i]);
  }
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    *reinterpret_cast<double2*>(FX4 + q * 80 + g * RP + n0) = make_double2(fx[0][q], fx[1][q]);
    *reinterpret_cast<double2*>(FY4 + q * 80 + g * RP + n0) = make_double2(fy[0][q], fy[1][q]);
  }
  __syncwarp();
}

// convective term of field c at the lane's node pair from the staged fluxes FX / FY of that
// field (wpe_flux_all) and the face fluxes fh[lane*NC + c]; rx[i] = sx / w[n0+i], ry = sy / w[g]
template <int NC>
__device__ __forceinline__ void wpe_conv(const MmaLane& K, const double* fh, int c, const double* FX,
                                         const double* FY, const double (&rx)[2], double ry, double& r0,
                                         double& r1) {
  constexpr int RP = 10, P = 7;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, n0 = 2 * t;
  double vx0 = 0.0, vx1 = 0.0, vy0 = 0.0, vy1 = 0.0;
  dmma(vx0, vx1, FX[g * RP + t], K.w0);
  dmma(vx0, vx1, FX[g * RP + 4 + t], K.w1);
  dmma(vy0, vy1, K.w0, FY[t * RP + g]);
  dmma(vy0, vy1, K.w1, FY[(4 + t) * RP + g]);
  if (n0 + 1 == P) vx1 -= fh[(FR * 8 + g) * NC + c];
  if (n0 == 0) vx0 += fh[(FL * 8 + g) * NC + c];
  if (g == P) { vy0 -= fh[(FT * 8 + n0) * NC + c]; vy1 -= fh[(FT * 8 + n0 + 1) * NC + c]; }
  if (g == 0) { vy0 += fh[(FB * 8 + n0) * NC + c]; vy1 += fh[(FB * 8 + n0 + 1) * NC + c]; }
  r0 = vx0 * rx[0] + vy0 * ry;
  r1 = vx1 * rx[1] + vy1 * ry;
}

template <int NC>
__global__ void __launch_bounds__(EV_WARPS * 32) k2_eval8(Op2DDev op, Cache2Args a) {
  extern __shared__ double sm[];
  using W = Ev<NC>;
  constexpr int RP = 10, P = 7;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ws = sm + warp * W::WARP;
  const int m = a.m_first + blockIdx.y;
  const long long nn = op.nn;
  const double* um = a.u + (size_t)m * op.ns;
  const double* up = m == 0 ? a.u0 : a.u + (size_t)(m - 1) * op.ns;
  double dtm = 0.0;   // static-index select: a dynamic index would copy the parameter block to local memory
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j == m) dtm = a.dts[j];
  double ph;
  const bool has_phys = phys2d(op, 0, ph);          // constant nu (no AV on this path)
  const bool need_si = a.mode != 0 && dtm != 0.0 && a.scheme != SISDC_EULER;
  const bool need_h = a.mode != 0 && dtm != 0.0;
  const bool conv_up = need_h && a.conv_prev == nullptr;
  MmaLane K;
  mma_lane_init(op, K);
  // reciprocal lane constants: the divisions by the mass weights were ~15% of this kernel's samples
  const double rcx[2] = {op.sx / K.wn[0], op.sx / K.wn[1]}, rcy = op.sy / K.wg;
  const double rhx[2] = {1.0 / K.hwx[0], 1.0 / K.hwx[1]}, rhy = 1.0 / K.hwy;
  const int g = lane >> 2, n0 = 2 * (lane & 3), r = g, cc = n0;
  const int f = lane >> 3, k = lane & 7;
  const int fnode = f == FR ? k * 8 : f == FL ? k * 8 + 7 : f == FT ? k : 56 + k;
  const int ownf = f == FR ? k * RP + P : f == FL ? k * RP : f == FT ? P * RP + k : k;   // own face node (padded)
  const int npos = nsw(k, (f == FR || f == FT) ? 0 : P);                                // neighbour node on line k
  const int swz = r * 8 + 2 * ((lane & 3) ^ (r >> 1));
  const int tr0 = nsw(lane & 7, lane >> 3), tr1 = nsw(lane & 7, 4 + (lane >> 3));
  if (has_phys) {
    for (int q = lane; q < W::NP; q += 32) ws[W::CPH + q] = ph;
    ws[W::CFP + lane] = ph;
  }
  const int ne = op.nex * op.ney;
  for (int e = blockIdx.x * EV_WARPS + warp; e < ne; e += gridDim.x * EV_WARPS) {
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    const int exr = ex + 1 == op.nex ? 0 : ex + 1, exl = ex == 0 ? op.nex - 1 : ex - 1;
    const int eyt = ynb(op, ey, 1), eyb = ynb(op, ey, -1);
    const unsigned eo = ((unsigned)ey * op.nex + ex) * 64u;
    const unsigned nb[4] = {((unsigned)ey * op.nex + exr) * 64u, ((unsigned)ey * op.nex + exl) * 64u,
                            ((unsigned)eyt * op.nex + ex) * 64u, ((unsigned)eyb * op.nex + ex) * 64u};
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double* uc = um + c * nn;
      cp_async16(ws + W::OWN + c * W::NP + r * RP + cc, uc + eo + 2 * lane);
      cp_async16(ws + W::NBR + (FR * NC + c) * 64 + swz, uc + nb[FR] + 2 * lane);
      cp_async16(ws + W::NBR + (FL * NC + c) * 64 + swz, uc + nb[FL] + 2 * lane);
      cp_async8(ws + W::NBR + (FT * NC + c) * 64 + tr0, uc + nb[FT] + lane);
      cp_async8(ws + W::NBR + (FT * NC + c) * 64 + tr1, uc + nb[FT] + 32 + lane);
      cp_async8(ws + W::NBR + (FB * NC + c) * 64 + tr0, uc + nb[FB] + lane);
      cp_async8(ws + W::NBR + (FB * NC + c) * 64 + tr1, uc + nb[FB] + 32 + lane);
      if (need_si || conv_up) cp_async16(ws + W::UPO + c * W::NP + r * RP + cc, up + c * nn + eo + 2 * lane);
      // the cached conv(u_{m-1}) rides with the staging (read in the field loop it stalled 19% of the samples)
      if (need_h && a.conv_prev)
        cp_async16(ws + W::CPV + c * W::NP + r * RP + cc, a.conv_prev + (size_t)(m - a.m_first) * op.ns + c * nn + eo + 2 * lane);
    }
    double upf[NC_MAX];   // u_{m-1} at this lane's neighbour face node
    const unsigned nbf = (f == FR ? nb[FR] : f == FL ? nb[FL] : f == FT ? nb[FT] : nb[FB]) + fnode;
#pragma unroll
    for (int c = 0; c < NC_MAX; ++c) upf[c] = (c < NC && (need_si || conv_up)) ? up[c * nn + nbf] : 1.0;
    cp_async_wait_all();
    __syncwarp();
    // SI coefficient (dt_m/2) lam(u_{m-1})^2 + phys at the own nodes and the neighbour face nodes
    if (need_si) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double st[NC_MAX];
#pragma unroll
        for (int q = 0; q < NC_MAX; ++q) st[q] = q < NC ? ws[W::UPO + q * W::NP + g * RP + n0 + i] : 1.0;
        const double lam = lam_max2d(op, st);
        const double half = 0.5 * dtm * (lam * lam);
        ws[W::CSI + g * RP + n0 + i] = op.problem == SISDC_NS2D ? half + (op.nu / st[0]) * op.nsi   // coef2d
                                                                : (has_phys ? half + ph : half);
      }
      const double lam = lam_max2d(op, upf);
      const double half = 0.5 * dtm * (lam * lam);
      ws[W::CFS + lane] = op.problem == SISDC_NS2D ? half + (op.nu / upf[0]) * op.nsi : (has_phys ? half + ph : half);
    }
    // Rusanov fluxes at this lane's face node for u_m (and u_{m-1})
    {
      double so[NC_MAX], sn[NC_MAX], fh[NC_MAX];
#pragma unroll
      for (int c = 0; c < NC_MAX; ++c) {
        so[c] = c < NC ? ws[W::OWN + c * W::NP + ownf] : 1.0;
        sn[c] = c < NC ? ws[W::NBR + (f * NC + c) * 64 + npos] : 1.0;
      }
      const int axis = f < FT ? 0 : 1;
      if (f == FR || f == FT) rusanov2d(op, so, sn, axis, fh); else rusanov2d(op, sn, so, axis, fh);
#pragma unroll
      for (int c = 0; c < NC; ++c) ws[W::FHM + lane * NC + c] = fh[c];
      if (conv_up) {
#pragma unroll
        for (int c = 0; c < NC_MAX; ++c) so[c] = c < NC ? ws[W::UPO + c * W::NP + ownf] : 1.0;
        if (f == FR || f == FT) rusanov2d(op, so, upf, axis, fh); else rusanov2d(op, upf, so, axis, fh);
#pragma unroll
        for (int c = 0; c < NC; ++c) ws[W::FHP + lane * NC + c] = fh[c];
      }
    }
    __syncwarp();
    const long long gi = (long long)eo + g * 8 + n0;
    wpe_flux_all<NC>(op, ws + W::OWN, ws + W::FX, ws + W::FY);   // fluxes of u_m, all fields, once
    double dsv[NC][2];   // SI-coefficient diffusion per field (needed again if conv(u_{m-1}) is rebuilt below)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double* Ue = ws + W::OWN + c * W::NP;
      const double* Nb = ws + W::NBR + c * 64;
      double bx0, bx1, by0, by1;
      double dp0 = 0.0, dp1 = 0.0, ds0 = 0.0, ds1 = 0.0;
      if (has_phys) {
        wpe_sip<NC>(op, K, Ue, Nb, ws + W::CPH, ws + W::CFP, ws + W::QX, ws + W::QY, ws + W::DOT, ws + W::FCON,
                    bx0, bx1, by0, by1);
        dp0 = -(bx0 * rhx[0]) - by0 * rhy;
        dp1 = -(bx1 * rhx[1]) - by1 * rhy;
      }
      if (need_si) {
        wpe_sip<NC>(op, K, Ue, Nb, ws + W::CSI, ws + W::CFS, ws + W::QX, ws + W::QY, ws + W::DOT, ws + W::FCON,
                    bx0, bx1, by0, by1);
        ds0 = -(bx0 * rhx[0]) - by0 * rhy;
        ds1 = -(bx1 * rhx[1]) - by1 * rhy;
      } else if (need_h) {   // implicit-Euler scheme: modified coefficient = physical
        ds0 = dp0;
        ds1 = dp1;
      }
      dsv[c][0] = ds0;
      dsv[c][1] = ds1;
      double cm0, cm1;
      wpe_conv<NC>(K, ws + W::FHM, c, ws + W::FX + c * W::NP, ws + W::FY + c * W::NP, rcx, rcy, cm0, cm1);
      const long long go = (size_t)m * op.ns + c * nn + gi;
      const double f0 = has_phys ? cm0 + dp0 : cm0, f1 = has_phys ? cm1 + dp1 : cm1;
      if (!isfinite(f0) || !isfinite(f1)) atomicMin(a.status, (int)(op.e0 + e));
      *reinterpret_cast<double2*>(a.f + go) = make_double2(f0, f1);
      if (a.mode == 0) continue;
      if (!need_h) {
        *reinterpret_cast<double2*>(a.h1 + go) = make_double2(0.0, 0.0);
        if (a.h2) *reinterpret_cast<double2*>(a.h2 + go) = make_double2(0.0, 0.0);
        continue;
      }
      if (a.h2) *reinterpret_cast<double2*>(a.h2 + go) = make_double2(dtm * (cm0 + ds0), dtm * (cm1 + ds1));
      if (a.conv_prev) {
        const double2 v = *reinterpret_cast<const double2*>(ws + W::CPV + c * W::NP + g * RP + n0);
        *reinterpret_cast<double2*>(a.h1 + go) = make_double2(dtm * (v.x + ds0), dtm * (v.y + ds1));
      }
    }
    if (conv_up) {   // no cached conv(u_{m-1}) (cache refresh): rebuild it from the staged u_{m-1}
      __syncwarp();
      wpe_flux_all<NC>(op, ws + W::UPO, ws + W::FX, ws + W::FY);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double cp0, cp1;
        wpe_conv<NC>(K, ws + W::FHP, c, ws + W::FX + c * W::NP, ws + W::FY + c * W::NP, rcx, rcy, cp0, cp1);
        const long long go = (size_t)m * op.ns + c * nn + gi;
        *reinterpret_cast<double2*>(a.h1 + go) = make_double2(dtm * (cp0 + dsv[c][0]), dtm * (cp1 + dsv[c][1]));
      }
    }
    __syncwarp();   // the next element overwrites the staged data
  }
}

// P = 7 (P1 = 8) stage rhs (k2_stage semantics), one warp per element: the
// convective term of conv_in on the fp64 tensor cores (wpe_conv), Rusanov
// fluxes from the neighbours' face nodes read directly (no neighbour
// staging: convection needs only the face traces), the quadrature of f_old
// and the base / g / h terms per node pair with 16-byte accesses.
template <int NC>
struct Stg {                 // per-warp shared region (doubles)
  static constexpr int RP = 10, NP = 80;
  static constexpr int OWN = 0;                  // [2 stages][NC][NP] conv_in element
  static constexpr int FX = OWN + 2 * NC * NP, FY = FX + NC * NP;   // fluxes of all fields [NC][NP]
  static constexpr int FH = FY + NC * NP;        // [32][NC] face fluxes
  static constexpr int WARP = FH + 32 * NC;
};
// MQ: the number of quadrature nodes when it is a compile-time count (the streamed operands of a field --
// f_old of every node, g, base, h -- are then all requested BEFORE the field's tensor-core contractions
// and consumed after them; with the loads behind the contractions 60% of the kernel's samples waited on
// them, ncu r02w); MQ = 0: runtime count, loads in the quadrature loop.  The own element and the
// neighbours' face nodes of the NEXT element are requested one element ahead (two-stage cp.async).
template <int NC, int MQ>
__global__ void __launch_bounds__(EV_WARPS * 32, 3) k2_stage8(Op2DDev op, Stage2Args a) {
  extern __shared__ double sm[];
  using W = Stg<NC>;
  constexpr int RP = 10, P = 7;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ws = sm + warp * W::WARP;
  const long long nn = op.nn;
  MmaLane K;
  mma_lane_init(op, K);
  const double rcx[2] = {op.sx / K.wn[0], op.sx / K.wn[1]}, rcy = op.sy / K.wg;
  const int g = lane >> 2, n0 = 2 * (lane & 3);
  const int f = lane >> 3, k = lane & 7;
  const int fnode = f == FR ? k * 8 : f == FL ? k * 8 + 7 : f == FT ? k : 56 + k;      // neighbour's face node
  const int ownf = f == FR ? k * RP + P : f == FL ? k * RP : f == FT ? P * RP + k : k;   // own face node (padded)
  const int ne = op.nex * op.ney;
  const int stride = gridDim.x * EV_WARPS;
  // request element e: own nodes into stage sb, the neighbours' face-node states into sn
  auto issue = [&](int e, int sb, double (&sn)[NC_MAX]) {
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    const int exr = ex + 1 == op.nex ? 0 : ex + 1, exl = ex == 0 ? op.nex - 1 : ex - 1;
    const int eyt = ynb(op, ey, 1), eyb = ynb(op, ey, -1);
    const unsigned eo = ((unsigned)ey * op.nex + ex) * 64u;
    const unsigned nbf = (f == FR ? ((unsigned)ey * op.nex + exr) : f == FL ? ((unsigned)ey * op.nex + exl)
                          : f == FT ? ((unsigned)eyt * op.nex + ex) : ((unsigned)eyb * op.nex + ex)) * 64u + fnode;
#pragma unroll
    for (int c = 0; c < NC; ++c)
      cp_async16(ws + W::OWN + (sb * NC + c) * W::NP + g * RP + n0, a.conv_in + c * nn + eo + 2 * lane);
#pragma unroll
    for (int c = 0; c < NC_MAX; ++c) sn[c] = c < NC ? a.conv_in[c * nn + nbf] : 1.0;
  };
  int e = blockIdx.x * EV_WARPS + warp;
  if (e >= ne) return;
  double sn[NC_MAX], snn[NC_MAX];
  issue(e, 0, sn);
  cp_async_commit();
  int sb = 0;
  for (; e < ne; e += stride, sb ^= 1) {
#pragma unroll
    for (int c = 0; c < NC_MAX; ++c) snn[c] = 1.0;
    if (e + stride < ne) issue(e + stride, sb ^ 1, snn);
    cp_async_commit();
    cp_async_wait_1();
    __syncwarp();
    const double* own = ws + W::OWN + sb * NC * W::NP;
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    const unsigned eo = ((unsigned)ey * op.nex + ex) * 64u;
    {
      double so[NC_MAX], fh[NC_MAX];
#pragma unroll
      for (int c = 0; c < NC_MAX; ++c) so[c] = c < NC ? own[c * W::NP + ownf] : 1.0;
      const int axis = f < FT ? 0 : 1;
      if (f == FR || f == FT) rusanov2d(op, so, sn, axis, fh); else rusanov2d(op, sn, so, axis, fh);
#pragma unroll
      for (int c = 0; c < NC; ++c) ws[W::FH + lane * NC + c] = fh[c];
    }
    __syncwarp();
    const long long gi = (long long)eo + g * 8 + n0;
    wpe_flux_all<NC>(op, own, ws + W::FX, ws + W::FY);
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const long long gc = c * nn + gi;
      // streamed operands of this field, requested ahead of the contractions
      double2 fo[MQ > 0 ? MQ : 1];
      double2 gv = make_double2(0.0, 0.0), hv = make_double2(0.0, 0.0);
      if constexpr (MQ > 0) {
        if (a.f_old) {
#pragma unroll
          for (int jj = 0; jj < MQ; ++jj) fo[jj] = __ldcs(reinterpret_cast<const double2*>(a.f_old + (size_t)jj * op.ns + gc));
        }
      }
      if (a.g) gv = __ldcs(reinterpret_cast<const double2*>(a.g + gc));
      const double2 bv = __ldcs(reinterpret_cast<const double2*>(a.base + gc));
      if (a.h) hv = __ldcs(reinterpret_cast<const double2*>(a.h + gc));
      double cv0, cv1;
      wpe_conv<NC>(K, ws + W::FH, c, ws + W::FX + c * W::NP, ws + W::FY + c * W::NP, rcx, rcy, cv0, cv1);
      if (a.conv_out) *reinterpret_cast<double2*>(a.conv_out + gc) = make_double2(cv0, cv1);
      double q0 = 0.0, q1 = 0.0;
      if (a.f_old) {
        double acc0 = 0.0, acc1 = 0.0;
        if constexpr (MQ > 0) {
#pragma unroll
          for (int jj = 0; jj < MQ; ++jj) {
            acc0 = fma(a.w[jj], fo[jj].x, acc0);
            acc1 = fma(a.w[jj], fo[jj].y, acc1);
          }
        } else {
          for (int jj = 0; jj < a.M; ++jj) {
            const double2 fv = *reinterpret_cast<const double2*>(a.f_old + (size_t)jj * op.ns + gc);
            acc0 = fma(a.w[jj], fv.x, acc0);
            acc1 = fma(a.w[jj], fv.y, acc1);
          }
        }
        q0 = a.dt * acc0;
        q1 = a.dt * acc1;
      }
      if (a.g) {
        q0 = q0 + gv.x;
        q1 = q1 + gv.y;
      }
      double r0 = (bv.x + q0) + a.dt_m * cv0, r1 = (bv.y + q1) + a.dt_m * cv1;
      if (a.h) {
        r0 = r0 - hv.x;
        r1 = r1 - hv.y;
      }
      *reinterpret_cast<double2*>(a.rhs + gc) = make_double2(r0, r1);
    }
#pragma unroll
    for (int c = 0; c < NC_MAX; ++c) sn[c] = snn[c];
    __syncwarp();   // FX / FY / FH and stage sb are rewritten by the next element
  }
  cp_async_wait_all();
}

// ------------------------------------------------------------------------
// P = 7 (P1 = 8) NS2D physical viscous operator (visc2d.cu k2_visc semantics:
// Stokes stress + Fourier heat flux as a tensor SIP, problems.py:221-237
// generalised to 2-D, oracle/dg2d.py apply_viscous), one warp per element on the
// fp64 tensor cores:
//   * own-node gradients of the four fields as the 8 x 8 contractions U D^T and
//     D U (mma.m8n8k4.f64, the lane's node pair in the accumulator fragment), one
//     viscous-flux evaluation per node, fluxes to the warp's shared region;
//   * faces: lane = face * 8 + k owns one face node.  The OWN side's flux is the one
//     the node pass just stored; only the neighbour side is evaluated here (normal
//     derivative: the D row dotted with the neighbour's line through the node;
//     tangential derivative: D[k][.] dotted with the neighbour's face trace), then
//     G_nn [u] of both sides.  The line-formulated kernel evaluated both sides of
//     every face node from scratch (twice the gradient work of the node pass);
//   * divergence: F^x DTW^T and DTW F^y on the tensor cores, face and adjoint-lift
//     terms per node pair, 16-byte stores.
// The warp runs a two-stage cp.async pipeline over its elements (the next
// element and its four face neighbours land while this one is contracted).
struct Vs8 {                 // per-warp shared region (doubles)
  static constexpr int RP = 10, NP = 80, NC = 4;
  static constexpr int OWN = 0;                       // [2 stages][NC][NP] own element (padded rows)
  static constexpr int NBR = OWN + 2 * NC * NP;       // [2 stages][4 faces][NC][64] neighbour lines (swizzled)
  static constexpr int FX = NBR + 2 * 4 * NC * 64;    // [NC][NP] viscous fluxes F^x, F^y at the own nodes
  static constexpr int FY = FX + NC * NP;
  static constexpr int GF = FY + NC * NP;             // [32 face nodes][NC] face fluxes
  static constexpr int LF = GF + 32 * NC;             // [32 face nodes][NC] own-side G_nn [u] (adjoint lifts)
  static constexpr int WARP = LF + 32 * NC;
};
constexpr int VS_WARPS = 4;

__global__ void __launch_bounds__(VS_WARPS * 32, 2) k2_visc8(Op2DDev op, const double* __restrict__ u,
                                                             double* __restrict__ fo, int m_first, int accumulate,
                                                             int* status) {
  extern __shared__ double sm[];
  using W = Vs8;
  constexpr int RP = 10, P = 7, NC = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ws = sm + warp * W::WARP;
  const int m = m_first + blockIdx.y;
  const long long nn = op.nn;
  const double* um = u + (size_t)m * op.ns;
  double* fm = fo + (size_t)m * op.ns;
  const double gpr = op.gamma / op.pr;
  MmaLane K;
  mma_lane_init(op, K);
  const double rhx[2] = {1.0 / K.hwx[0], 1.0 / K.hwx[1]}, rhy = 1.0 / K.hwy;   // 1 / (h w / 2): the mass
  const int g = lane >> 2, t = lane & 3, n0 = 2 * t, cc = n0;
  const int f = lane >> 3, k = lane & 7;
  const int axis = f < FT ? 0 : 1;
  const bool own_minus = f == FR || f == FT;
  const int ownf = f == FR ? k * RP + P : f == FL ? k * RP : f == FT ? P * RP + k : k;   // own face node (padded)
  const int fpos = own_minus ? 0 : P;                   // the neighbour's face node on each of its lines
  const int npos = nsw(k, fpos);
  const int swz = g * 8 + 2 * ((lane & 3) ^ (g >> 1));
  const int tr0 = nsw(lane & 7, lane >> 3), tr1 = nsw(lane & 7, 4 + (lane >> 3));
  double dtan[8];   // D[k][.]: tangential derivative along the face at this lane's face node
  {
    const double* D = op.tab + TabOff::D(8);
#pragma unroll
    for (int q = 0; q < 8; ++q) dtan[q] = D[k * 8 + q];
  }
  const int ne = op.nex * op.ney;
  const int stride = gridDim.x * VS_WARPS;
  auto issue = [&](int e, int sb) {
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    const int exr = ex + 1 == op.nex ? 0 : ex + 1, exl = ex == 0 ? op.nex - 1 : ex - 1;
    const int eyt = ynb(op, ey, 1), eyb = ynb(op, ey, -1);
    const unsigned eo = ((unsigned)ey * op.nex + ex) * 64u;
    const unsigned nbR = ((unsigned)ey * op.nex + exr) * 64u, nbL = ((unsigned)ey * op.nex + exl) * 64u;
    const unsigned nbT = ((unsigned)eyt * op.nex + ex) * 64u, nbB = ((unsigned)eyb * op.nex + ex) * 64u;
    double* own = ws + W::OWN + sb * NC * W::NP;
    double* nbr = ws + W::NBR + sb * 4 * NC * 64;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double* uc = um + c * nn;
      cp_async16(own + c * W::NP + g * RP + cc, uc + eo + 2 * lane);
      cp_async16(nbr + (FR * NC + c) * 64 + swz, uc + nbR + 2 * lane);
      cp_async16(nbr + (FL * NC + c) * 64 + swz, uc + nbL + 2 * lane);
      cp_async8(nbr + (FT * NC + c) * 64 + tr0, uc + nbT + lane);
      cp_async8(nbr + (FT * NC + c) * 64 + tr1, uc + nbT + 32 + lane);
      cp_async8(nbr + (FB * NC + c) * 64 + tr0, uc + nbB + lane);
      cp_async8(nbr + (FB * NC + c) * 64 + tr1, uc + nbB + 32 + lane);
    }
  };
  int e = blockIdx.x * VS_WARPS + warp;
  if (e >= ne) return;
  issue(e, 0);
  cp_async_commit();
  int sb = 0;
  for (; e < ne; e += stride, sb ^= 1) {
    if (e + stride < ne) issue(e + stride, sb ^ 1);
    cp_async_commit();    // one group per element (possibly empty)
    cp_async_wait_1();    // this element's group has landed
    __syncwarp();
    const double* own = ws + W::OWN + sb * NC * W::NP;
    const double* nbr = ws + W::NBR + sb * 4 * NC * 64;
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    const long long gi = (long long)(((unsigned)ey * op.nex + ex) * 64u) + g * 8 + n0;
    // accumulate mode: this node pair's f values are fetched now, behind the contractions
    double2 facc[NC];
    if (accumulate) {
#pragma unroll
      for (int c = 0; c < NC; ++c) facc[c] = *reinterpret_cast<const double2*>(fm + c * nn + gi);
    }
    // ---- own nodes: gradients on the tensor cores, one flux evaluation per node
    {
      double gx[2][NC], gy[2][NC], s[2][NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double* Ue = own + c * W::NP;
        double qx0 = 0.0, qx1 = 0.0, qy0 = 0.0, qy1 = 0.0;
        dmma(qx0, qx1, Ue[g * RP + t], K.d0);
        dmma(qx0, qx1, Ue[g * RP + 4 + t], K.d1);
        dmma(qy0, qy1, K.d0, Ue[t * RP + g]);
        dmma(qy0, qy1, K.d1, Ue[(4 + t) * RP + g]);
        gx[0][c] = op.sx * qx0; gx[1][c] = op.sx * qx1;
        gy[0][c] = op.sy * qy0; gy[1][c] = op.sy * qy1;
        const double2 v = *reinterpret_cast<const double2*>(Ue + g * RP + n0);
        s[0][c] = v.x; s[1][c] = v.y;
      }
      double Fx[2][NC], Fy[2][NC];
      visc_flux(op, gpr, s[0], gx[0], gy[0], Fx[0], Fy[0]);
      visc_flux(op, gpr, s[1], gx[1], gy[1], Fx[1], Fy[1]);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        *reinterpret_cast<double2*>(ws + W::FX + c * W::NP + g * RP + n0) = make_double2(Fx[0][c], Fx[1][c]);
        *reinterpret_cast<double2*>(ws + W::FY + c * W::NP + g * RP + n0) = make_double2(Fy[0][c], Fy[1][c]);
      }
    }
    __syncwarp();
    // ---- faces: this lane's face node (face f, line k)
    {
      double so[NC], sn[NC], jmp[NC], gn[NC], gt[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double* ln = nbr + (f * NC + c) * 64 + k * 8;       // the neighbour's line through the node
        double an = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {                              // nodes 2j, 2j + 1 of the line, in order
          const double2 v = *reinterpret_cast<const double2*>(ln + 2 * (j ^ (k >> 1)));
          an = fma(K.drow[2 * j], v.x, an);
          an = fma(K.drow[2 * j + 1], v.y, an);
        }
        const double* fc = nbr + (f * NC + c) * 64;                // its face trace: node fpos of every line
        double at = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) at = fma(dtan[q], fc[nsw(q, fpos)], at);
        gn[c] = an;
        gt[c] = at;
        so[c] = own[c * W::NP + ownf];
        sn[c] = fc[npos];
        jmp[c] = own_minus ? so[c] - sn[c] : sn[c] - so[c];        // [u] = u- - u+
      }
      double gxn[NC], gyn[NC], Fxn[NC], Fyn[NC], g_nb[NC], g_own[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        gxn[c] = op.sx * (axis == 0 ? gn[c] : gt[c]);
        gyn[c] = op.sy * (axis == 0 ? gt[c] : gn[c]);
      }
      visc_flux(op, gpr, sn, gxn, gyn, Fxn, Fyn);
      apply_gnn(op, gpr, sn, jmp, axis, g_nb);
      apply_gnn(op, gpr, so, jmp, axis, g_own);
      const double mu0 = axis == 0 ? op.mux : op.muy;
      const double* Fo = ws + (axis == 0 ? W::FX : W::FY);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double q_own = Fo[c * W::NP + ownf], q_nb = axis == 0 ? Fxn[c] : Fyn[c];
        // minus side first, as the line-formulated kernel sums them
        const double gsum = own_minus ? g_own[c] + g_nb[c] : g_nb[c] + g_own[c];
        const double qsum = own_minus ? q_own + q_nb : q_nb + q_own;
        ws[W::GF + lane * NC + c] = mu0 * (0.5 * gsum) - 0.5 * qsum;
        ws[W::LF + lane * NC + c] = g_own[c];
      }
    }
    __syncwarp();
    // ---- divergence
    bool bad = false;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double* FX = ws + W::FX + c * W::NP;
      const double* FY = ws + W::FY + c * W::NP;
      double bx0 = 0.0, bx1 = 0.0, by0 = 0.0, by1 = 0.0;
      dmma(bx0, bx1, FX[g * RP + t], K.w0);
      dmma(bx0, bx1, FX[g * RP + 4 + t], K.w1);
      dmma(by0, by1, K.w0, FY[t * RP + g]);
      dmma(by0, by1, K.w1, FY[(4 + t) * RP + g]);
      const double* GF = ws + W::GF + c;
      const double* LF = ws + W::LF + c;
      if (n0 + 1 == P) bx1 += GF[(FR * 8 + g) * NC];
      if (n0 == 0) bx0 -= GF[(FL * 8 + g) * NC];
      const double lr = op.sx * (0.5 * LF[(FR * 8 + g) * NC]), ll = op.sx * (0.5 * LF[(FL * 8 + g) * NC]);
      bx0 -= lr * K.dPn[0];
      bx1 -= lr * K.dPn[1];
      bx0 -= ll * K.d0n[0];
      bx1 -= ll * K.d0n[1];
      if (g == P) { by0 += GF[(FT * 8 + n0) * NC]; by1 += GF[(FT * 8 + n0 + 1) * NC]; }
      if (g == 0) { by0 -= GF[(FB * 8 + n0) * NC]; by1 -= GF[(FB * 8 + n0 + 1) * NC]; }
      by0 -= (op.sy * (0.5 * LF[(FT * 8 + n0) * NC])) * K.dPg;
      by1 -= (op.sy * (0.5 * LF[(FT * 8 + n0 + 1) * NC])) * K.dPg;
      by0 -= (op.sy * (0.5 * LF[(FB * 8 + n0) * NC])) * K.d0g;
      by1 -= (op.sy * (0.5 * LF[(FB * 8 + n0 + 1) * NC])) * K.d0g;
      const double fv0 = -bx0 * rhx[0] + -by0 * rhy, fv1 = -bx1 * rhx[1] + -by1 * rhy;
      const double o0 = accumulate ? facc[c].x + fv0 : fv0, o1 = accumulate ? facc[c].y + fv1 : fv1;
      *reinterpret_cast<double2*>(fm + c * nn + gi) = make_double2(o0, o1);
      bad |= !isfinite(o0) || !isfinite(o1);
    }
    if (bad && status) atomicMin(status, (int)(op.e0 + e));
    __syncwarp();   // FX / FY / GF / LF and stage sb are rewritten by the next element
  }
  cp_async_wait_all();
}

template <int P1, int NC>
__global__ void __launch_bounds__(256, 2) k2_cg(Cg2Args A) {
  extern __shared__ double sm[];
  using L = CgSm<P1, NC>;
  using T = CT<P1>;
  cg::grid_group grid = cg::this_grid();
  const Op2DDev& op = A.op;
  constexpr int NN = P1 * P1, P = P1 - 1, EB = Blk<P1>::EB;
  constexpr int nc = NC;
  // p / x deferred into phase B only where phase B is issue bound (P = 7 tensor-core
  // path); the register-lean lower-degree matvecs are latency bound, and extra
  // dependent loads there cost more than the streaming pass saves
  constexpr bool DEFER = P1 == 8;
  const long long nn = op.nn;
  const int G = gridDim.x;
  const int tpr = (op.nex + EB - 1) / EB, ntiles = tpr * op.ney;
  const long long nthr = (long long)G * blockDim.x;
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool vec = (nn & 1) == 0 && ((reinterpret_cast<uintptr_t>(A.x) & 15) == 0);
  double* red = sm + L::RED;
  // per-block partials of three sums -> slot[blockIdx]
  auto block_part = [&](double v0, double v1, double v2, double* slot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
      v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    __syncthreads();
    if (lane == 0) { red[wid * 4] = v0; red[wid * 4 + 1] = v1; red[wid * 4 + 2] = v2; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;
      for (int ww = 0; ww < nw; ++ww) { t0 += red[ww * 4]; t1 += red[ww * 4 + 1]; t2 += red[ww * 4 + 2]; }
      slot[blockIdx.x * 4] = t0; slot[blockIdx.x * 4 + 1] = t1; slot[blockIdx.x * 4 + 2] = t2;
    }
  };
  // after a grid barrier: every block sums all slots in the same fixed order
  auto grid_total = [&](const double* slot, double (&t)[3]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int b = threadIdx.x; b < G; b += blockDim.x) { v0 += slot[b * 4]; v1 += slot[b * 4 + 1]; v2 += slot[b * 4 + 2]; }
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
      v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    __syncthreads();
    if (lane == 0) { red[wid * 4] = v0; red[wid * 4 + 1] = v1; red[wid * 4 + 2] = v2; }
    __syncthreads();
    t[0] = t[1] = t[2] = 0.0;
    for (int ww = 0; ww < nw; ++ww) { t[0] += red[ww * 4]; t[1] += red[ww * 4 + 1]; t[2] += red[ww * 4 + 2]; }
  };
  double* slot0 = A.part;
  double* slot1 = A.part + 4 * G;
  if (A.timing != nullptr && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == G - 1))
    A.timing[blockIdx.x == 0 ? 30 : 40] = gtimer();   // kernel start (setup stamps 30.. / 40..)

  // ---- setup 1: C per in-field node (pointwise, every node in flight at once),
  // then dinv = 1 / diag(M + a B2) in closed form from C (own element row and
  // column, the four neighbours' face nodes); same values and operations as a
  // per-element tile evaluation
  const int ne_own = op.nex * op.ney;
  const long long nown = (long long)ne_own * NN;
  if (A.mode != 2) {   // mode 2: Cf and DINV were filled by k2_coef / k2p_dinv at full occupancy
  for (long long f0 = gtid; f0 < nown; f0 += 4 * nthr) {   // 4 nodes per thread in flight
    double cv[4];
    long long fs[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long f = f0 + q * nthr;
      const long long fc = f < nown ? f : f0;
      const int e = (int)(fc / NN), nd = (int)(fc - (long long)e * NN);
      const int oy = e / op.nex, ex = e - oy * op.nex;
      fs[q] = f < nown ? (long long)((oy + op.row0) * op.nex + ex) * NN + nd : -1;
      cv[q] = coef2d(op, A.coef, oy + op.row0, ex, nd / P1, nd - (nd / P1) * P1);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (fs[q] >= 0) A.Cf[fs[q]] = cv[q];
  }
  grid.sync();
  for (long long f = gtid; f < nown; f += nthr) {
    const int e = (int)(f / NN), nd = (int)(f - (long long)e * NN);
    const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
    const int j = nd / P1, i = nd - j * P1;
    const int exr = wrapi(ex + 1, op.nex), exl = wrapi(ex - 1, op.nex);
    const int eyt = ynb(op, ey, 1), eyb = ynb(op, ey, -1);
    const double* CS = A.Cf + (long long)(ey * op.nex + ex) * NN;
    double dx_ = 0.0, dy_ = 0.0;
#pragma unroll
    for (int q = 0; q < P1; ++q) {
      dx_ = fma(c_tab2[T::D2W + i * P1 + q], CS[j * P1 + q], dx_);
      dy_ = fma(c_tab2[T::D2W + j * P1 + q], CS[q * P1 + i], dy_);
    }
    const double DPP = c_tab2[T::D + P * P1 + P], D00 = c_tab2[T::D];
    dx_ *= op.sx;
    dy_ *= op.sy;
    if (i == P) dx_ += op.mux * (0.5 * (CS[j * P1 + P] + A.Cf[(long long)(ey * op.nex + exr) * NN + j * P1])) -
                       op.sx * CS[j * P1 + P] * DPP;
    if (i == 0) dx_ += op.mux * (0.5 * (A.Cf[(long long)(ey * op.nex + exl) * NN + j * P1 + P] + CS[j * P1])) +
                       op.sx * CS[j * P1] * D00;
    if (j == P) dy_ += op.muy * (0.5 * (CS[P * P1 + i] + A.Cf[(long long)(eyt * op.nex + ex) * NN + i])) -
                       op.sy * CS[P * P1 + i] * DPP;
    if (j == 0) dy_ += op.muy * (0.5 * (A.Cf[(long long)(eyb * op.nex + ex) * NN + P * P1 + i] + CS[i])) +
                       op.sy * CS[i] * D00;
    const double hwx = 0.5 * op.dx * c_tab2[T::W + i], hwy = 0.5 * op.dy * c_tab2[T::W + j];
    A.DINV[(long long)(ey * op.nex + ex) * NN + nd] = 1.0 / (hwx * hwy + A.a * (hwy * dx_ + hwx * dy_));
  }
  }
  const bool stamps = A.timing != nullptr && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == G - 1);
  long long* ts = A.timing + (blockIdx.x == 0 ? 30 : 40);
  if (stamps) ts[1] = gtimer();   // setup 1 tiles done
  // (no initialisation pass: setup 2 writes x0 = rhs and p = 0, the first
  // iteration's phase A' reads s = 0)
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // phase-A chunk counters
    reinterpret_cast<unsigned*>(A.scal)[0] = 0u;
    reinterpret_cast<unsigned*>(A.scal)[1] = 0u;
  }
  grid.sync();
  if (stamps) ts[2] = gtimer();
  // ---- setup 2: r0 = b - A x0 (x0 = rhs, b = M rhs), u0 = r0 dinv, x = x0 and
  // p = 0 in the same epilogue; partials (b,b), #nonzero -> slot 0
  double ru0 = 0.0, rr0 = 0.0;
  {
    double bb = 0.0, nz = 0.0;
    auto epi = [&](long long g, double ax, double v) {   // v = x0 at g = rhs[g]
      const int nd = (int)(g % NN);
      const double mi = (0.5 * op.dx * c_tab2[T::W + nd % P1]) * (0.5 * op.dy * c_tab2[T::W + nd / P1]);
      const double b = mi * v;
      const double r = b - ax;
      A.R[g] = r;
      const double u = r * A.DINV[g % nn];
      A.U[g] = u;
      A.x[g] = v;      // x0 = rhs
      A.Pv[g] = 0.0;   // p_{-1} = 0
      bb = fma(b, b, bb);
      nz += b != 0.0 ? 1.0 : 0.0;
    };
    if constexpr (P1 == 8) {
      wpe_phase<NC>(op, sm, A.rhs, A.Cf, A.a, [&](long long g, double w0, double w1, double v0, double v1) {
        epi(g, w0, v0);
        epi(g + 1, w1, v1);
      });
    } else if constexpr (P1 == 4) {
      wph_phase<NC>(op, A.rhs, A.Cf, A.a, epi);
    } else {
      for (int tile = blockIdx.x; tile < ntiles; tile += G) cg_tile<P1, NC>(op, sm, tile, tpr, A.rhs, nullptr, A.Cf, A.a, epi);
    }
    block_part(bb, nz, 0.0, slot0);
  }
  grid.sync();
  double tot[3];
  grid_total(slot0, tot);
  const double thr = A.dbg ? -1.0 : A.rtol2 * tot[0];   // diagnostics: fixed iteration count
  if (tot[1] == 0.0) {   // b == 0 -> zeros (dgsem.py:510-511)
    for (long long t = gtid; t < op.n; t += nthr) A.x[t] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (A.mode != 0) A.scal[7] = 0.0;   // nothing left for k2_cgf
      int idx = atomicAdd(&A.status[2], 1);
      if (idx < A.log_cap) { A.log_it[idx] = 0; A.log_margin[idx] = 0.0; }
    }
    return;
  }
  // phase B body: w = A un; partial (w,un); with Up, the deferred p / x update
  // of this iteration (p = Up + beta p, x += alpha p) at the same nodes
  auto phase_B = [&](const double* Un, const double* Up, double al, double be) {
    double wu = 0.0;
    if constexpr (P1 == 8) {
      long long ta[3] = {0, 0, 0};
      const bool tw = A.timing != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
      wpe_phase<NC>(op, sm, Un, A.Cf, A.a, [&](long long g, double w0, double w1, double v0, double v1) {
        *reinterpret_cast<double2*>(A.W + g) = make_double2(w0, w1);
        wu = fma(w0, v0, wu);
        wu = fma(w1, v1, wu);
      }, tw ? ta : nullptr, PxArgs{Up, A.Pv, A.x, al, be});
      if (tw) { A.timing[20] += ta[0]; A.timing[21] += ta[1]; A.timing[22] += ta[2]; }
    } else {
      auto epi = [&](long long g, double wv, double u) {
        A.W[g] = wv;
        wu = fma(wv, u, wu);
        if (Up) cg_px1(A, Up, g, al, be);
      };
      if constexpr (P1 == 4) {
        wph_phase<NC>(op, Un, A.Cf, A.a, epi);
      } else {
        for (int tile = blockIdx.x; tile < ntiles; tile += G) cg_tile<P1, NC>(op, sm, tile, tpr, Un, nullptr, A.Cf, A.a, epi);
      }
    }
    return wu;
  };
  // ---- setup 3: w0 = A u0 (u0 from setup 2); gamma, delta, rho -> slot 1.  The
  // partials (r0,u0), (r0,r0) keep their node-major summation order (a read-only
  // pass: u0 = r0 dinv is recomputed bitwise, not stored again)
  {
    for (long long f = gtid; f < nn; f += nthr) {
      const double di = A.DINV[f];
#pragma unroll
      for (int c = 0; c < NC_MAX; ++c)
        if (c < nc) {
          const double r = A.R[c * nn + f], u = r * di;
          ru0 = fma(r, u, ru0);
          rr0 = fma(r, r, rr0);
        }
    }
    if (stamps) ts[3] = gtimer();
    const double wu = phase_B(A.U, nullptr, 0.0, 0.0);
    block_part(ru0, wu, rr0, slot1);
  }
  grid.sync();
  if (stamps) ts[4] = gtimer();
  grid_total(slot1, tot);
  double rho = tot[2];
  double alpha = tot[0] / tot[1], beta = 0.0;
  double rgam = 1.0 / tot[0], ralpha = 1.0 / alpha;
  if (A.mode != 0) {   // setup only: the iterations run in k2_cgf
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.scal[2] = thr; A.scal[3] = rho; A.scal[4] = alpha; A.scal[5] = rgam; A.scal[6] = ralpha; A.scal[7] = 1.0;
    }
    return;
  }
  int k = 0;
  bool ok = true;
  const bool stampb = A.timing != nullptr && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == G - 1);
  long long* tm = A.timing + (blockIdx.x == 0 ? 0 : 10);
  while (rho > thr) {
    if (k >= (A.dbg ? 10 : A.maxit)) { ok = false; break; }
    const bool stamp = stampb && k == 2;
    if (stamp) tm[0] = gtimer();
    // phase A': s = w + beta s, r -= alpha s, u_new = r dinv (p, x in phase B)
    double* const Un = (k & 1) ? A.U : A.U2;     // register selects: no local-memory array
    const double* const Up = (k & 1) ? A.U2 : A.U;
    double ru = 0.0, rr = 0.0;
    if (vec) {   // grid-stride over in-field pairs (no per-chunk block barrier)
      const long long nh = nn >> 1;
      for (long long h = gtid; h < nh; h += nthr) {
        if constexpr (DEFER) cg_update2s<NC>(A, Un, h, nh, alpha, beta, ru, rr, k == 0);
        else cg_update2<NC>(A, Un, h, nh, alpha, beta, ru, rr, k == 0);
      }
    } else {
      for (long long f = gtid; f < nn; f += nthr) {
        if constexpr (DEFER) cg_update1s<NC>(A, Un, f, nn, alpha, beta, ru, rr, k == 0);
        else cg_update1<NC>(A, Un, f, nn, alpha, beta, ru, rr, k == 0);
      }
    }
    if (stamp) tm[1] = gtimer();
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<unsigned*>(A.scal)[k & 1] = 0u;   // next use: k+2
    if (stamp) tm[2] = gtimer();
    const double wu = phase_B(Un, DEFER ? Up : nullptr, alpha, beta);
    if (stamp) tm[3] = gtimer();
    double* slot = (k & 1) ? slot1 : slot0;
    block_part(ru, wu, rr, slot);
    if (stamp) tm[4] = gtimer();
    grid.sync();
    if (stamp) tm[5] = gtimer();
    grid_total(slot, tot);
    if (stamp) tm[6] = gtimer();
    const double gn = tot[0];
    const double be = gn * rgam;
    const double al = gn / (tot[1] - be * (gn * ralpha));
    rho = tot[2];
    alpha = al;
    beta = be;
    rgam = 1.0 / gn;
    ralpha = 1.0 / al;
    ++k;
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

// ------------------------------------------------------------------------
// P = 7 fused single-pass PCG iteration (k2_cgf).  k2_cg streams every vector
// twice per iteration (phase A' then phase B: 13.5 vector passes = 108 B/DOF).
// Here ONE pass per iteration does the vector update and the matvec:
//   s' = w + beta s, r' = r - alpha s', u' = r' dinv, p = u + beta p,
//   x += alpha p, w' = (M + a B2) u', partials (r',u'), (w',u'), (r',r')
// -- 10.5 vector passes = 84 B/DOF.  w' at an element needs u' of its four face
// neighbours, which do not exist in memory: every u' is REBUILT on chip from
// (r, s, w, dinv) with the owner's exact operations (bitwise the same u', as
// the 1-D cluster CG does for its halo); r, s, w are double-buffered across
// iterations so that neighbours always read the previous iterate.
//   A block marches a band of 8 element rows (one warp per row) along a strip
// of SL elements of one field, one element column per step.  Warp y builds u'
// of element (y, j+1) once -- into its private 3-slot ring (x-neighbours: the
// ring holds columns j-1, j, j+1) and, transposed, into the block's ring RT,
// where the warps of rows y-1 / y+1 read it as their top / bottom neighbour.
// Only the two rows bordering the band are rebuilt redundantly (by a warp
// that rotates with the step).  The warps of a block are coupled by ONE mbarrier
// per step, split into arrive (column j+1 written) and wait (before the
// matvec of column j reads the neighbours' column j), so a warp only waits when
// a neighbour is a whole step behind; RT has four slots for that.  Operands arrive
// by TMA bulk copies (cp.async.bulk, one 512-byte run per element vector, five
// per warp and step from one lane) on per-warp mbarriers, two steps ahead.
// SUB = 2 (P = 3 levels with even nex, ney): a tile is a 2 x 2 block of 4 x 4-node elements.  With
// block-diagonal D / DTW (blockdiag(D4, D4)) the 8 x 8 contractions are the four elements' own
// contractions (the zero blocks add exact zeros), the tile's outer faces are handled as for SUB = 1
// (the zero half of the face rows drops the far sub-element) and the faces BETWEEN the sub-elements
// are extra lines whose both sides sit in the tile.  Per node the operations and their order are
// wph_phase's; the coarse level gets the single pass, the band / strip pipeline and the tensor-core
// contractions instead of ~30 shuffles per node and field.
template <int NC, int SUB = 1>
struct Fz {
  static constexpr int SL = SUB == 1 ? 16 : 8;      // strip length (tiles)
  static constexpr int NW = 8;                      // warps per block = rows per band
  static constexpr int NN = 64;
  // per-warp region (doubles)
  static constexpr int RAW = 0;                     // [2 stages][r, s, w, dinv of column j+1 | cf of column j][64]
  static constexpr int CFN = RAW + 2 * 5 * NN;      // [32] neighbour face coefficients
  static constexpr int RING = CFN + 32;             // [3][64] u' of columns j-1, j, j+1 (sw8 layout)
  static constexpr int QX = RING + 3 * NN, QY = QX + NN, DOT = QY + NN, FCON = DOT + 32;
  static constexpr int WARP = FCON + 64 * SUB;      // SUB = 2: + the internal faces' constants
  // block region
  static constexpr int RT = NW * WARP;              // [4 slots][NW + 2 rows][64] u' transposed + swizzled
  static constexpr int HRAW = RT + 4 * (NW + 2) * NN;   // [2 halo rows][2 stages][r, s, w, dinv][64]
  static constexpr int RED = HRAW + 2 * 2 * 4 * NN; // [32][4] block reduction scratch
  static constexpr int MBAR = RED + 128;            // [NW][2] own stages, [2][2] halo stages, column barrier
  static constexpr int SIZE = MBAR + 2 * NW + 6;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar2_init(uint32_t m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(m), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar2_expect(uint32_t m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar2_wait(uint32_t m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(m),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on the mbarrier (UBLKCP)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const double* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// 8 x 8 tiles of the fused pass (ring slots, RT rows, QX / QY): node (row, col) at
// row * 8 + 16-byte chunk (col / 2) ^ S(row), S = (0, 2, 1, 3)[row / 2].  Bank-conflict
// free for every access pattern of fz_sip: the lane's node pair (128-bit, rows g), the
// tensor-core A fragments (row g, col t / t + 4) and B fragments (row t / t + 4, col g)
// as 64-bit loads, and whole rows read by eight lanes (face lines).  Rows padded to 10
// cost two wavefronts per quarter warp on the 128-bit pair accesses and 4 instead of 2
// on the fragment loads (ncu: 36% excessive shared wavefronts, l1tex pipe at 79%).
__device__ __forceinline__ int sw8(int row, int col) {
  const int sr = ((row >> 1) & 1) * 2 + ((row >> 2) & 1);
  return row * 8 + ((((col >> 1) ^ sr)) << 1) + (col & 1);
}

// wpe_sip for the fused pass: own element Ue and the x-neighbours UR / UL (ring
// slots), the y-neighbours UT / UB transposed (face lines are rows), all in the
// sw8 layout; Ce row-major as the bulk copy delivers it.  FC: [16 lines][fp, fm]
// then [16 lines][adjoint + , adjoint -].  Same operations and order as wpe_sip.
struct FzLane {   // per-lane tile offsets (doubles), computed once per kernel
  int oA0, oA1, oB0, oB1, oP;   // A / B fragments, node pair
  int ln, lsw;                  // face line of this lane: row offset k * 8, chunk swizzle S(k)
  int up, u0, cu, c0, nP, n0_;  // lanes < 16: own face nodes (sw8 and raw order), neighbour face nodes
  int lraw;                     // this lane's node pair in the raw stage order (SUB = 1: 2 lane)
  int i3, i4, ci3, ci4;         // SUB = 2, lanes 16..31: the internal face's two nodes (sw8 / raw order)
};
// raw (memory) order of tile node (row, col): SUB = 1 row-major; SUB = 2 [element row][element][4][4]
template <int SUB>
__device__ __forceinline__ int raw_idx(int row, int col) {
  if constexpr (SUB == 1) return row * 8 + col;
  return (row >> 2) * 32 + (col >> 2) * 16 + (row & 3) * 4 + (col & 3);
}
template <int SUB>
__device__ __forceinline__ void fz_lane_init(FzLane& L) {
  constexpr int P = 7;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, k = lane & 7;
  L.oA0 = sw8(g, t); L.oA1 = sw8(g, t + 4); L.oB0 = sw8(t, g); L.oB1 = sw8(t + 4, g); L.oP = sw8(g, 2 * t);
  L.ln = k * 8;
  L.lsw = ((k >> 1) & 1) * 2 + ((k >> 2) & 1);
  const bool yd = (lane & 8) != 0;   // lanes 8..15 / 24..31: y-lines
  L.up = yd ? sw8(P, k) : sw8(k, P);
  L.u0 = yd ? sw8(0, k) : sw8(k, 0);
  L.cu = yd ? raw_idx<SUB>(P, k) : raw_idx<SUB>(k, P);
  L.c0 = yd ? raw_idx<SUB>(0, k) : raw_idx<SUB>(k, 0);
  L.nP = sw8(k, P);
  L.n0_ = sw8(k, 0);
  L.lraw = raw_idx<SUB>(g, 2 * t);
  L.i3 = yd ? sw8(3, k) : sw8(k, 3);
  L.i4 = yd ? sw8(4, k) : sw8(k, 4);
  L.ci3 = yd ? raw_idx<SUB>(3, k) : raw_idx<SUB>(k, 3);
  L.ci4 = yd ? raw_idx<SUB>(4, k) : raw_idx<SUB>(k, 4);
}
// MmaLane of a SUB = 2 tile from the P = 3 tables: block-diagonal D / DTW, the weights repeated
__device__ __forceinline__ void mma_lane_init_sub2(const Op2DDev& op, MmaLane& K) {
  const double* D = op.tab + TabOff::D(4);
  const double* DTW = op.tab + TabOff::DTW(4);
  const double* w = op.tab + TabOff::w(4);
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, f = lane >> 3, n0 = 2 * t;
  auto d8 = [&](const double* M, int r, int c) { return (r >> 2) == (c >> 2) ? M[(r & 3) * 4 + (c & 3)] : 0.0; };
  K.d0 = d8(D, g, t);
  K.d1 = d8(D, g, 4 + t);
  K.w0 = d8(DTW, g, t);
  K.w1 = d8(DTW, g, 4 + t);
  const int rr = (f == FL || f == FB) ? 7 : 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) K.drow[q] = d8(D, rr, q);
#pragma unroll
  for (int i = 0; i < 2; ++i) {   // per sub-element: D[P][.] and D[0][.] at this node's local column
    K.dPn[i] = D[3 * 4 + ((n0 + i) & 3)];
    K.d0n[i] = D[(n0 + i) & 3];
    K.hwx[i] = 0.5 * op.dx * w[(n0 + i) & 3];
  }
  K.dPg = D[3 * 4 + (g & 3)];
  K.d0g = D[g & 3];
  K.hwy = 0.5 * op.dy * w[g & 3];
  K.hh[0] = K.hwx[0] * K.hwy;
  K.hh[1] = K.hwx[1] * K.hwy;
  K.wn[0] = w[n0 & 3];
  K.wn[1] = w[(n0 + 1) & 3];
  K.wg = w[g & 3];
}
template <int SUB>
__device__ __forceinline__ void fz_sip(const Op2DDev& op, const MmaLane& K, const FzLane& L, const double* Ue,
                                       const double* UR, const double* UL, const double* UT, const double* UB,
                                       const double* Ce, const double* cfn, double* QX, double* QY, double* DT,
                                       double* FC, double& bx0, double& bx1, double& by0, double& by1) {
  constexpr int P = 7;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, n0 = 2 * t;
  const int oA0 = L.oA0, oA1 = L.oA1, oB0 = L.oB0, oB1 = L.oB1, oP = L.oP;
  double qx0 = 0.0, qx1 = 0.0, qy0 = 0.0, qy1 = 0.0;
  dmma(qx0, qx1, Ue[oA0], K.d0);
  dmma(qx0, qx1, Ue[oA1], K.d1);
  dmma(qy0, qy1, K.d0, Ue[oB0]);
  dmma(qy0, qy1, K.d1, Ue[oB1]);
  {
    const double2 cg = *reinterpret_cast<const double2*>(Ce + L.lraw);   // row g, columns n0, n0 + 1
    *reinterpret_cast<double2*>(QX + oP) = make_double2(cg.x * (op.sx * qx0), cg.y * (op.sx * qx1));
    *reinterpret_cast<double2*>(QY + oP) = make_double2(cg.x * (op.sy * qy0), cg.y * (op.sy * qy1));
  }
  {
    const int f = lane >> 3;
    const double* ln = (f == FR ? UR : f == FL ? UL : f == FT ? UT : UB) + L.ln;
    const int sw = L.lsw;
    double gd = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(ln + 2 * (j ^ sw));
      gd = fma(K.drow[2 * j], v.x, gd);
      gd = fma(K.drow[2 * j + 1], v.y, gd);
    }
    DT[lane] = cfn[lane] * ((f < FT ? op.sx : op.sy) * gd);
  }
  __syncwarp();
  bx0 = bx1 = by0 = by1 = 0.0;
  dmma(bx0, bx1, QX[oA0], K.w0);
  dmma(bx0, bx1, QX[oA1], K.w1);
  dmma(by0, by1, K.w0, QY[oB0]);
  dmma(by0, by1, K.w1, QY[oB1]);
  if (lane < 16) {
    const bool yd = lane >= 8;
    const int r = lane & 7;
    const int up = L.up, u0 = L.u0;     // own face nodes
    const int cu = L.cu, c0_ = L.c0;    // the same in raw order (Ce)
    const double jp = Ue[up] - (yd ? UT : UR)[L.n0_];
    const double jm = (yd ? UB : UL)[L.nP] - Ue[u0];
    const double cP = Ce[cu], c0 = Ce[c0_];
    const double fcp = cfn[(yd ? 16 : 0) + r], fcm = cfn[(yd ? 24 : 8) + r];
    const double qP = (yd ? QY : QX)[up], q0 = (yd ? QY : QX)[u0];
    const double qnp = DT[(yd ? 16 : 0) + r], qnm = DT[(yd ? 24 : 8) + r];
    const double mu = yd ? op.muy : op.mux, sc = yd ? op.sy : op.sx;
    const double fp = -(0.5 * (qP + qnp)) + (mu * (0.5 * (cP + fcp))) * jp;
    const double fm = -(0.5 * (qnm + q0)) + (mu * (0.5 * (fcm + c0))) * jm;
    *reinterpret_cast<double2*>(FC + lane * 2) = make_double2(fp, fm);
    *reinterpret_cast<double2*>(FC + 32 + lane * 2) = make_double2(sc * ((0.5 * cP) * jp), sc * ((0.5 * c0) * jm));
  } else if constexpr (SUB == 2) {
    // the face between the two sub-elements of line r (lanes 16..23: x-row r, 24..31: y-column r): both
    // sides in the tile.  Seen from the lower / left element it is the P face (own node 3, neighbour
    // node 4), from the upper / right one the 0 face; the numerical flux is the same expression with
    // the same operands in the same order for both (wph_phase's fpx and fmx), so it is formed once
    const bool yd = lane >= 24;
    const int ll = lane - 16;
    const double u3 = Ue[L.i3], u4 = Ue[L.i4], c3 = Ce[L.ci3], c4 = Ce[L.ci4];
    const double q3 = (yd ? QY : QX)[L.i3], q4 = (yd ? QY : QX)[L.i4];
    const double mu = yd ? op.muy : op.mux, sc = yd ? op.sy : op.sx;
    const double jmp = u3 - u4;
    const double fi = -(0.5 * (q3 + q4)) + (mu * (0.5 * (c3 + c4))) * jmp;
    *reinterpret_cast<double2*>(FC + 64 + ll * 2) = make_double2(fi, 0.0);
    *reinterpret_cast<double2*>(FC + 96 + ll * 2) = make_double2(sc * ((0.5 * c3) * jmp), sc * ((0.5 * c4) * jmp));
  }
  __syncwarp();
  if constexpr (SUB == 1) {
    const double2 rx = *reinterpret_cast<const double2*>(FC + g * 2);
    const double2 rz = *reinterpret_cast<const double2*>(FC + 32 + g * 2);
    if (n0 + 1 == P) bx1 += rx.x;
    if (n0 == 0) bx0 -= rx.y;
    bx0 -= rz.x * K.dPn[0];
    bx1 -= rz.x * K.dPn[1];
    bx0 -= rz.y * K.d0n[0];
    bx1 -= rz.y * K.d0n[1];
    // y-columns n0, n0 + 1: (fp, fm) of both in one 32-byte run, likewise the adjoint pair
    const double4 cf = *reinterpret_cast<const double4*>(FC + (8 + n0) * 2);
    const double4 cz = *reinterpret_cast<const double4*>(FC + 32 + (8 + n0) * 2);
    if (g == P) { by0 += cf.x; by1 += cf.z; }
    if (g == 0) { by0 -= cf.y; by1 -= cf.w; }
    by0 -= cz.x * K.dPg;
    by1 -= cz.z * K.dPg;
    by0 -= cz.y * K.d0g;
    by1 -= cz.w * K.d0g;
  } else {
    // per sub-element: P-face terms then 0-face terms (wph_phase's order).  Left / lower element: P face =
    // the internal one, 0 face = the tile's outer L / B; right / upper element: P face = outer R / T, 0 face
    // = internal.  K.dPn / d0n / dPg / d0g hold D4[3][.] / D4[0][.] at the node's local index.
    {
      const double2 ox = *reinterpret_cast<const double2*>(FC + g * 2);        // outer (fp R, fm L) of x-row g
      const double2 oz = *reinterpret_cast<const double2*>(FC + 32 + g * 2);   // outer adjoint (R, L)
      const double2 ix = *reinterpret_cast<const double2*>(FC + 64 + g * 2);   // internal flux
      const double2 iz = *reinterpret_cast<const double2*>(FC + 96 + g * 2);   // internal adjoint (node 3 side, node 4 side)
      const bool left = n0 < 4;
      const double fP = left ? ix.x : ox.x, f0 = left ? ox.y : ix.x;
      const double lP = left ? iz.x : oz.x, l0 = left ? oz.y : iz.y;
      if (((n0 + 1) & 3) == 3) bx1 += fP;
      if ((n0 & 3) == 0) bx0 -= f0;
      bx0 -= lP * K.dPn[0];
      bx1 -= lP * K.dPn[1];
      bx0 -= l0 * K.d0n[0];
      bx1 -= l0 * K.d0n[1];
    }
    {
      const double4 of = *reinterpret_cast<const double4*>(FC + (8 + n0) * 2);        // outer (fp T, fm B) of columns n0, n0+1
      const double4 oz = *reinterpret_cast<const double4*>(FC + 32 + (8 + n0) * 2);
      const double4 iy = *reinterpret_cast<const double4*>(FC + 64 + (8 + n0) * 2);   // internal flux of columns n0, n0+1
      const double4 iz = *reinterpret_cast<const double4*>(FC + 96 + (8 + n0) * 2);
      const bool low = g < 4;
      const double fP0 = low ? iy.x : of.x, fP1 = low ? iy.z : of.z;
      const double f00 = low ? of.y : iy.x, f01 = low ? of.w : iy.z;
      const double lP0 = low ? iz.x : oz.x, lP1 = low ? iz.z : oz.z;
      const double l00 = low ? oz.y : iz.y, l01 = low ? oz.w : iz.w;
      if ((g & 3) == 3) { by0 += fP0; by1 += fP1; }
      if ((g & 3) == 0) { by0 -= f00; by1 -= f01; }
      by0 -= lP0 * K.dPg;
      by1 -= lP1 * K.dPg;
      by0 -= l00 * K.d0g;
      by1 -= l01 * K.d0g;
    }
  }
}

// per-block partials of three sums -> slot[blockIdx] (fixed order)
__device__ __forceinline__ void blk_part3(double v0, double v1, double v2, double* red, double* slot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  }
  __syncthreads();
  if (lane == 0) { red[wid * 4] = v0; red[wid * 4 + 1] = v1; red[wid * 4 + 2] = v2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int ww = 0; ww < nw; ++ww) { t0 += red[ww * 4]; t1 += red[ww * 4 + 1]; t2 += red[ww * 4 + 2]; }
    slot[blockIdx.x * 4] = t0; slot[blockIdx.x * 4 + 1] = t1; slot[blockIdx.x * 4 + 2] = t2;
  }
}

// MODE 0: the iterations.  MODE 1 / 2: the two setup passes of a solve as single passes of the same
// pipeline (separate instantiations = separate launches, registers and code):
//   1  r0 = b - A x0 (x0 = rhs, b = M rhs) -> R, partials (b,b), #nonzero b -> slot 2
//   2  u0 = r0 dinv (rebuilt on chip), w0 = A u0 -> W, partials (r0,u0), (w0,u0), (r0,r0) -> slot 3
// MODE 0 then derives thr, rho, alpha from slots 2 / 3 itself (every block, one fixed order), reads x0 = rhs
// and p = 0 in its first iteration (no initialisation pass) and zero-fills x when b == 0.  With A.mode == 2
// (setup by k2_cg) it reads the scalars k2_cg left instead.
template <int NC, int SUB = 1, int MODE = 0>
__global__ void __launch_bounds__(256, 2) k2_cgf(Cg2Args A) {
  extern __shared__ double sm[];
  using F = Fz<NC, SUB>;
  // tile geometry: a tile is SUB x SUB elements of EN nodes; TW doubles of one element row per tile
  constexpr unsigned EN = 64u / (SUB * SUB), TW = 64u / SUB;
  constexpr uint32_t RUN = 512u / SUB;   // bytes of one contiguous run of a tile vector (SUB runs)
  cg::grid_group grid = cg::this_grid();
  const Op2DDev& op = A.op;
  constexpr int SL = F::SL, NW = F::NW;
  const long long nn = op.nn;
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);   // warp-uniform for the compiler
  double* ws = sm + warp * F::WARP;
  double* red = sm + F::RED;
  double* RT = sm + F::RT;
  const uint32_t mb_own = smem_u32(reinterpret_cast<unsigned long long*>(sm + F::MBAR) + 2 * warp);   // + 8 stage
  const uint32_t mb_halo = smem_u32(reinterpret_cast<unsigned long long*>(sm + F::MBAR) + 2 * NW);    // + 16 h + 8 stage
  const uint32_t mb_col = mb_halo + 32u;   // NW arrivals (one per warp) per step
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * NW + 4; ++i) mbar2_init(smem_u32(reinterpret_cast<unsigned long long*>(sm + F::MBAR) + i), 1);
    mbar2_init(mb_col, NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // single-pass mode (A.sc set: the split solve of an element-row partition, part2d.cu): ONE pass with the
  // scalars of the solve's CgPScal, buffer parity A.px, block partials to part / part2; no grid barrier
  const bool single = MODE != 0 || A.sc != nullptr;   // one pass, then block partials and return
  const bool own_setup = MODE == 0 && A.sc == nullptr && A.mode == 3;   // the solve was set up by MODE 1 / 2 launches
  double* const slot2 = A.part + 8 * G;    // MODE 1 partials
  double* const slot3 = A.part + 12 * G;   // MODE 2 partials
  // every block sums G slots of three values in one fixed order (bitwise-identical totals everywhere)
  auto slot_total = [&](const double* slot, double (&t)[3]) {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int b = threadIdx.x; b < G; b += blockDim.x) { v0 += slot[b * 4]; v1 += slot[b * 4 + 1]; v2 += slot[b * 4 + 2]; }
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
      v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    __syncthreads();
    if (lane == 0) { red[warp * 4] = v0; red[warp * 4 + 1] = v1; red[warp * 4 + 2] = v2; }
    __syncthreads();
    t[0] = t[1] = t[2] = 0.0;
    for (int ww = 0; ww < NW; ++ww) { t[0] += red[ww * 4]; t[1] += red[ww * 4 + 1]; t[2] += red[ww * 4 + 2]; }
    __syncthreads();
  };
  double thr = 0.0, rho = 1.0, alpha = 0.0, beta = 0.0, rgam = 0.0, ralpha = 0.0;
  if constexpr (MODE == 0) {
    if (A.sc != nullptr) {   // split solve of a partition: scalars of the solve's CgPScal
      if (A.sc->done != 0) return;
      alpha = A.sc->alpha;
      beta = A.sc->beta;
    } else if (own_setup) {
      double t2[3], t3[3];
      slot_total(slot2, t2);
      if (t2[1] == 0.0) {   // b == 0 -> zeros (dgsem.py:510-511)
        const long long nthr = (long long)G * blockDim.x;
        for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < op.n; t += nthr) A.x[t] = 0.0;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
          int idx = atomicAdd(&A.status[2], 1);
          if (idx < A.log_cap) { A.log_it[idx] = 0; A.log_margin[idx] = 0.0; }
        }
        return;
      }
      slot_total(slot3, t3);
      thr = A.dbg ? -1.0 : A.rtol2 * t2[0];
      rho = t3[2];
      alpha = t3[0] / t3[1];
      rgam = 1.0 / t3[0];
      ralpha = 1.0 / alpha;
    } else {                 // setup by k2_cg (mode 2)
      if (A.scal[7] == 0.0) return;   // b == 0 (x = 0 written by the setup)
      thr = A.scal[2]; rho = A.scal[3]; alpha = A.scal[4]; rgam = A.scal[5]; ralpha = A.scal[6];
    }
  } else if constexpr (MODE == 2) {
    if (A.sc == nullptr) {   // (a partition's own b may vanish while the solve's does not: no local shortcut)
      double t2[3];
      slot_total(slot2, t2);
      if (t2[1] == 0.0) return;   // b == 0: MODE 0 writes x = 0
    }
  }
  MmaLane K;
  if constexpr (SUB == 1) mma_lane_init(op, K); else mma_lane_init_sub2(op, K);
  FzLane L;
  fz_lane_init<SUB>(L);
  const unsigned epitch = (unsigned)op.nex * EN;   // doubles of one element row of one field
  // offset of tile node (row, col) from the tile's first node in memory
  auto toff = [&](int row, int col) -> unsigned {
    if constexpr (SUB == 1) return (unsigned)(row * 8 + col);
    return (unsigned)(row >> 2) * epitch + (unsigned)((col >> 2) * 16 + (row & 3) * 4 + (col & 3));
  };
  const unsigned lglob = toff(lane >> 2, 2 * (lane & 3));   // this lane's node pair
  double* slot0 = A.part;
  double* slot1 = A.part + 4 * G;
  const int g = lane >> 2, n0 = 2 * (lane & 3);
  const int f = lane >> 3, kf = lane & 7;
  const unsigned fnode = f == FR ? toff(kf, 0) : f == FL ? toff(kf, 7) : f == FT ? toff(0, kf) : toff(7, kf);   // neighbour's face node
  const int tr0 = sw8(lane & 7, lane >> 3), tr1 = sw8(lane & 7, 4 + (lane >> 3));   // node v -> line v%8, pos v/8
  const int hr0 = raw_idx<SUB>(lane >> 3, lane & 7), hr1 = raw_idx<SUB>(4 + (lane >> 3), lane & 7);   // the same nodes, raw order
  const int oP = L.oP;   // this lane's node pair in a tile
  // transposed position of this lane's own node pair (row g, columns n0, n0+1); odd rows store the second
  // node first so that one store instruction hits all 16 bank pairs
  const int ta = (g & 1) ? sw8(n0 + 1, g) : sw8(n0, g), tb = (g & 1) ? sw8(n0, g) : sw8(n0 + 1, g);
  const int nexT = op.nex / SUB, neyT = op.ney / SUB;   // tiles per row / tile rows (SUB = 2: even sizes only)
  const int nstr = (nexT + SL - 1) / SL, nbands = (neyT + NW - 1) / NW;
  // bands of this launch (A.bsel, single-pass mode): all; the interior ones; the two that read ghost rows
  const int nbsel = A.bsel == 0 ? nbands : A.bsel == 1 ? nbands - 2 : 2;
  const long long nunits = (long long)nbsel * nstr * NC;
  unsigned oc = 0, hc = 0;   // completed uses of this warp's own stages / of the halo stages (stage = use & 1)
  unsigned ac = 0;           // this warp's arrivals on the column barrier (= steps done)
  int st = 0;                // RT slot of column j (slots advance with j, four of them)
  int k = 0;
  bool ok = true;
  const bool stampb = A.timing != nullptr && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == G - 1);
  long long* tm = A.timing + (blockIdx.x == 0 ? 0 : 10);
  const int maxit = A.dbg ? 10 : A.maxit;
  while (rho > thr) {
    if (k >= maxit) { ok = false; break; }
    const bool stamp = stampb && k == 2;
    if (stamp) tm[0] = tm[1] = tm[2] = gtimer();
    const bool first = MODE != 0 ? true : (A.sc != nullptr ? A.sc->k == 0 : k == 0);
    const int par = MODE != 0 ? 0 : (A.sc != nullptr ? A.px : (k & 1));
    const bool x_from_rhs = own_setup && k == 0;   // x0 = rhs, p = 0: read, never initialised
    double bb = 0.0, nz = 0.0;                     // MODE 1 partials
    const double* const Ro = par ? A.R2 : A.R;
    const double* const So = par ? A.S2 : A.S;
    const double* const Wo = par ? A.W2 : A.W;
    double* const Rn = par ? A.R : A.R2;
    double* const Sn = par ? A.S : A.S2;
    double* const Wn = par ? A.W : A.W2;
    double ru = 0.0, rr = 0.0, wu = 0.0;
    for (long long un = blockIdx.x; un < nunits; un += G) {
      const int c = (int)(un % NC);
      const long long tq = un / NC;
      // bands fastest: the blocks in flight work on vertically adjacent bands of one strip column, so the
      // rows bordering a band (rebuilt from their raw r, s, w) are L2 hits, not a second DRAM read
      const int bq = (int)(tq % nbsel), sx = (int)(tq / nbsel);
      const int band = A.bsel == 0 ? bq : A.bsel == 1 ? bq + 1 : (bq == 0 ? 0 : nbands - 1);
      const int y0 = band * NW, nrows = neyT - y0 < NW ? neyT - y0 : NW;
      const bool valid = warp < nrows;
      // SUB = 1: the (storage) element row, a partition's ghost rows through ynb; SUB = 2: the tile row (trow maps it)
      const int ey = (valid ? y0 + warp : y0) + (SUB == 1 ? op.row0 : 0);
      const int x0 = sx * SL, x1 = x0 + SL < nexT ? x0 + SL : nexT;
      // offsets in doubles fit 32 bits (checked by the launcher: n < 2^32)
      const unsigned fo = (unsigned)(c * nn);
      // first node of a tile row: SUB = 1 the element row (ghost rows of a partition through ynb); SUB = 2
      // (single domain only) the lower of its two element rows, periodic in tile rows
      auto trow = [&](int ty, int d) -> unsigned {
        if constexpr (SUB == 1) return (unsigned)(d == 0 ? ty : ynb(op, ty, d)) * epitch;
        const int t2 = ty + d;
        if (op.row0 == 0) return (unsigned)((t2 < 0 ? neyT - 1 : t2 >= neyT ? 0 : t2) * SUB) * epitch;
        // partition: tile row t2 starts at storage element row row0 + 2 t2.  The tile row above the partition
        // has only its lower element row in storage (the top ghost row), the one below only its upper one
        // (the bottom ghost row; t2 = -1 wraps, and only offset + epitch is ever dereferenced): see issue_halo
        return (unsigned)(op.row0 + t2 * SUB) * epitch;
      };
      const bool top_out = SUB == 2 && op.row0 != 0 && y0 + nrows == neyT;   // the band's upper neighbour is the ghost row
      const bool bot_out = SUB == 2 && op.row0 != 0 && y0 == 0;
      const unsigned rowC = trow(ey, 0), rowT = trow(ey, 1), rowB = trow(ey, -1);
      const unsigned hrow0 = trow((SUB == 1 ? op.row0 : 0) + y0 + nrows - 1, 1);   // above the band
      const unsigned hrow1 = trow((SUB == 1 ? op.row0 : 0) + y0, -1);              // below the band
      const unsigned oC = fo + rowC + lglob;
      const unsigned cfb = (f == FT ? rowT : f == FB ? rowB : rowC) + fnode;   // this lane's face coefficient row
      // own stage of step js: r, s, w, dinv of column js+1, cf of column js (js >= x0)
      auto issue_own = [&](int js, unsigned use) {
        if (lane == 0) {
          const uint32_t mb = mb_own + 8u * (use & 1u);
          const uint32_t dst = smem_u32(ws + F::RAW + (use & 1u) * 320);
          int en = js + 1;
          en = en < 0 ? nexT - 1 : en >= nexT ? 0 : en;
          const unsigned e1 = fo + rowC + (unsigned)en * TW;
          const bool cf = js >= x0;
          constexpr uint32_t NV = MODE == 0 ? 4u : MODE == 1 ? 1u : 2u;   // r s w dinv | rhs | r dinv
          mbar2_expect(mb, (cf ? NV + 1u : NV) * 512u);
#pragma unroll
          for (int rn = 0; rn < SUB; ++rn) {   // SUB runs per tile vector (one per element row)
            const unsigned eo_ = e1 + rn * epitch;
            const uint32_t d = dst + rn * RUN;
            bulk_g2s(d, (MODE == 1 ? A.rhs : Ro) + eo_, RUN, mb);
            if constexpr (MODE == 0) {
              bulk_g2s(d + 512u, So + eo_, RUN, mb);
              bulk_g2s(d + 1024u, Wo + eo_, RUN, mb);
            }
            if constexpr (MODE != 1) bulk_g2s(d + 1536u, A.DINV + (eo_ - fo), RUN, mb);
            if (cf) bulk_g2s(d + 2048u, A.Cf + (rowC + rn * epitch + (unsigned)js * TW), RUN, mb);
          }
        }
      };
      // halo stage h (0 above, 1 below the band) of step js: r, s, w, dinv of column js+1
      auto issue_halo = [&](int h, int js, unsigned use) {
        if (lane == 0) {
          const uint32_t mb = mb_halo + 16u * h + 8u * (use & 1u);
          const uint32_t dst = smem_u32(sm + F::HRAW + (h * 2 + (use & 1u)) * 256);
          const unsigned e1 = fo + (h ? hrow1 : hrow0) + (unsigned)(js + 1) * TW;
          constexpr uint32_t NV = MODE == 0 ? 4u : MODE == 1 ? 1u : 2u;
          mbar2_expect(mb, NV * 512u);
#pragma unroll
          for (int rn = 0; rn < SUB; ++rn) {
            // a partition's ghost tile row holds ONE element row: the missing one is read from the ghost row
            // too (finite values that the block-diagonal face rows multiply by exact zeros)
            const int rs = (h == 0 && top_out) ? 0 : (h == 1 && bot_out) ? 1 : rn;
            const unsigned eo_ = e1 + rs * epitch;
            const uint32_t d = dst + rn * RUN;
            bulk_g2s(d, (MODE == 1 ? A.rhs : Ro) + eo_, RUN, mb);
            if constexpr (MODE == 0) {
              bulk_g2s(d + 512u, So + eo_, RUN, mb);
              bulk_g2s(d + 1024u, Wo + eo_, RUN, mb);
            }
            if constexpr (MODE != 1) bulk_g2s(d + 1536u, A.DINV + (eo_ - fo), RUN, mb);
          }
        }
      };
      auto cfn_load = [&](int col) {   // neighbour face coefficients of column col
        const int exr = col + 1 == nexT ? 0 : col + 1, exl = col == 0 ? nexT - 1 : col - 1;
        return A.Cf[cfb + (unsigned)(f == FR ? exr : f == FL ? exl : col) * TW];
      };
      // (no block barrier between units: warp 0 issues the halo stages below after its last wait on the
      // column barrier, which every warp passed after its last halo rebuild)
      // halo steps: js + 1 in [x0, x1 - 1]; two uses ahead
      if (valid) {
        issue_own(x0 - 2, oc);
        issue_own(x0 - 1, oc + 1);
      }
      if (warp == 0) {
        issue_halo(0, x0 - 1, hc);
        issue_halo(1, x0 - 1, hc);
        if (x0 + 1 < x1) {
          issue_halo(0, x0, hc + 1);
          issue_halo(1, x0, hc + 1);
        }
      }
      double cfn_reg = cfn_load(x0);
      double2 pp = make_double2(0.0, 0.0), xx = pp;
      int sl = 0;   // ring slot of column j - 1 (slots advance with j)
      // one step, specialised at compile time on own (column j + 1 lies inside the strip: its s', r',
      // p, x are written, the rows bordering the band are rebuilt) and sip (column j gets its w')
      auto step = [&](const int j, auto own_c, auto sip_c) {
        constexpr bool own = decltype(own_c)::value, sip = decltype(sip_c)::value;
        const int jn = j + 1;
        const int sN = sl == 0 ? 2 : sl - 1;        // slot of column j + 1: (sl + 2) % 3
        const int sJ = sl == 2 ? 0 : sl + 1;        // slot of column j
        const int tN = (st + 1) & 3;                // RT slot of column j + 1 (free: see the column barrier below)
        if (valid) {
          const unsigned gn = oC + (unsigned)jn * TW;   // used inside the strip only
          const double* raw = ws + F::RAW + (oc & 1u) * 320;
          mbar2_wait(mb_own + 8u * (oc & 1u), (oc >> 1) & 1u);
          if constexpr (MODE != 0) {   // setup passes: u' = x0 (MODE 1) or r0 dinv (MODE 2), nothing written here
            const double2 r = *reinterpret_cast<const double2*>(raw + L.lraw);
            double2 uu = r;
            if constexpr (MODE == 2) {
              const double2 di = *reinterpret_cast<const double2*>(raw + 192 + L.lraw);
              uu.x = r.x * di.x;
              uu.y = r.y * di.y;
            }
            *reinterpret_cast<double2*>(ws + F::RING + sN * 64 + oP) = uu;
            if (own) {
              double* rt = RT + (tN * (NW + 2) + warp) * 64;
              rt[ta] = (g & 1) ? uu.y : uu.x;
              rt[tb] = (g & 1) ? uu.x : uu.y;
              if constexpr (MODE == 2) {
                ru = fma(r.x, uu.x, ru);
                rr = fma(r.x, r.x, rr);
                ru = fma(r.y, uu.y, ru);
                rr = fma(r.y, r.y, rr);
              }
            }
          } else {   // u' of column j + 1 (and, inside the strip, its s', r', p, x)
            const double2 r = *reinterpret_cast<const double2*>(raw + L.lraw);
            double2 s = *reinterpret_cast<const double2*>(raw + 64 + L.lraw);
            const double2 w = *reinterpret_cast<const double2*>(raw + 128 + L.lraw);
            const double2 di = *reinterpret_cast<const double2*>(raw + 192 + L.lraw);
            if (first) s = make_double2(0.0, 0.0);
            double2 sn, rn, uu;
            sn.x = fma(beta, s.x, w.x);
            sn.y = fma(beta, s.y, w.y);
            rn.x = fma(-alpha, sn.x, r.x);
            rn.y = fma(-alpha, sn.y, r.y);
            uu.x = rn.x * di.x;
            uu.y = rn.y * di.y;
            *reinterpret_cast<double2*>(ws + F::RING + sN * 64 + oP) = uu;
            if (own) {
              double* rt = RT + (tN * (NW + 2) + warp) * 64;
              rt[ta] = (g & 1) ? uu.y : uu.x;
              rt[tb] = (g & 1) ? uu.x : uu.y;
              *reinterpret_cast<double2*>(Sn + gn) = sn;
              *reinterpret_cast<double2*>(Rn + gn) = rn;
              ru = fma(rn.x, uu.x, ru);
              rr = fma(rn.x, rn.x, rr);
              ru = fma(rn.y, uu.y, ru);
              rr = fma(rn.y, rn.y, rr);
              pp.x = fma(beta, pp.x, r.x * di.x);   // p = u_prev + beta p, u_prev = r_old dinv
              pp.y = fma(beta, pp.y, r.y * di.y);
              xx.x = fma(alpha, pp.x, xx.x);
              xx.y = fma(alpha, pp.y, xx.y);
              __stcs(reinterpret_cast<double2*>(A.Pv + gn), pp);
              __stcs(reinterpret_cast<double2*>(A.x + gn), xx);
            }
          }
          if (sip) ws[F::CFN + lane] = cfn_reg;   // face coefficients of column j
          __syncwarp();
        }
        {   // register prefetches for the next step: p, x of column j + 2, face coefficients of column
            // j + 1.  Unconditional (clamped columns): a load inside a branch makes the compiler wait
            // for it at the join, which serialised the whole step on these loads
          const int j2 = j + 2 < x0 ? x0 : j + 2 < x1 ? j + 2 : x1 - 1;
          const unsigned g2 = oC + (unsigned)j2 * TW;
          if constexpr (MODE == 0) {
            pp = __ldcs(reinterpret_cast<const double2*>(A.Pv + g2));                      // (p = 0 in the first
            xx = __ldcs(reinterpret_cast<const double2*>((x_from_rhs ? A.rhs : A.x) + g2));   // iteration: below)
            if (x_from_rhs) pp = make_double2(0.0, 0.0);
          }
          cfn_reg = cfn_load(j + 1 < x0 ? x0 : j + 1 < x1 ? j + 1 : x1 - 1);
        }
        if (own) {   // u' of the rows above / below the band at column j + 1, by a warp that rotates with j
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (warp == ((j + 4 * h) & (NW - 1))) {
              const double* raw = sm + F::HRAW + (h * 2 + (hc & 1u)) * 256;
              mbar2_wait(mb_halo + 16u * h + 8u * (hc & 1u), (hc >> 1) & 1u);
              double* rt = RT + (tN * (NW + 2) + NW + h) * 64;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int v = q ? hr1 : hr0;   // node lane + 32 q of the tile, in raw order
                if constexpr (MODE == 1) {
                  rt[q ? tr1 : tr0] = raw[v];
                } else if constexpr (MODE == 2) {
                  rt[q ? tr1 : tr0] = raw[v] * raw[192 + v];
                } else {
                  const double s = first ? 0.0 : raw[64 + v];
                  const double sn = fma(beta, s, raw[128 + v]);
                  const double rn = fma(-alpha, sn, raw[v]);
                  rt[q ? tr1 : tr0] = rn * raw[192 + v];
                }
              }
              __syncwarp();
              if (j + 3 < x1) issue_halo(h, j + 2, hc + 2);
            }
          }
          ++hc;
        }
        // column barrier.  Wait: every warp has arrived for step j - 1, i.e. written column j (and is
        // past the matvec of column j - 2, whose RT slot the NEXT step overwrites).  Then arrive for
        // this step (column j + 1 written).  Waiting before arriving keeps the phase parity unambiguous.
        if (ac > 0) mbar2_wait(mb_col, (ac - 1) & 1u);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb_col) : "memory");
        ++ac;
        if (sip && valid) {
          const double* Ue = ws + F::RING + sJ * 64;
          const double* rtj = RT + st * (NW + 2) * 64;
          double bx0, bx1, by0, by1;
          fz_sip<SUB>(op, K, L, Ue, ws + F::RING + sN * 64, ws + F::RING + sl * 64,
                 rtj + (warp + 1 < nrows ? warp + 1 : NW) * 64, rtj + (warp > 0 ? warp - 1 : NW + 1) * 64,
                 ws + F::RAW + (oc & 1u) * 320 + 256, ws + F::CFN, ws + F::QX, ws + F::QY, ws + F::DOT, ws + F::FCON, bx0, bx1, by0, by1);
          const double2 v = *reinterpret_cast<const double2*>(Ue + oP);
          const double w0 = fma(A.a, fma(K.hwy, bx0, K.hwx[0] * by0), K.hh[0] * v.x);
          const double w1 = fma(A.a, fma(K.hwy, bx1, K.hwx[1] * by1), K.hh[1] * v.y);
          if constexpr (MODE == 1) {   // r0 = b - A x0, b = M rhs (v = x0 = rhs at this node pair)
            const double b0 = K.hh[0] * v.x, b1 = K.hh[1] * v.y;
            *reinterpret_cast<double2*>(A.R + (oC + (unsigned)j * TW)) = make_double2(b0 - w0, b1 - w1);
            bb = fma(b0, b0, bb);
            nz += b0 != 0.0 ? 1.0 : 0.0;
            bb = fma(b1, b1, bb);
            nz += b1 != 0.0 ? 1.0 : 0.0;
          } else {
            *reinterpret_cast<double2*>((MODE == 2 ? A.W : Wn) + (oC + (unsigned)j * TW)) = make_double2(w0, w1);
            wu = fma(w0, v.x, wu);
            wu = fma(w1, v.y, wu);
          }
          __syncwarp();   // scratch is rewritten by the next step
        }
        if (valid) {   // this step's stage (its cf was read by the matvec) is free: refill it for step j + 2
          if (j + 2 < x1) issue_own(j + 2, oc + 2);
          ++oc;
        }
        sl = sJ;
        st = tN;
      };
      using T_ = std::true_type;
      using F_ = std::false_type;
      step(x0 - 2, F_{}, F_{});
      step(x0 - 1, T_{}, F_{});
#pragma unroll 1
      for (int j = x0; j < x1 - 1; ++j) step(j, T_{}, T_{});
      step(x1 - 1, F_{}, T_{});
    }
    if (stamp) tm[3] = gtimer();
    if constexpr (MODE == 1) {
      blk_part3(bb, nz, 0.0, red, slot2);
      return;
    } else if constexpr (MODE == 2) {
      blk_part3(ru, wu, rr, red, slot3);
      return;
    }
    if (A.sc != nullptr) {   // block partials in the split solve's slots: part (r,u), (r,r); part2 (w,u)
      blk_part3(ru, rr, 0.0, red, A.part);
      blk_part3(wu, 0.0, 0.0, red, A.part2);
      return;
    }
    double* slot = (k & 1) ? slot1 : slot0;
    {   // per-block partials -> slot[blockIdx]
      double v0 = ru, v1 = wu, v2 = rr;
      for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      }
      __syncthreads();
      if (lane == 0) { red[warp * 4] = v0; red[warp * 4 + 1] = v1; red[warp * 4 + 2] = v2; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
        for (int ww = 0; ww < NW; ++ww) { t0 += red[ww * 4]; t1 += red[ww * 4 + 1]; t2 += red[ww * 4 + 2]; }
        slot[blockIdx.x * 4] = t0; slot[blockIdx.x * 4 + 1] = t1; slot[blockIdx.x * 4 + 2] = t2;
      }
    }
    if (stamp) tm[4] = gtimer();
    grid.sync();
    if (stamp) tm[5] = gtimer();
    double tot[3];
    {   // every block sums all slots in the same fixed order
      double v0 = 0.0, v1 = 0.0, v2 = 0.0;
      for (int b = threadIdx.x; b < G; b += blockDim.x) { v0 += slot[b * 4]; v1 += slot[b * 4 + 1]; v2 += slot[b * 4 + 2]; }
      for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      }
      __syncthreads();
      if (lane == 0) { red[warp * 4] = v0; red[warp * 4 + 1] = v1; red[warp * 4 + 2] = v2; }
      __syncthreads();
      tot[0] = tot[1] = tot[2] = 0.0;
      for (int ww = 0; ww < NW; ++ww) { tot[0] += red[ww * 4]; tot[1] += red[ww * 4 + 1]; tot[2] += red[ww * 4 + 2]; }
    }
    if (stamp) tm[6] = gtimer();
    const double gn_ = tot[0];
    const double be = gn_ * rgam;
    const double al = gn_ / (tot[1] - be * (gn_ * ralpha));
    rho = tot[2];
    alpha = al;
    beta = be;
    rgam = 1.0 / gn_;
    ralpha = 1.0 / al;
    ++k;
  }
  if (own_setup && k == 0) {   // converged before the first iteration: x = x0 = rhs was never written
    const long long nthr = (long long)G * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < op.n; t += nthr) A.x[t] = A.rhs[t];
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

// ------------------------------------------------ partitioned (split) 2-D PCG
// k2_cg's Chronopoulos-Gear iteration for one element-row partition with ghost
// rows, one kernel per phase, so that the face halo of u and the allreduce of
// the three dot products (NCCL across ranks, part2d.cu) sit between launches:
//   per iteration  update (phase A) -> halo(u) -> matvec (phase B) -> reduce
//                  -> allreduce -> scalars
// Per-node arithmetic is k2_cg's; the reductions are fixed-order per block,
// per partition and then over partitions / ranks, and every rank derives
// alpha, beta from the same allreduced sums (CgPScal), so the ranks stay in
// lock step.  Kernels launched after convergence return immediately.
// Workspace per partition (doubles): R W U P S (n each) | DINV Cf (nn each) |
// partA partB (4 G each).
__device__ __forceinline__ long long own0(const Op2DDev& op) { return (long long)op.row0 * op.nex * op.p1 * op.p1; }
__device__ __forceinline__ long long nown(const Op2DDev& op) { return (long long)op.ney * op.nex * op.p1 * op.p1; }

// Cf at every storage node (the ghost rows' coefficient source was exchanged
// first), x0 = rhs, p = s = 0
template <int P1>
__global__ void k2p_init(Cg2Args A) {
  const Op2DDev& op = A.op;
  constexpr int NN = P1 * P1;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < op.n; t += nt) {
    if (t < op.nn) {
      const long long es = t / NN;
      const int nd = (int)(t - es * NN);
      A.Cf[t] = coef2d(op, A.coef, (int)(es / op.nex), (int)(es % op.nex), nd / P1, nd % P1);
    }
    A.x[t] = A.rhs[t];
    A.Pv[t] = 0.0;
    A.S[t] = 0.0;
  }
}

// closed-form Jacobi diagonal of M + a B2 at the owned nodes (k2_cg setup 1)
template <int P1>
__global__ void k2p_dinv(Cg2Args A) {
  const Op2DDev& op = A.op;
  using T = CT<P1>;
  constexpr int NN = P1 * P1, P = P1 - 1;
  const long long nt = (long long)gridDim.x * blockDim.x, no = nown(op);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < no; t += nt) {
    const long long eo = t / NN;
    const int nd = (int)(t - eo * NN), j = nd / P1, i = nd - j * P1;
    const int oy = (int)(eo / op.nex), ex = (int)(eo - (long long)oy * op.nex), ey = oy + op.row0;
    const int exr = ex + 1 == op.nex ? 0 : ex + 1, exl = ex == 0 ? op.nex - 1 : ex - 1;
    const int eyt = ynb(op, ey, 1), eyb = ynb(op, ey, -1);
    const long long es = (long long)ey * op.nex + ex;
    const double* CS = A.Cf + es * NN;
    double dx_ = 0.0, dy_ = 0.0;
    // lane-varying table rows from the global operator table (divergent constant-bank reads serialise)
    const double* d2w = op.tab + TabOff::D2W(P1);
#pragma unroll
    for (int q = 0; q < P1; ++q) {
      dx_ = fma(__ldg(d2w + i * P1 + q), CS[j * P1 + q], dx_);
      dy_ = fma(__ldg(d2w + j * P1 + q), CS[q * P1 + i], dy_);
    }
    const double DPP = c_tab2[T::D + P * P1 + P], D00 = c_tab2[T::D];
    dx_ *= op.sx;
    dy_ *= op.sy;
    if (i == P) {
      const double fr = A.Cf[((long long)ey * op.nex + exr) * NN + j * P1];
      dx_ += op.mux * (0.5 * (CS[j * P1 + P] + fr)) - op.sx * CS[j * P1 + P] * DPP;
    }
    if (i == 0) {
      const double fl = A.Cf[((long long)ey * op.nex + exl) * NN + j * P1 + P];
      dx_ += op.mux * (0.5 * (fl + CS[j * P1])) + op.sx * CS[j * P1] * D00;
    }
    if (j == P) {
      const double ft = A.Cf[((long long)eyt * op.nex + ex) * NN + i];
      dy_ += op.muy * (0.5 * (CS[P * P1 + i] + ft)) - op.sy * CS[P * P1 + i] * DPP;
    }
    if (j == 0) {
      const double fb = A.Cf[((long long)eyb * op.nex + ex) * NN + P * P1 + i];
      dy_ += op.muy * (0.5 * (fb + CS[i])) + op.sy * CS[i] * D00;
    }
    const double hwx = 0.5 * op.dx * __ldg(op.tab + TabOff::w(P1) + i), hwy = 0.5 * op.dy * __ldg(op.tab + TabOff::w(P1) + j);
    A.DINV[es * NN + nd] = 1.0 / (hwx * hwy + A.a * (hwy * dx_ + hwx * dy_));
  }
}

// r0 = b - A x0 (b = M rhs); partials (b,b), #nonzero -> part2
template <int P1, int NC>
__global__ void __launch_bounds__(256, 2) k2p_resid(Cg2Args A) {
  extern __shared__ double sm[];
  using L = CgSm<P1, NC>;
  using T = CT<P1>;
  constexpr int NN = P1 * P1, EB = Blk<P1>::EB;
  const Op2DDev& op = A.op;
  double bb = 0.0, nz = 0.0;
  auto epi = [&](long long g, double ax, double) {
    const int nd = (int)(g % NN);
    const double mi = (0.5 * op.dx * c_tab2[T::W + nd % P1]) * (0.5 * op.dy * c_tab2[T::W + nd / P1]);
    const double b = mi * A.rhs[g];
    A.R[g] = b - ax;
    bb = fma(b, b, bb);
    nz += b != 0.0 ? 1.0 : 0.0;
  };
  if constexpr (P1 == 8) {
    wpe_phase<NC>(op, sm, A.x, A.Cf, A.a, [&](long long g, double w0, double w1, double v0, double v1) {
      epi(g, w0, v0);
      epi(g + 1, w1, v1);
    });
  } else if constexpr (P1 == 4) {
    wph_phase<NC>(op, A.x, A.Cf, A.a, epi);
  } else {
    const int tpr = (op.nex + EB - 1) / EB, ntiles = tpr * op.ney;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) cg_tile<P1, NC>(op, sm, tile, tpr, A.x, nullptr, A.Cf, A.a, epi);
  }
  blk_part3(bb, nz, 0.0, sm + L::RED, A.part2);
}

// u0 = r0 dinv; partials (r,u), (r,r) -> part.  b == 0: x = 0 (dgsem.py:510-511)
template <int NC>
__global__ void __launch_bounds__(256) k2p_u0(Cg2Args A) {
  __shared__ double red[32 * 4];
  const Op2DDev& op = A.op;
  const long long nn = op.nn, o0 = own0(op), o1 = o0 + nown(op);
  const long long nt = (long long)gridDim.x * blockDim.x, g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (A.sc->zero) {
    for (long long f = o0 + g0; f < o1; f += nt)
#pragma unroll
      for (int c = 0; c < NC; ++c) A.x[c * nn + f] = 0.0;
    return;
  }
  double ru = 0.0, rr = 0.0;
  for (long long f = o0 + g0; f < o1; f += nt) {
    const double di = A.DINV[f];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double r = A.R[c * nn + f], u = r * di;
      A.U[c * nn + f] = u;
      ru = fma(r, u, ru);
      rr = fma(r, r, rr);
    }
  }
  blk_part3(ru, rr, 0.0, red, A.part);
}

// phase A': s = w + beta s, r -= alpha s, u = r dinv into A.U (p, x in the matvec)
template <int NC>
__global__ void __launch_bounds__(256) k2p_update(Cg2Args A) {
  __shared__ double red[32 * 4];
  if (A.sc->done) return;
  const double alpha = A.sc->alpha, beta = A.sc->beta;
  const Op2DDev& op = A.op;
  const long long nn = op.nn, o0 = own0(op), o1 = o0 + nown(op);
  const long long nt = (long long)gridDim.x * blockDim.x, g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool vec = ((nn | o0 | o1) & 1) == 0 && (A.defer || (reinterpret_cast<uintptr_t>(A.x) & 15) == 0);
  double ru = 0.0, rr = 0.0;
  if (vec) {
    const long long nh = nn >> 1;
    for (long long h = (o0 >> 1) + g0; h < (o1 >> 1); h += nt) {
      if (A.defer) cg_update2s<NC>(A, A.U, h, nh, alpha, beta, ru, rr, false);
      else cg_update2<NC>(A, A.U, h, nh, alpha, beta, ru, rr, false);
    }
  } else {
    for (long long f = o0 + g0; f < o1; f += nt) {
      if (A.defer) cg_update1s<NC>(A, A.U, f, nn, alpha, beta, ru, rr, false);
      else cg_update1<NC>(A, A.U, f, nn, alpha, beta, ru, rr, false);
    }
  }
  blk_part3(ru, rr, 0.0, red, A.part);
}

// phase B: w = A u; partial (w,u) -> part2; with A.px the deferred p / x
// update of this iteration from the previous u (A.U2)
template <int P1, int NC>
__global__ void __launch_bounds__(256, 2) k2p_matvec(Cg2Args A) {
  extern __shared__ double sm[];
  using L = CgSm<P1, NC>;
  constexpr int EB = Blk<P1>::EB;
  if (A.sc->done) return;
  const Op2DDev& op = A.op;
  const double alpha = A.sc->alpha, beta = A.sc->beta;
  const double* Up = A.px && A.defer ? A.U2 : nullptr;
  double wu = 0.0;
  if constexpr (P1 == 8) {
    wpe_phase<NC>(op, sm, A.U, A.Cf, A.a, [&](long long g, double w0, double w1, double v0, double v1) {
      *reinterpret_cast<double2*>(A.W + g) = make_double2(w0, w1);
      wu = fma(w0, v0, wu);
      wu = fma(w1, v1, wu);
    }, nullptr, PxArgs{Up, A.Pv, A.x, alpha, beta});
  } else {
    auto epi = [&](long long g, double wv, double u) {
      A.W[g] = wv;
      wu = fma(wv, u, wu);
      if (Up) cg_px1(A, Up, g, alpha, beta);
    };
    if constexpr (P1 == 4) {
      wph_phase<NC>(op, A.U, A.Cf, A.a, epi);
    } else {
      const int tpr = (op.nex + EB - 1) / EB, ntiles = tpr * op.ney;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) cg_tile<P1, NC>(op, sm, tile, tpr, A.U, nullptr, A.Cf, A.a, epi);
    }
  }
  blk_part3(wu, 0.0, 0.0, sm + L::RED, A.part2);
}

// fixed-order sum of the block partials of every local partition, then of the
// partition totals in partition order.  mode 0: (b,b), #nonzero; mode 1:
// (r,u), (w,u), (r,r).  One block.
struct RedPArgs {
  int nparts, G, mode;
  const double* pa[MAXPART];
  const double* pb[MAXPART];
  double* out;
};
__global__ void __launch_bounds__(256) k2p_reduce(RedPArgs R) {
  __shared__ double red[32 * 4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double tot[3] = {0.0, 0.0, 0.0};
  for (int p = 0; p < R.nparts; ++p) {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int b = threadIdx.x; b < R.G; b += blockDim.x) {
      if (R.mode == 0) {
        v0 += R.pb[p][b * 4];
        v1 += R.pb[p][b * 4 + 1];
      } else if (R.mode == 2) {   // one slot array holding (r,u), (w,u), (r,r): the fused setup pass (MODE 2)
        v0 += R.pa[p][b * 4];
        v1 += R.pa[p][b * 4 + 1];
        v2 += R.pa[p][b * 4 + 2];
      } else {
        v0 += R.pa[p][b * 4];
        v1 += R.pb[p][b * 4];
        v2 += R.pa[p][b * 4 + 1];
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
      v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    __syncthreads();
    if (lane == 0) { red[wid * 4] = v0; red[wid * 4 + 1] = v1; red[wid * 4 + 2] = v2; }
    __syncthreads();
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int ww = 0; ww < nw; ++ww) { t0 += red[ww * 4]; t1 += red[ww * 4 + 1]; t2 += red[ww * 4 + 2]; }
    tot[0] += t0;
    tot[1] += t1;
    tot[2] += t2;
  }
  if (threadIdx.x == 0) { R.out[0] = tot[0]; R.out[1] = tot[1]; R.out[2] = tot[2]; }
}

// solve scalars from the allreduced sums (k2_cg's recurrences and stopping
// rule); mode 0 after r0, 1 after w0, 2 after every iteration, 3 closes a captured batch.  One thread.
struct ScalPArgs {
  int mode, maxit;
  double rtol2;
  const double* tot;
  CgPScal* sc;
  int* status;
  int* log_it;
  double* log_margin;
  int log_cap;
};
__global__ void k2p_scalar(ScalPArgs S) {
  CgPScal& s = *S.sc;
  const double* t = S.tot;
  auto log = [&](int it, double margin) {
    const int idx = atomicAdd(&S.status[2], 1);
    if (idx < S.log_cap) { S.log_it[idx] = it; S.log_margin[idx] = margin; }
  };
  if (S.mode == 0) {
    s.thr = S.rtol2 * t[0];
    s.zero = t[1] == 0.0 ? 1 : 0;
    s.done = s.zero;
    s.ok = 1;
    s.k = 0;
    s.rho = 0.0;
    s.alpha = s.beta = 0.0;
    if (s.zero) log(0, 0.0);
    return;
  }
  if (S.mode == 3) {   // end of a captured fixed-length iteration batch: not converged = failure
    if (!s.done) {
      s.done = 1;
      s.ok = 0;
      log(-1, s.thr > 0.0 ? sqrt(s.rho / s.thr) : 0.0);
      atomicAdd(&S.status[1], 1);
    }
    return;
  }
  if (s.done) return;
  if (S.mode == 1) {
    s.rho = t[2];
    s.alpha = t[0] / t[1];
    s.beta = 0.0;
    s.rgam = 1.0 / t[0];
    s.ralpha = 1.0 / s.alpha;
  } else {
    const double gn = t[0];
    const double be = gn * s.rgam;
    const double al = gn / (t[1] - be * (gn * s.ralpha));
    s.rho = t[2];
    s.alpha = al;
    s.beta = be;
    s.rgam = 1.0 / gn;
    s.ralpha = 1.0 / al;
    ++s.k;
  }
  if (!(s.rho > s.thr)) {
    s.done = 1;
    log(s.k, s.thr > 0.0 ? sqrt(s.rho / s.thr) : 0.0);
  } else if (s.k >= S.maxit) {
    s.done = 1;
    s.ok = 0;
    log(-1, s.thr > 0.0 ? sqrt(s.rho / s.thr) : 0.0);
    atomicAdd(&S.status[1], 1);
  }
}

// in-process face halo between the local partitions of one operator: ghost
// row 0 of partition r <- last owned row of r-1, ghost row ney+1 <- first owned
// row of r+1 (periodic in y), for nc fields and mcount node vectors
struct HaloPArgs {
  int nparts, nc, nex, nnod, mcount;
  long long mstride;             // vector stride, or (mstride < 0) n of each partition: its own state size
  double* base[MAXPART];
  int ney[MAXPART];
  long long nn[MAXPART];
};
__global__ void k2p_halo(HaloPArgs H) {
  const long long row = (long long)H.nex * H.nnod;
  const int y = blockIdx.y, side = y & 1, rc = y >> 1, c = rc % H.nc, r = rc / H.nc;
  const int src = side == 0 ? (r + 1) % H.nparts : (r + H.nparts - 1) % H.nparts;
  const long long so = side == 0 ? row : (long long)H.ney[src] * row;        // first / last owned row
  const long long dof = side == 0 ? (long long)(H.ney[r] + 1) * row : 0;    // top / bottom ghost row
  const long long ms = H.mstride < 0 ? H.nn[src] * H.nc : H.mstride, md = H.mstride < 0 ? H.nn[r] * H.nc : H.mstride;
  const double* s = H.base[src] + blockIdx.z * ms + c * H.nn[src] + so;
  double* d = H.base[r] + blockIdx.z * md + c * H.nn[r] + dof;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < row; t += (long long)gridDim.x * blockDim.x)
    d[t] = s[t];
}

// NCCL halo of one partition, packed: the boundary rows of all (vector, field) pairs go through ONE
// contiguous buffer per side (2 sends + 2 receives per exchange instead of 4 per pair -- 48 NCCL calls
// per fused CG iteration before, the host cost that starved the GPU on the short coarse iterations).
// dir 0: buf[side][m][c][row] <- first (side 0) / last (side 1) owned row; dir 1: top ghost row
// (ney + 1) <- buf[0], bottom ghost row (0) <- buf[1].
struct HaloPackArgs {
  int nc, nex, nnod, mcount, ney, dir;
  long long mstride, nn;
  double* vec;
  double* buf;
};
__global__ void k2p_halo_pack(HaloPackArgs H) {
  const long long row = (long long)H.nex * H.nnod;
  const int y = blockIdx.y, side = y & 1, c = y >> 1, m = blockIdx.z;
  double* b = H.buf + ((long long)(side * H.mcount + m) * H.nc + c) * row;
  double* v = H.vec + m * H.mstride + c * H.nn;
  if (H.dir == 0) {
    const double* s = v + (side == 0 ? row : (long long)H.ney * row);
    for (long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; t < row; t += (long long)gridDim.x * blockDim.x * 2)
      *reinterpret_cast<double2*>(b + t) = *reinterpret_cast<const double2*>(s + t);
  } else {
    double* d = v + (side == 0 ? (long long)(H.ney + 1) * row : 0);
    for (long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; t < row; t += (long long)gridDim.x * blockDim.x * 2)
      *reinterpret_cast<double2*>(d + t) = *reinterpret_cast<const double2*>(b + t);
  }
}

// constant-bank copy of the reference-element matrices for one P1 (idempotent:
// they depend on P1 only); called at operator creation, outside any capture
int set_cg2_tables(Ctx* c, int p1, const double* tab) {
  if (p1 < 2 || p1 > 9) return c->fail(SISDC_ERR_UNSUPPORTED, "2-D degree outside 1..8");
  std::vector<double> h(3 * p1 * p1 + p1);
  for (int t = 0; t < p1 * p1; ++t) {
    h[t] = tab[TabOff::D(p1) + t];
    h[p1 * p1 + t] = tab[TabOff::DTW(p1) + t];
    h[2 * p1 * p1 + t] = tab[TabOff::D2W(p1) + t];
  }
  for (int t = 0; t < p1; ++t) h[3 * p1 * p1 + t] = tab[TabOff::w(p1) + t];
  cudaError_t e = cudaMemcpyToSymbol(c_tab2, h.data(), h.size() * sizeof(double), ctab_off(p1) * sizeof(double));
  if (e != cudaSuccess) return c->cuda(e, "2-D constant tables");
  return SISDC_OK;
}

// ------------------------------------------------------------- launchers
template <int P1>
static size_t smem2() { return sizeof(double) * Sm2<P1>::SIZE; }
template <int P1, int NC>
static size_t smem_cg() { return sizeof(double) * CgSm<P1, NC>::SIZE; }
template <int P1, int NC>
static cudaError_t launch_cg_coop(void** args, int nblocks, cudaStream_t st) {
  cudaFuncSetAttribute(k2_cg<P1, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cg<P1, NC>());
  return cudaLaunchCooperativeKernel((void*)k2_cg<P1, NC>, dim3(nblocks), dim3(Blk<P1>::NT), args,
                                     smem_cg<P1, NC>(), st);
}
template <int P1, int NC>
static cudaError_t cg_occupancy(int* per_sm) {
  cudaFuncSetAttribute(k2_cg<P1, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cg<P1, NC>());
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k2_cg<P1, NC>, Blk<P1>::NT, smem_cg<P1, NC>());
}

// fused solve: resident blocks x SMs (the partial slots are sized for cg_blocks), capped by the
// (band, strip, field) units; the two setup passes (MODE 1, 2) and the iterations (MODE 0) use the
// same grid, so that the slot sums cover exactly the blocks that wrote them
template <int NC, int SUB>
static cudaError_t cgf_grid(int device, const Op2DDev& op, int max_blocks, int* nb_out) {
  using F = Fz<NC, SUB>;
  constexpr int smem = (int)(sizeof(double) * F::SIZE);
  static int resident = 0;
  if (resident == 0) {
    int per_sm = 0, p1 = 0, p2 = 0, sms = 0;
    cudaError_t e = cudaFuncSetAttribute(k2_cgf<NC, SUB, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k2_cgf<NC, SUB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k2_cgf<NC, SUB, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_cgf<NC, SUB, 0>, F::NW * 32, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, k2_cgf<NC, SUB, 1>, F::NW * 32, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, k2_cgf<NC, SUB, 2>, F::NW * 32, smem);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    if (per_sm < 1 || p1 < 1 || p2 < 1) return cudaErrorLaunchOutOfResources;
    resident = per_sm * sms;   // only MODE 0 needs co-residency (grid barrier)
  }
  long long nb = (long long)((op.ney / SUB + F::NW - 1) / F::NW) * ((op.nex / SUB + F::SL - 1) / F::SL) * NC;   // units
  if (nb > resident) nb = resident;
  if (nb > max_blocks) nb = max_blocks;
  if (nb < 1) nb = 1;
  *nb_out = (int)nb;
  return cudaSuccess;
}
template <int NC, int SUB>
static cudaError_t launch_cgf(int device, Cg2Args& A, void** args, const Op2DDev& op, int max_blocks, bool own_setup,
                              cudaStream_t st) {
  using F = Fz<NC, SUB>;
  constexpr int smem = (int)(sizeof(double) * F::SIZE);
  int nb = 0;
  cudaError_t e = cgf_grid<NC, SUB>(device, op, max_blocks, &nb);
  if (e != cudaSuccess) return e;
  if (own_setup) {
    k2_cgf<NC, SUB, 1><<<nb, F::NW * 32, smem, st>>>(A);
    k2_cgf<NC, SUB, 2><<<nb, F::NW * 32, smem, st>>>(A);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaLaunchCooperativeKernel((void*)k2_cgf<NC, SUB, 0>, dim3((unsigned)nb), dim3(F::NW * 32), args, smem, st);
}

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
  if (op.problem == SISDC_NS2D && k.kind == SISDC_COEF_PHYS && op.nu_art == nullptr)   // the physical term is the NS viscous operator
    return launch2_visc(c, op, u, out, 0, 1, 0);
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_sip<P1>);
    k2_sip<P1><<<grid2<P1>(op), Blk<P1>::NT, smem2<P1>(), c->stream>>>(op, k, u, out);
  });
  if (int rc = c->after_launch("k2_sip")) return rc;
  if (op.problem == SISDC_NS2D && k.kind == SISDC_COEF_PHYS)   // with AV: nu_art Laplacian (above) + viscous operator
    return launch2_visc(c, op, u, out, 0, 1, 1);
  return SISDC_OK;
}

// Persson-Peraire modal sensor on a tensor-product element (the 2-D generalisation of
// dgsem.py:537-559, oracle/dg2d.py persson_viscosity): Legendre modes m_kl = sum Vinv[k][j] Vinv[l][i]
// u[j][i] of field 0, energies m_kl^2 (2 / (2k+1)) (2 / (2l+1)), sensor = log10(energy of the modes with
// max(k, l) = P / total), the reference's ramp around s0 = -4 log10 P, and eps0 = c_s h lam_max / P with
// h = max(dx, dy) and the element's largest signal speed.  On y-invariant data only the l = 0 modes
// are non-zero and the sensor is the reference's 1-D value.  One warp per element; fixed-order sums.
template <int P1>
__global__ void __launch_bounds__(128) k2_persson(Op2DDev op, const double* __restrict__ u, double kappa, double cs,
                                                  double* __restrict__ nu_art) {
  constexpr int NN = P1 * P1, P = P1 - 1;
  __shared__ double sU[4][NN], sT[4][NN], sV[NN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < NN; t += blockDim.x) sV[t] = op.tab[TabOff::Vinv(P1) + t];
  __syncthreads();
  const int ne = op.nex * op.ney;
  const int e = blockIdx.x * 4 + warp;
  if (e >= ne) return;
  const int oy = e / op.nex, ex = e - oy * op.nex, ey = oy + op.row0;
  double lam = 0.0;
  for (int t = lane; t < NN; t += 32) {
    double s[NC_MAX];
#pragma unroll
    for (int c = 0; c < NC_MAX; ++c) s[c] = c < op.nc ? u[nidx(op, c, ey, ex, t / P1, t % P1)] : 1.0;
    sU[warp][t] = s[0];
    lam = fmax(lam, lam_max2d(op, s));
  }
  for (int o = 16; o > 0; o >>= 1) lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, o));
  __syncwarp();
  for (int t = lane; t < NN; t += 32) {   // T[j][l] = sum_i Vinv[l][i] u[j][i]
    const int j = t / P1, l = t % P1;
    double a = 0.0;
    for (int i = 0; i < P1; ++i) a = fma(sV[l * P1 + i], sU[warp][j * P1 + i], a);
    sT[warp][t] = a;
  }
  __syncwarp();
  for (int t = lane; t < NN; t += 32) {   // m[k][l] = sum_j Vinv[k][j] T[j][l] -> energy
    const int k = t / P1, l = t % P1;
    double a = 0.0;
    for (int j = 0; j < P1; ++j) a = fma(sV[k * P1 + j], sT[warp][j * P1 + l], a);
    sU[warp][t] = a * a * ((2.0 / (2.0 * k + 1.0)) * (2.0 / (2.0 * l + 1.0)));
  }
  __syncwarp();
  if (lane == 0) {
    double tot = 0.0, top = 0.0;
    for (int t = 0; t < NN; ++t) {
      const double en = sU[warp][t];
      tot += en;
      if (t / P1 == P || t % P1 == P) top += en;
    }
    const double s = tot > 0.0 ? log10(fmax(top, 1e-300) / tot) : -INFINITY;
    const double s0 = -4.0 * log10((double)P);
    const double eps0 = cs * fmax(op.dx, op.dy) * lam / P;
    const double ramp = s < s0 - kappa ? 0.0 : (s > s0 + kappa ? 1.0 : 0.5 * (1.0 + sin(0.5 * M_PI * (s - s0) / kappa)));
    nu_art[(long long)ey * op.nex + ex] = eps0 * ramp;
  }
}

int launch2_persson(Ctx* c, const Op2DDev& op, const double* u, double kappa, double cs, double* nu_art) {
  const int ne = op.nex * op.ney;
  SISDC_P1_SWITCH(op.p1, { k2_persson<P1><<<(ne + 3) / 4, 128, 0, c->stream>>>(op, u, kappa, cs, nu_art); });
  return c->after_launch("k2_persson");
}
// P = 7 viscous operator on the tensor cores (called by launch2_visc, visc2d.cu); returns
// SISDC_ERR_UNSUPPORTED-free: the caller checks the shape (p1 == 8, four fields, 16-byte alignment)
int launch2_visc8(Ctx* c, const Op2DDev& op, const double* u, double* f, int m_first, int m_count, int accumulate) {
  const size_t smem = sizeof(double) * VS_WARPS * Vs8::WARP;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(k2_visc8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_visc8, VS_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int ne = op.nex * op.ney;
  // a few elements per warp (the pipeline needs a next element to prefetch), grid a multiple of the
  // resident block count
  long long gx = (long long)per_sm * sms * 2 / m_count;
  if (gx < per_sm * sms / 2) gx = per_sm * sms / 2;
  const long long need = (ne + VS_WARPS - 1) / VS_WARPS;
  if (gx > need) gx = need;
  if (gx < 1) gx = 1;
  k2_visc8<<<dim3((unsigned)gx, m_count), VS_WARPS * 32, smem, c->stream>>>(op, u, f, m_first, accumulate, c->d_status);
  return c->after_launch("k2_visc8");
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
  const bool al16 = ((reinterpret_cast<uintptr_t>(u0) | reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(f) |
                      reinterpret_cast<uintptr_t>(h1) | reinterpret_cast<uintptr_t>(h2) |
                      reinterpret_cast<uintptr_t>(conv_prev)) & 15) == 0;
  if (op.p1 == 8 && op.nu_art == nullptr && op.nc == 4 && al16) {   // tensor-core warp-per-element path
    const size_t smem = sizeof(double) * EV_WARPS * Ev<4>::WARP;
    cudaFuncSetAttribute(k2_eval8<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int ne = op.nex * op.ney;
    int nb = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k2_eval8<4>, EV_WARPS * 32, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    long long gx = (long long)(nb > 0 ? nb : 1) * sms * 4 / m_count;
    if (gx < 1) gx = 1;
    const long long need = (ne + EV_WARPS - 1) / EV_WARPS;
    if (gx > need) gx = need;
    k2_eval8<4><<<dim3((unsigned)gx, m_count), EV_WARPS * 32, smem, c->stream>>>(op, a);
    if (int rc = c->after_launch("k2_eval8")) return rc;
    return launch2_visc(c, op, u, f, m_first, m_count, 1);   // NS2D: f += physical viscous term
  }
  SISDC_P1_SWITCH(op.p1, {
    set_smem<P1>(k2_node_eval<P1>);
    k2_node_eval<P1><<<grid2<P1>(op, m_count), Blk<P1>::NT, smem2<P1>(), c->stream>>>(op, a);
  });
  if (int rc = c->after_launch("k2_node_eval")) return rc;
  return launch2_visc(c, op, u, f, m_first, m_count, 1);   // NS2D: f += physical viscous term
}
int launch2_stage(Ctx* c, const Op2DDev& op, const double* base, const double* conv_in, double dt_m,
                  const double* f_old, int M, const double* w_row, double dt, const double* g,
                  const double* h, double* rhs, double* conv_out) {
  if (M > 16) return c->fail(SISDC_ERR_ARG, "too many collocation nodes");
  Stage2Args a{};
  a.base = base; a.conv_in = conv_in; a.dt_m = dt_m; a.f_old = f_old; a.M = M; a.dt = dt;
  for (int j = 0; j < M; ++j) a.w[j] = (f_old && w_row) ? w_row[j] : 0.0;
  a.g = g; a.h = h; a.rhs = rhs; a.conv_out = conv_out;
  const bool al16 = ((reinterpret_cast<uintptr_t>(base) | reinterpret_cast<uintptr_t>(conv_in) |
                      reinterpret_cast<uintptr_t>(f_old) | reinterpret_cast<uintptr_t>(g) |
                      reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(rhs) |
                      reinterpret_cast<uintptr_t>(conv_out)) & 15) == 0;
  if (op.p1 == 8 && op.nc == 4 && al16) {   // tensor-core warp-per-element path
    const size_t smem = sizeof(double) * EV_WARPS * Stg<4>::WARP;
    const int ne = op.nex * op.ney;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    auto go = [&](auto kern) {
      int nb = 0;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, EV_WARPS * 32, smem);
      long long gx = (long long)(nb > 0 ? nb : 1) * sms * 4;
      const long long need = (ne + EV_WARPS - 1) / EV_WARPS;
      if (gx > need) gx = need;
      kern<<<(unsigned)gx, EV_WARPS * 32, smem, c->stream>>>(op, a);
    };
    // the quadrature length as a compile-time count where it is one of the schedules' node counts
    const int mq = f_old ? M : 0;
    if (mq == 5) go(k2_stage8<4, 5>);
    else if (mq == 4) go(k2_stage8<4, 4>);
    else if (mq == 3) go(k2_stage8<4, 3>);
    else go(k2_stage8<4, 0>);
    return c->after_launch("k2_stage8");
  }
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
  const size_t sm = sizeof(double) * (2 * x.Mf * x.pf * x.pf + 2 * x.Mf * x.pc * x.pc + 2 * x.Mf * x.pf * x.pc);
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
  const size_t sm = sizeof(double) * (2 * x.Mf * x.pf * x.pf + 2 * x.Mf * x.pc * x.pc + 2 * x.Mf * x.pf * x.pc);
  k2x_down<<<x.nslab, 128, sm, c->stream>>>(x, 1, 1, nullptr, v, (long long)x.nslab * x.pf * x.pf,
                                            (long long)x.nslab * x.pc * x.pc, 1, fa, rr);
  return c->after_launch("k2x_fas");
}
int launch2x_interp(Ctx* c, const Xfer2Dev& x, int accumulate, const double* uc, const double* vc, double* uf) {
  const size_t sm = sizeof(double) * (x.Mc * x.pc * x.pc + x.Mf * x.pc * x.pc + x.Mf * x.pc * x.pf);
  k2x_interp<<<x.nslab, 128, sm, c->stream>>>(x, accumulate, uc, vc, uf, (long long)x.nslab * x.pf * x.pf,
                                              (long long)x.nslab * x.pc * x.pc);
  return c->after_launch("k2x_interp");
}

// CG workspace lives in the context, grown on demand (outside graph capture)
int launch2_cg(Ctx* c, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws,
               int nblocks) {
  if (op.p1 == 8 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(rhs)) & 15))
    return c->fail(SISDC_ERR_ARG, "2-D implicit solve: rhs and x must be 16-byte aligned");
  Cg2Args A{};
  A.op = op; A.coef = k; A.a = a; A.rhs = rhs; A.x = x;
  A.rtol2 = c->rtol * c->rtol; A.maxit = c->maxit;
  double* p = ws;
  A.R = p; p += op.n;
  A.W = p; p += op.n;
  A.U = p; p += op.n;
  A.Pv = p; p += op.n;
  A.S = p; p += op.n;
  A.U2 = p; p += op.n;
  A.W2 = p; p += op.n;   // fused pass only (cg2_ws_doubles)
  A.DINV = p; p += op.nn;
  A.Cf = p; p += op.nn;
  A.scal = p; p += 16;
  A.part = p;
  A.R2 = A.U2;           // fused pass: (r, s, w) double-buffered; u0 of the setup lives in the second s buffer
  A.S2 = A.U;
  A.status = c->d_status; A.log_it = c->d_log_it; A.log_margin = c->d_log_margin; A.log_cap = c->log_cap;
  A.timing = c->d_timing;
  if (c->d_timing) {
    const char* dbg = getenv("SISDC_CG_DBG");
    A.dbg = dbg ? atoi(dbg) : 0;
  }
  void* args[] = {&A};
  cudaError_t e = cudaSuccess;
  // P = 7: setup by k2_cg (mode 1), iterations by the fused single-pass kernel
  // (SISDC_CG_FUSED=0 keeps the two-phase iteration for A/B runs)
  static const bool fused_on = [] {
    const char* v = getenv("SISDC_CG_FUSED");
    return !(v && v[0] == '0');
  }();
  // P = 7 elements, or P = 3 elements in 2 x 2 tiles (even mesh; SISDC_CG_FUSED3=0 keeps the two-phase kernel)
  static const bool fused3_on = [] {
    const char* v = getenv("SISDC_CG_FUSED3");
    return !(v && v[0] == '0');
  }();
  const bool sub2 = op.p1 == 4 && fused3_on && op.nex % 2 == 0 && op.ney % 2 == 0 && op.nex >= 2 && op.ney >= 2;
  const bool fused = fused_on && (op.p1 == 8 || sub2) && op.row0 == 0 && (op.nc == 4 || op.nc == 1);
  if (fused) {
    if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(rhs)) & 15))
      return c->fail(SISDC_ERR_ARG, "2-D implicit solve: rhs and x must be 16-byte aligned");
    // coefficient and Jacobi diagonal at full occupancy (fp64 sqrt / division chains want more warps
    // than the 128-register cooperative kernel has), then k2_cg's setup 2 / 3 only (mode 2)
    const unsigned nb1 = (unsigned)((op.nn + 255) / 256);
    if (sub2) k2_coef<4><<<nb1, 256, 0, c->stream>>>(op, k, A.Cf);
    else k2_coef<8><<<nb1, 256, 0, c->stream>>>(op, k, A.Cf);
    int rc = c->after_launch("k2_coef (CG setup)");
    if (rc) return rc;
    if (sub2) k2p_dinv<4><<<nb1, 256, 0, c->stream>>>(A);
    else k2p_dinv<8><<<nb1, 256, 0, c->stream>>>(A);
    rc = c->after_launch("k2p_dinv (CG setup)");
    if (rc) return rc;
    // setup passes: the fused pipeline itself (A.mode 3; SISDC_CG_SETUP=0: k2_cg in mode 2)
    static const bool own_setup_on = [] {
      const char* v = getenv("SISDC_CG_SETUP");
      return !(v && v[0] == '0');
    }();
    A.mode = own_setup_on ? 3 : 2;
  }
  if (A.mode == 3) {
    cudaError_t e3;
    if (sub2)
      e3 = op.nc == 4 ? launch_cgf<4, 2>(c->device, A, args, op, nblocks, true, c->stream)
                      : launch_cgf<1, 2>(c->device, A, args, op, nblocks, true, c->stream);
    else
      e3 = op.nc == 4 ? launch_cgf<4, 1>(c->device, A, args, op, nblocks, true, c->stream)
                      : launch_cgf<1, 1>(c->device, A, args, op, nblocks, true, c->stream);
    if (e3 != cudaSuccess) return c->cuda(e3, "k2_cgf solve launch");
    c->launches += 2;
    return c->after_launch("k2_cgf");
  }
  SISDC_P1_SWITCH(op.p1, {
    if (op.nc == 4) e = launch_cg_coop<P1, 4>(args, nblocks, c->stream);
    else e = launch_cg_coop<P1, 1>(args, nblocks, c->stream);
  });
  if (e != cudaSuccess) return c->cuda(e, "k2_cg cooperative launch");
  if (fused) {
    int rc = c->after_launch("k2_cg (setup)");
    if (rc) return rc;
    if (sub2)
      e = op.nc == 4 ? launch_cgf<4, 2>(c->device, A, args, op, nblocks, false, c->stream)
                     : launch_cgf<1, 2>(c->device, A, args, op, nblocks, false, c->stream);
    else
      e = op.nc == 4 ? launch_cgf<4, 1>(c->device, A, args, op, nblocks, false, c->stream)
                     : launch_cgf<1, 1>(c->device, A, args, op, nblocks, false, c->stream);
    if (e != cudaSuccess) return c->cuda(e, "k2_cgf cooperative launch");
    return c->after_launch("k2_cgf");
  }
  return c->after_launch("k2_cg");
}
size_t cg2_ws_doubles(const Op2DDev& op, int nblocks) {   // part: four slot arrays of [nblocks][4]
  return 7 * (size_t)op.n + 2 * (size_t)op.nn + 16 + 16 * (size_t)nblocks;
}
// blocks for the cooperative CG: resident blocks x SMs, capped by the element tiles
int cg2_blocks(Ctx* c, const Op2DDev& op, int* nblocks) {
  int per_sm = 0, sms = 0;
  cudaError_t e = cudaSuccess;
  SISDC_P1_SWITCH(op.p1, {
    e = op.nc == 4 ? cg_occupancy<P1, 4>(&per_sm) : cg_occupancy<P1, 1>(&per_sm);
    const int ntiles = (op.nex + Blk<P1>::EB - 1) / Blk<P1>::EB * op.ney;   // strip tiles
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    long long nb = (long long)per_sm * sms;
    if (nb > ntiles) nb = ntiles;
    if (nb < 1) nb = 1;
    *nblocks = (int)nb;
  });
  if (e != cudaSuccess) return c->cuda(e, "k2_cg occupancy");
  return SISDC_OK;
}


// ------------------------------------------------ partitioned solve launchers
// P = 7 partitions iterate with the fused single pass (k2_cgf in single-pass mode):
// workspace R0 S0 W0 R1 S1 W1 P (n each; the setup's u0 lives in S1) | DINV Cf | partA partB
bool cg2p_fused(const Op2DDev& op) {
  static const bool on = [] {
    const char* v = getenv("SISDC_CG_FUSED");
    return !(v && v[0] == '0');
  }();
  return on && (op.p1 == 8 || (op.p1 == 4 && op.fused_sub2 != 0));
}
size_t cg2p_ws_doubles(const Op2DDev& op, int G) { return 7 * (size_t)op.n + 2 * (size_t)op.nn + 16 * (size_t)G; }   // partA partB | setup slots 2, 3
size_t cg2p_part_off(const Op2DDev& op) { return (cg2p_fused(op) ? 7 : 6) * (size_t)op.n + 2 * (size_t)op.nn; }
size_t cg2p_dinv_off(const Op2DDev& op) { return (cg2p_fused(op) ? 7 : 6) * (size_t)op.n; }
// the two u buffers of the split solve: which 0 -> U, 1 -> U2 (fused: the setup's u0 only, in S1)
double* cg2p_U(const Op2DDev& op, double* ws, int which) {
  if (cg2p_fused(op)) return ws + 4 * op.n;
  return ws + (which ? 5 : 2) * op.n;
}
// fused: the (r, s, w) triple of parity par, three consecutive vectors (one halo call)
double* cg2p_RSW(const Op2DDev& op, double* ws, int par) { return ws + (par ? 3 : 0) * op.n; }

static Cg2Args cg2p_args(const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws, int G,
                         const CgPScal* sc, int ucur) {
  Cg2Args A{};
  A.op = op; A.coef = k; A.a = a; A.rhs = rhs; A.x = x;
  double* p = ws;
  if (cg2p_fused(op)) {
    A.R = p; p += op.n;
    A.S = p; p += op.n;
    A.W = p; p += op.n;
    A.R2 = p; p += op.n;
    A.S2 = p; A.U = p; p += op.n;   // u0 of the setup
    A.W2 = p; p += op.n;
    A.Pv = p; p += op.n;
    A.U2 = nullptr;
  } else {
    A.R = p; p += op.n;
    A.W = p; p += op.n;
    A.U = p; p += op.n;
    A.Pv = p; p += op.n;
    A.S = p; p += op.n;
    A.U2 = p; p += op.n;
  }
  A.DINV = p; p += op.nn;
  A.Cf = p; p += op.nn;
  A.part = p; p += 4 * G;
  A.part2 = p;
  A.sc = sc;
  // ucur: 0 / 1 = which buffer holds this iteration's u (the other the previous u);
  // -1: setup (u0 into buffer 0, no p / x update)
  if (ucur == 1 && !cg2p_fused(op)) {
    double* t = A.U;
    A.U = A.U2;
    A.U2 = t;
  }
  A.px = ucur >= 0 ? 1 : 0;
  A.defer = op.p1 == 8 ? 1 : 0;
  return A;
}

template <int P1, int NC>
static cudaError_t p2_phase(int phase, const Cg2Args& A, int G, cudaStream_t st) {
  const size_t smem = smem_cg<P1, NC>();
  switch (phase) {
    // pointwise passes with fp64 sqrt / division chains: one thread per node, full occupancy
    // (no per-block partials, so the grid is free)
    case P2_INIT: k2p_init<P1><<<(unsigned)((A.op.n + 255) / 256), 256, 0, st>>>(A); break;
    case P2_DINV: k2p_dinv<P1><<<(unsigned)((A.op.nn + 255) / 256), 256, 0, st>>>(A); break;
    case P2_RESID:
      cudaFuncSetAttribute(k2p_resid<P1, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k2p_resid<P1, NC><<<G, Blk<P1>::NT, smem, st>>>(A);
      break;
    case P2_U0: k2p_u0<NC><<<G, 256, 0, st>>>(A); break;
    case P2_UPDATE: k2p_update<NC><<<G, 256, 0, st>>>(A); break;
    case P2_MATVEC:
      cudaFuncSetAttribute(k2p_matvec<P1, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k2p_matvec<P1, NC><<<G, Blk<P1>::NT, smem, st>>>(A);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int launch2p_phase(Ctx* c, int phase, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x,
                   double* ws, int G, const CgPScal* sc, int ucur) {
  const Cg2Args A = cg2p_args(op, k, a, rhs, x, ws, G, sc, ucur);
  cudaError_t e = cudaSuccess;
  SISDC_P1_SWITCH(op.p1, {
    e = op.nc == 4 ? p2_phase<P1, 4>(phase, A, G, c->stream) : p2_phase<P1, 1>(phase, A, G, c->stream);
  });
  ++c->launches;
  if (e != cudaSuccess) return c->cuda(e, "k2p phase launch");
  return SISDC_OK;
}

// one fused iteration pass on a partition (k2_cgf in single-pass mode); par: parity of the (r, s, w) read.
// bsel / slot0 / nblk: the bands of this launch (Cg2Args::bsel), its first block-partial slot and its grid
// (the interior and the edge launch of one iteration share the partition's G slots: slot0 + nblk <= G)
int launch2p_fpass(Ctx* c, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws, int G,
                   const CgPScal* sc, int par, int bsel, int slot0, int nblk) {
  Cg2Args A = cg2p_args(op, k, a, rhs, x, ws, G, sc, -1);
  A.px = par;
  A.maxit = c->maxit;
  A.bsel = bsel;
  if (nblk < 0) nblk = G;
  A.part += 4 * slot0;
  A.part2 += 4 * slot0;
  cudaError_t e = cudaSuccess;
  if (op.p1 == 4 && (op.nc == 4 || op.nc == 1)) {   // P = 3: 2 x 2-element tiles (even nex, even rows: fused_sub2)
    if (op.nc == 4) {
      using F = Fz<4, 2>;
      constexpr int smem = (int)(sizeof(double) * F::SIZE);
      cudaFuncSetAttribute(k2_cgf<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k2_cgf<4, 2><<<nblk, F::NW * 32, smem, c->stream>>>(A);
    } else {
      using F = Fz<1, 2>;
      constexpr int smem = (int)(sizeof(double) * F::SIZE);
      cudaFuncSetAttribute(k2_cgf<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k2_cgf<1, 2><<<nblk, F::NW * 32, smem, c->stream>>>(A);
    }
  } else if (op.nc == 4) {
    using F = Fz<4>;
    constexpr int smem = (int)(sizeof(double) * F::SIZE);
    cudaFuncSetAttribute(k2_cgf<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k2_cgf<4><<<nblk, F::NW * 32, smem, c->stream>>>(A);
  } else if (op.nc == 1) {
    using F = Fz<1>;
    constexpr int smem = (int)(sizeof(double) * F::SIZE);
    cudaFuncSetAttribute(k2_cgf<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k2_cgf<1><<<nblk, F::NW * 32, smem, c->stream>>>(A);
  } else {
    return c->fail(SISDC_ERR_UNSUPPORTED, "fused 2-D pass: 1 or 4 fields");
  }
  e = cudaGetLastError();
  ++c->launches;
  if (e != cudaSuccess) return c->cuda(e, "k2_cgf single-pass launch");
  return SISDC_OK;
}
// the two setup passes of a fused partition solve as single passes of the fused pipeline (k2_cgf MODE 1:
// r0 = b - A x0 -> R, partials (b,b), #nonzero -> slot 2; MODE 2: u0 = r0 dinv rebuilt on chip, w0 = A u0 -> W,
// partials (r,u), (w,u), (r,r) -> slot 3), instead of the split kernels k2p_resid / k2p_u0 / k2p_matvec
template <int NC, int SUB>
static cudaError_t fsetup_launch(int mode, const Cg2Args& A, int G, cudaStream_t st) {
  using F = Fz<NC, SUB>;
  constexpr int smem = (int)(sizeof(double) * F::SIZE);
  if (mode == 1) {
    cudaFuncSetAttribute(k2_cgf<NC, SUB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k2_cgf<NC, SUB, 1><<<G, F::NW * 32, smem, st>>>(A);
  } else {
    cudaFuncSetAttribute(k2_cgf<NC, SUB, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k2_cgf<NC, SUB, 2><<<G, F::NW * 32, smem, st>>>(A);
  }
  return cudaGetLastError();
}
int launch2p_fsetup(Ctx* c, int mode, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws,
                    int G, const CgPScal* sc) {
  Cg2Args A = cg2p_args(op, k, a, rhs, x, ws, G, sc, -1);
  A.maxit = c->maxit;
  cudaError_t e = cudaSuccess;
  if (op.p1 == 4) e = op.nc == 4 ? fsetup_launch<4, 2>(mode, A, G, c->stream) : fsetup_launch<1, 2>(mode, A, G, c->stream);
  else e = op.nc == 4 ? fsetup_launch<4, 1>(mode, A, G, c->stream) : fsetup_launch<1, 1>(mode, A, G, c->stream);
  ++c->launches;
  if (e != cudaSuccess) return c->cuda(e, "k2_cgf setup-pass launch");
  return SISDC_OK;
}
// bands of the fused pass on a partition (8 element rows each; P = 3: 8 rows of 2 x 2-element tiles)
int cg2p_bands(const Op2DDev& op) { return ((op.p1 == 4 ? op.ney / 2 : op.ney) + Fz<4>::NW - 1) / Fz<4>::NW; }

// mode 0: (b,b), #nonzero from partB (fsetup: from the fused setup pass's slot 2); mode 1: the iteration's
// partA / partB; mode 2: (r,u), (w,u), (r,r) from the fused setup pass's slot 3
int launch2p_reduce(Ctx* c, int nparts, double* const* ws, const Op2DDev* ops, int G, int mode, double* out,
                    int fsetup) {
  if (nparts < 1 || nparts > MAXPART) return c->fail(SISDC_ERR_ARG, "partition count");
  RedPArgs R{};
  R.nparts = nparts; R.G = G; R.mode = mode; R.out = out;
  for (int p = 0; p < nparts; ++p) {
    const double* base = ws[p] + cg2p_part_off(ops[p]);
    R.pa[p] = mode == 2 ? base + 12 * G : base;
    R.pb[p] = (mode == 0 && fsetup) ? base + 8 * G : base + 4 * G;
  }
  k2p_reduce<<<1, 256, 0, c->stream>>>(R);
  return c->after_launch("k2p_reduce");
}

int launch2p_scalar(Ctx* c, int mode, const double* tot, CgPScal* sc) {
  ScalPArgs S{};
  S.mode = mode; S.maxit = c->maxit; S.rtol2 = c->rtol * c->rtol; S.tot = tot; S.sc = sc;
  S.status = c->d_status; S.log_it = c->d_log_it; S.log_margin = c->d_log_margin; S.log_cap = c->log_cap;
  k2p_scalar<<<1, 1, 0, c->stream>>>(S);
  return c->after_launch("k2p_scalar");
}

int launch2p_halo(Ctx* c, int nparts, const Op2DDev* ops, double* const* base, int nc, int mcount, long long mstride) {
  if (nparts < 1 || nparts > MAXPART || mcount < 1) return c->fail(SISDC_ERR_ARG, "halo arguments");
  HaloPArgs H{};
  H.nparts = nparts; H.nc = nc; H.nex = ops[0].nex; H.nnod = ops[0].p1 * ops[0].p1; H.mcount = mcount;
  H.mstride = mstride;
  for (int p = 0; p < nparts; ++p) {
    H.base[p] = base[p];
    H.ney[p] = ops[p].ney;
    H.nn[p] = ops[p].nn;
  }
  const long long row = (long long)H.nex * H.nnod;
  const unsigned gx = (unsigned)((row + 255) / 256 < 64 ? (row + 255) / 256 : 64);
  k2p_halo<<<dim3(gx, 2 * nc * nparts, mcount), 256, 0, c->stream>>>(H);
  return c->after_launch("k2p_halo");
}

int launch2p_halo_pack(Ctx* c, const Op2DDev& op, double* vec, double* buf, int nc, int mcount, long long mstride,
                       int dir) {
  HaloPackArgs H{};
  H.nc = nc; H.nex = op.nex; H.nnod = op.p1 * op.p1; H.mcount = mcount; H.ney = op.ney; H.dir = dir;
  H.mstride = mstride; H.nn = op.nn; H.vec = vec; H.buf = buf;
  const long long row = (long long)H.nex * H.nnod;   // even (nnod = p1^2 rows of a 16-byte aligned field: checked by the caller)
  const unsigned gx = (unsigned)((row / 2 + 255) / 256 < 64 ? (row / 2 + 255) / 256 : 64);
  k2p_halo_pack<<<dim3(gx, 2 * nc, mcount), 256, 0, c->stream>>>(H);
  return c->after_launch("k2p_halo_pack");
}

// blocks of the split-solve kernels: resident blocks of the matvec x SMs,
// capped by the partition's work units
int cg2p_blocks(Ctx* c, const Op2DDev& op, int* G) {
  int per_sm = 0, sms = 0;
  cudaError_t e = cudaSuccess;
  SISDC_P1_SWITCH(op.p1, {
    const size_t smem = smem_cg<P1, 4>() > smem_cg<P1, 1>() ? smem_cg<P1, 4>() : smem_cg<P1, 1>();
    if (op.nc == 4) {
      cudaFuncSetAttribute(k2p_matvec<P1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2p_matvec<P1, 4>, Blk<P1>::NT, smem_cg<P1, 4>());
    } else {
      cudaFuncSetAttribute(k2p_matvec<P1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2p_matvec<P1, 1>, Blk<P1>::NT, smem_cg<P1, 1>());
    }
    const long long units = P1 == 8 ? ((long long)op.nex * op.ney + 7) / 8
                                    : (long long)((op.nex + Blk<P1>::EB - 1) / Blk<P1>::EB) * op.ney;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    long long nb = (long long)(per_sm > 0 ? per_sm : 1) * sms;
    if (nb > units) nb = units;
    if (nb < 1) nb = 1;
    *G = (int)nb;
  });
  if (e != cudaSuccess) return c->cuda(e, "k2p occupancy");
  return SISDC_OK;
}

}  // namespace sisdc
