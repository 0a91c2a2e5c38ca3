// Physical viscous operator of 2-D compressible Navier-Stokes (SISDC_NS2D):
// the 2-D generalisation of the reference's matrix SIP with the
// CompressibleFlow viscous coefficient (problems.py:221-237,
// dgsem.py:251-309), restated in oracle/dg2d.py (Op2D.apply_viscous).
//
// Per direction (x: faces R/L with F^x and the block G_xx; y: T/B, F^y, G_yy)
//   B  = sum_k D_ki w_k F(.., k)                      (volume, full flux incl. cross terms)
//   B(P) += Gf(right face), B(0) -= Gf(left face),
//   Gf = mu0 (G_nn(u-) [u] + G_nn(u+) [u]) / 2 - (F- + F+) / 2,   [u] = u- - u+
//   B -= s ((G_nn(u_own) [u]) / 2 D[P][.] at the right face, ... D[0][.] at the left)
// and f_visc = -(B_x / (hx w_i) + B_y / (hy w_j)).  On y-invariant data with
// v = 0 this is the reference's 1-D CompressibleFlow term (tests/test_oracle2d.py).
//
// One thread per node; a block stages EB elements and their four face
// neighbours (all four fields) in shared memory, forms every own node's
// viscous flux, the face fluxes of its element (computing the neighbour's
// flux at the shared face nodes from the staged neighbour), then the
// divergence.  Not on the CG hot path: it runs once per right-hand-side
// evaluation (node caches, FAS defects), after the convection/SI kernels.
#include "sisdc_dev2d.cuh"
#include "sisdc_host.h"

namespace sisdc {
namespace {

constexpr int NCV = 4;   // (rho, rho u, rho v, rho E)
enum { FR = 0, FL = 1, FT = 2, FB = 3 };   // right, left, top, bottom faces

template <int P1>
struct Vb {
  static constexpr int NN = P1 * P1;
  static constexpr int EB = NN >= 256 ? 1 : 256 / NN;      // elements per block
  static constexpr int NT = EB * NN;
  static constexpr int US = 5 * NCV * NN;                   // staged u per element: own, R, L, T, B
  static constexpr int U = 0;                               // [EB][5][NCV][NN]
  static constexpr int FX = U + EB * US, FY = FX + EB * NCV * NN;   // own fluxes [EB][NCV][NN]
  static constexpr int GF = FY + EB * NCV * NN;             // face fluxes [EB][4 faces][P1][NCV]
  static constexpr int LF = GF + EB * 4 * P1 * NCV;         // own lifts   [EB][4 faces][P1][NCV]
  static constexpr int SIZE = LF + EB * 4 * P1 * NCV;
};

struct Prim {
  double rho, vx, vy, Es, nu;
};
__device__ __forceinline__ Prim prim(const Op2DDev& op, const double* s) {
  const double rho = s[0];
  return Prim{rho, s[1] / rho, s[2] / rho, s[3] / rho, op.nu / rho};
}

// viscous flux at a node from the state and its gradients (oracle NS2D.visc_flux)
__device__ __forceinline__ void visc_flux(const Op2DDev& op, const double* s, const double* gx, const double* gy,
                                          double* Fx, double* Fy) {
  const Prim q = prim(op, s);
  const double k = op.gamma * q.nu / op.pr;
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
__device__ __forceinline__ void apply_gnn(const Op2DDev& op, const double* s, const double* v, int axis, double* r) {
  const Prim q = prim(op, s);
  const double k = op.gamma * q.nu / op.pr;
  const double a = v[1] - q.vx * v[0], b = v[2] - q.vy * v[0];
  const double r1 = q.nu * (axis == 0 ? (4.0 / 3.0) * a : a);
  const double r2 = q.nu * (axis == 0 ? b : (4.0 / 3.0) * b);
  r[0] = 0.0;
  r[1] = r1;
  r[2] = r2;
  r[3] = q.vx * r1 + q.vy * r2 + k * (v[3] - q.Es * v[0] - q.vx * a - q.vy * b);
}

// gradients (all fields) at node (j, i) of a staged element X = [NCV][NN]
template <int P1>
__device__ __forceinline__ void grad_at(const Op2DDev& op, const double* X, const double* D, int j, int i, double* gx,
                                        double* gy) {
  constexpr int NN = P1 * P1;
#pragma unroll
  for (int c = 0; c < NCV; ++c) {
    double ax = 0.0, ay = 0.0;
#pragma unroll
    for (int q = 0; q < P1; ++q) {
      ax = fma(D[i * P1 + q], X[c * NN + j * P1 + q], ax);
      ay = fma(D[j * P1 + q], X[c * NN + q * P1 + i], ay);
    }
    gx[c] = op.sx * ax;
    gy[c] = op.sy * ay;
  }
}

// face flux Gf between the staged elements A (minus side) and B (plus side)
// at A's node (ja, ia) and B's node (jb, ib); also the minus / plus lifts
template <int P1>
__device__ __forceinline__ void face_terms(const Op2DDev& op, const double* A, const double* B, const double* D, int ja,
                                           int ia, int jb, int ib, int axis, double* Gf, double* gm_out, double* gp_out) {
  constexpr int NN = P1 * P1;
  double sa[NCV], sb[NCV], jmp[NCV], gx[NCV], gy[NCV], Fxa[NCV], Fya[NCV], Fxb[NCV], Fyb[NCV];
#pragma unroll
  for (int c = 0; c < NCV; ++c) {
    sa[c] = A[c * NN + ja * P1 + ia];
    sb[c] = B[c * NN + jb * P1 + ib];
    jmp[c] = sa[c] - sb[c];
  }
  grad_at<P1>(op, A, D, ja, ia, gx, gy);
  visc_flux(op, sa, gx, gy, Fxa, Fya);
  grad_at<P1>(op, B, D, jb, ib, gx, gy);
  visc_flux(op, sb, gx, gy, Fxb, Fyb);
  double gm[NCV], gp[NCV];
  apply_gnn(op, sa, jmp, axis, gm);
  apply_gnn(op, sb, jmp, axis, gp);
  const double mu0 = axis == 0 ? op.mux : op.muy;
#pragma unroll
  for (int c = 0; c < NCV; ++c) {
    const double qa = axis == 0 ? Fxa[c] : Fya[c], qb = axis == 0 ? Fxb[c] : Fyb[c];
    Gf[c] = mu0 * (0.5 * (gm[c] + gp[c])) - 0.5 * (qa + qb);
    gm_out[c] = gm[c];
    gp_out[c] = gp[c];
  }
}

template <int P1>
__global__ void __launch_bounds__(Vb<P1>::NT) k2_visc(Op2DDev op, const double* __restrict__ u, double* __restrict__ f,
                                                      int m_first, int accumulate, int* status) {
  using L = Vb<P1>;
  constexpr int NN = P1 * P1, P = P1 - 1;
  extern __shared__ double sm[];
  __shared__ double sD[P1 * P1], sDTW[P1 * P1], sW[P1];
  const int m = m_first + blockIdx.y;
  const double* um = u + (size_t)m * op.ns;
  double* fm = f + (size_t)m * op.ns;
  for (int t = threadIdx.x; t < NN; t += blockDim.x) {
    sD[t] = op.tab[TabOff::D(P1) + t];
    sDTW[t] = op.tab[TabOff::DTW(P1) + t];
  }
  for (int t = threadIdx.x; t < P1; t += blockDim.x) sW[t] = op.tab[TabOff::w(P1) + t];
  const int ne = op.nex * op.ney;
  const int e0 = blockIdx.x * L::EB;
  // ---- stage own + face neighbours, all fields (coalesced element runs)
  for (int t = threadIdx.x; t < L::EB * 5 * NCV * NN; t += blockDim.x) {
    const int el = t / (5 * NCV * NN), r = t - el * (5 * NCV * NN);
    const int k = r / (NCV * NN), r2 = r - k * (NCV * NN);
    const int c = r2 / NN, nd = r2 - c * NN;
    const int eg = e0 + el;
    double v = 0.0;
    if (eg < ne) {
      const int oy = eg / op.nex, ex = eg - oy * op.nex, ey = oy + op.row0;
      int sx_ = ex, sy_ = ey;
      if (k == 1) sx_ = ex + 1 == op.nex ? 0 : ex + 1;
      if (k == 2) sx_ = ex == 0 ? op.nex - 1 : ex - 1;
      if (k == 3) sy_ = ynb(op, ey, 1);
      if (k == 4) sy_ = ynb(op, ey, -1);
      v = um[nidx(op, c, sy_, sx_, 0, 0) + nd];
    }
    sm[L::U + t] = v;
  }
  __syncthreads();
  const int el = threadIdx.x / NN, nd = threadIdx.x - el * NN;
  const int j = nd / P1, i = nd - j * P1;
  const int eg = e0 + el;
  const double* Uo = sm + L::U + el * L::US;   // own; neighbours at + k * NCV * NN
  // ---- own node fluxes
  {
    double s[NCV], gx[NCV], gy[NCV], Fx[NCV], Fy[NCV];
#pragma unroll
    for (int c = 0; c < NCV; ++c) s[c] = Uo[c * NN + nd];
    grad_at<P1>(op, Uo, sD, j, i, gx, gy);
    visc_flux(op, s, gx, gy, Fx, Fy);
#pragma unroll
    for (int c = 0; c < NCV; ++c) {
      sm[L::FX + (el * NCV + c) * NN + nd] = Fx[c];
      sm[L::FY + (el * NCV + c) * NN + nd] = Fy[c];
    }
  }
  // ---- face terms of this element: threads of row / column 0 own the four faces' lines
  {
    double Gf[NCV], gm[NCV], gp[NCV];
    double* GF = sm + L::GF + el * 4 * P1 * NCV;
    double* LF = sm + L::LF + el * 4 * P1 * NCV;
    if (i == 0) {   // x-faces of row j: right (own minus, R plus), left (L minus, own plus)
      face_terms<P1>(op, Uo, Uo + 1 * NCV * NN, sD, j, P, j, 0, 0, Gf, gm, gp);
#pragma unroll
      for (int c = 0; c < NCV; ++c) { GF[(FR * P1 + j) * NCV + c] = Gf[c]; LF[(FR * P1 + j) * NCV + c] = gm[c]; }
      face_terms<P1>(op, Uo + 2 * NCV * NN, Uo, sD, j, P, j, 0, 0, Gf, gm, gp);
#pragma unroll
      for (int c = 0; c < NCV; ++c) { GF[(FL * P1 + j) * NCV + c] = Gf[c]; LF[(FL * P1 + j) * NCV + c] = gp[c]; }
    }
    if (j == 0) {   // y-faces of column i: top (own minus, T plus), bottom (B minus, own plus)
      face_terms<P1>(op, Uo, Uo + 3 * NCV * NN, sD, P, i, 0, i, 1, Gf, gm, gp);
#pragma unroll
      for (int c = 0; c < NCV; ++c) { GF[(FT * P1 + i) * NCV + c] = Gf[c]; LF[(FT * P1 + i) * NCV + c] = gm[c]; }
      face_terms<P1>(op, Uo + 4 * NCV * NN, Uo, sD, P, i, 0, i, 1, Gf, gm, gp);
#pragma unroll
      for (int c = 0; c < NCV; ++c) { GF[(FB * P1 + i) * NCV + c] = Gf[c]; LF[(FB * P1 + i) * NCV + c] = gp[c]; }
    }
  }
  __syncthreads();
  if (eg >= ne) return;
  const int oy = eg / op.nex, ex = eg - oy * op.nex, ey = oy + op.row0;
  const double* GF = sm + L::GF + el * 4 * P1 * NCV;
  const double* LF = sm + L::LF + el * 4 * P1 * NCV;
  const double hx = 0.5 * op.dx, hy = 0.5 * op.dy;
  bool bad = false;
#pragma unroll
  for (int c = 0; c < NCV; ++c) {
    const double* Fx = sm + L::FX + (el * NCV + c) * NN;
    const double* Fy = sm + L::FY + (el * NCV + c) * NN;
    double bx = 0.0, by = 0.0;
#pragma unroll
    for (int q = 0; q < P1; ++q) {
      bx = fma(sDTW[i * P1 + q], Fx[j * P1 + q], bx);
      by = fma(sDTW[j * P1 + q], Fy[q * P1 + i], by);
    }
    if (i == P) bx += GF[(FR * P1 + j) * NCV + c];
    if (i == 0) bx -= GF[(FL * P1 + j) * NCV + c];
    bx -= op.sx * (0.5 * LF[(FR * P1 + j) * NCV + c]) * sD[P * P1 + i];
    bx -= op.sx * (0.5 * LF[(FL * P1 + j) * NCV + c]) * sD[i];
    if (j == P) by += GF[(FT * P1 + i) * NCV + c];
    if (j == 0) by -= GF[(FB * P1 + i) * NCV + c];
    by -= op.sy * (0.5 * LF[(FT * P1 + i) * NCV + c]) * sD[P * P1 + j];
    by -= op.sy * (0.5 * LF[(FB * P1 + i) * NCV + c]) * sD[j];
    const double fv = -bx / (hx * sW[i]) + -by / (hy * sW[j]);
    const long long g = nidx(op, c, ey, ex, j, i);
    const double out = accumulate ? fm[g] + fv : fv;
    fm[g] = out;
    bad |= !isfinite(out);
  }
  if (bad && status) atomicMin(status, (int)(op.e0 + eg));
}

}  // namespace

int launch2_visc(Ctx* c, const Op2DDev& op, const double* u, double* f, int m_first, int m_count, int accumulate) {
  if (op.problem != SISDC_NS2D) return SISDC_OK;
  if (op.nc != 4) return c->fail(SISDC_ERR_ARG, "NS2D needs four fields");
#define SISDC_VISC(P1_)                                                                                       \
  case P1_: {                                                                                                 \
    using L = Vb<P1_>;                                                                                        \
    const size_t smem = sizeof(double) * L::SIZE;                                                             \
    cudaFuncSetAttribute(k2_visc<P1_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);               \
    const int ne = op.nex * op.ney;                                                                           \
    k2_visc<P1_><<<dim3((ne + L::EB - 1) / L::EB, m_count), L::NT, smem, c->stream>>>(op, u, f, m_first,      \
                                                                                       accumulate, c->d_status); \
    return c->after_launch("k2_visc");                                                                        \
  }
  switch (op.p1) {
    SISDC_VISC(2)
    SISDC_VISC(3)
    SISDC_VISC(4)
    SISDC_VISC(5)
    SISDC_VISC(6)
    SISDC_VISC(7)
    SISDC_VISC(8)
    SISDC_VISC(9)
    default: return c->fail(SISDC_ERR_UNSUPPORTED, "NS2D degree outside 1..8");
  }
#undef SISDC_VISC
}

}  // namespace sisdc
