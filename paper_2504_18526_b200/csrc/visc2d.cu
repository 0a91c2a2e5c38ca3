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
// viscous flux, the face fluxes of its element ((face node, side) work items
// spread over all threads; the neighbour's flux at the shared face nodes is
// computed from the staged neighbour), then the divergence.  Not on the CG hot path: it runs once per right-hand-side
// evaluation (node caches, FAS defects), after the convection/SI kernels.
#include <cstdint>
#include <cstdlib>
#include "sisdc_dev2d.cuh"
#include "sisdc_host.h"

namespace sisdc {
namespace {

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
  static constexpr int XS = LF + EB * 4 * P1 * NCV;         // plus-side (q, g) of every face node [EB][4][P1][2 NCV]
  static constexpr int SIZE = XS + EB * 4 * P1 * 2 * NCV;
  static constexpr int DP = P1 + 1;                         // padded table rows (lane-varying row index: conflict free)
};

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
      ax = fma(D[i * (P1 + 1) + q], X[c * NN + j * P1 + q], ax);
      ay = fma(D[j * (P1 + 1) + q], X[c * NN + q * P1 + i], ay);
    }
    gx[c] = op.sx * ax;
    gy[c] = op.sy * ay;
  }
}

// one side of a face node: the normal viscous flux q of the staged element X at its node
// (jx, ix) and g = G_nn(s) [u] with the jump [u] = u- - u+ (sm, sp: the minus / plus states)
template <int P1>
__device__ __forceinline__ void face_side(const Op2DDev& op, double gpr, const double* X, const double* D, int jx,
                                          int ix, const double* s_mine, const double* jmp, int axis, double* q,
                                          double* g) {
  double gx[NCV], gy[NCV], Fx[NCV], Fy[NCV];
  grad_at<P1>(op, X, D, jx, ix, gx, gy);
  visc_flux(op, gpr, s_mine, gx, gy, Fx, Fy);
  apply_gnn(op, gpr, s_mine, jmp, axis, g);
#pragma unroll
  for (int c = 0; c < NCV; ++c) q[c] = axis == 0 ? Fx[c] : Fy[c];
}

template <int P1>
__global__ void __launch_bounds__(Vb<P1>::NT, P1 == 8 ? 3 : 2) k2_visc(Op2DDev op, const double* __restrict__ u, double* __restrict__ f,
                                                      int m_first, int accumulate, int* status) {
  using L = Vb<P1>;
  constexpr int NN = P1 * P1, P = P1 - 1;
  extern __shared__ double sm[];
  __shared__ double sD[P1 * (P1 + 1)], sDTW[P1 * (P1 + 1)], sW[P1], sWy[P1];
  const int m = m_first + blockIdx.y;
  const double gpr = op.gamma / op.pr;
  const double* um = u + (size_t)m * op.ns;
  double* fm = f + (size_t)m * op.ns;
  for (int t = threadIdx.x; t < NN; t += blockDim.x) {
    sD[(t / P1) * (P1 + 1) + t % P1] = op.tab[TabOff::D(P1) + t];
    sDTW[(t / P1) * (P1 + 1) + t % P1] = op.tab[TabOff::DTW(P1) + t];
  }
  for (int t = threadIdx.x; t < P1; t += blockDim.x) {   // 1 / (h w_i): the divergence divides by the mass
    sW[t] = 1.0 / (0.5 * op.dx * op.tab[TabOff::w(P1) + t]);
    sWy[t] = 1.0 / (0.5 * op.dy * op.tab[TabOff::w(P1) + t]);
  }
  const int ne = op.nex * op.ney;
  const int e0 = blockIdx.x * L::EB;
  // ---- stage own + face neighbours, all fields: EB * 5 * NCV contiguous runs of NN doubles, one run per
  // warp pass with the index arithmetic per RUN (it was per 8-byte element: a runtime division, a modulo
  // and a 64-bit index per copy, 35% of the kernel's samples)
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // lanes per run: NN / 2 sixteen-byte copies (NN even) or NN eight-byte copies; short runs (low degrees)
    // share a warp pass, GPW runs side by side
    constexpr int CPR = NN % 2 == 0 ? NN / 2 : NN;           // copies per run
    constexpr int GL = CPR < 32 ? CPR : 32;                  // lanes per run
    constexpr int GPW = 32 / GL;                             // runs per warp pass
    const int grp = lane / GL, gl = lane - grp * GL;
    for (int run = wid * GPW + grp; run < L::EB * 5 * NCV; run += nw * GPW) {
      if (grp >= GPW) break;
      const int el_ = run / (5 * NCV), r = run - el_ * (5 * NCV);
      const int k = r / NCV, c = r - k * NCV;
      const int eg_ = e0 + el_;
      double* dst = sm + L::U + run * NN;
      if (eg_ < ne) {
        const int oy = eg_ / op.nex, ex = eg_ - oy * op.nex, ey = oy + op.row0;
        int sx_ = ex, sy_ = ey;
        if (k == 1) sx_ = ex + 1 == op.nex ? 0 : ex + 1;
        if (k == 2) sx_ = ex == 0 ? op.nex - 1 : ex - 1;
        if (k == 3) sy_ = ynb(op, ey, 1);
        if (k == 4) sy_ = ynb(op, ey, -1);
        const double* src = um + nidx(op, c, sy_, sx_, 0, 0);
        if constexpr (NN % 2 == 0) {   // 16-byte copies (element runs are 16-byte aligned when NN is even)
          for (int t = 2 * gl; t < NN; t += 2 * GL) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(dst + t);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + t) : "memory");
          }
        } else {
          for (int t = gl; t < NN; t += GL) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(dst + t);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src + t) : "memory");
          }
        }
      } else {
        for (int t = gl; t < NN; t += GL) dst[t] = 0.0;
      }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
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
    visc_flux(op, gpr, s, gx, gy, Fx, Fy);
#pragma unroll
    for (int c = 0; c < NCV; ++c) {
      sm[L::FX + (el * NCV + c) * NN + nd] = Fx[c];
      sm[L::FY + (el * NCV + c) * NN + nd] = Fy[c];
    }
  }
  // accumulate mode: this node's f values are read now, behind the face work (the read-modify-write at
  // the end stalled 10% of the samples on them)
  double facc[NCV] = {0.0, 0.0, 0.0, 0.0};
  if (accumulate && eg < ne) {
    const int oy_ = eg / op.nex, ex_ = eg - oy_ * op.nex;
#pragma unroll
    for (int c = 0; c < NCV; ++c) facc[c] = fm[nidx(op, c, oy_ + op.row0, ex_, j, i)];
  }
  // ---- face terms of this element.  4 faces x P1 nodes x 2 sides: every (face node, side) is one
  // unit of work (gradient, flux, G_nn [u] of that side's element), spread over all threads of the
  // element instead of the P1 threads of row / column 0 (which left 7/8 of each warp idle through
  // four full flux evaluations).  The plus side hands (q, g) to the minus side through XS.
  {
    double* GF = sm + L::GF + el * 4 * P1 * NCV;
    double* LF = sm + L::LF + el * 4 * P1 * NCV;
    double* XS = sm + L::XS + el * 4 * P1 * 2 * NCV;
    for (int w0 = 0; w0 < 4 * P1 * 2; w0 += NN) {   // uniform trip count: block barrier inside
      const bool act = w0 + nd < 4 * P1 * 2;
      const int w = act ? w0 + nd : 0;
      const int fc = w / (2 * P1), k = (w >> 1) % P1, side = w & 1;   // side 0: minus, 1: plus
      const int axis = fc >= FT ? 1 : 0;
      // minus / plus elements (0 own, 1 R, 2 L, 3 T, 4 B) and their face nodes
      const int em = fc == FL ? 2 : fc == FB ? 4 : 0, ep = fc == FR ? 1 : fc == FT ? 3 : 0;
      const int jm = axis ? P : k, im = axis ? k : P, jp = axis ? 0 : k, ip = axis ? k : 0;
      const double* Xm = Uo + em * NCV * NN;
      const double* Xp = Uo + ep * NCV * NN;
      double sm_[NCV], sp_[NCV], jmp[NCV], q[NCV], g[NCV];
#pragma unroll
      for (int c = 0; c < NCV; ++c) {
        sm_[c] = Xm[c * NN + jm * P1 + im];
        sp_[c] = Xp[c * NN + jp * P1 + ip];
        jmp[c] = sm_[c] - sp_[c];
      }
      if (side) face_side<P1>(op, gpr, Xp, sD, jp, ip, sp_, jmp, axis, q, g);
      else face_side<P1>(op, gpr, Xm, sD, jm, im, sm_, jmp, axis, q, g);
      double* xs = XS + (fc * P1 + k) * 2 * NCV;
      if (act && side) {
#pragma unroll
        for (int c = 0; c < NCV; ++c) { xs[c] = q[c]; xs[NCV + c] = g[c]; }
      }
      __syncthreads();   // the two sides of a face node may sit in different warps (odd P1)
      if (act && !side) {
        const double mu0 = axis == 0 ? op.mux : op.muy;
        const bool own_minus = fc == FR || fc == FT;   // the own element's lift uses its own side's g
#pragma unroll
        for (int c = 0; c < NCV; ++c) {
          const double qb = xs[c], gp = xs[NCV + c];
          GF[(fc * P1 + k) * NCV + c] = mu0 * (0.5 * (g[c] + gp)) - 0.5 * (q[c] + qb);
          LF[(fc * P1 + k) * NCV + c] = own_minus ? g[c] : gp;
        }
      }
    }
  }
  __syncthreads();
  if (eg >= ne) return;
  const int oy = eg / op.nex, ex = eg - oy * op.nex, ey = oy + op.row0;
  const double* GF = sm + L::GF + el * 4 * P1 * NCV;
  const double* LF = sm + L::LF + el * 4 * P1 * NCV;
  bool bad = false;
#pragma unroll
  for (int c = 0; c < NCV; ++c) {
    const double* Fx = sm + L::FX + (el * NCV + c) * NN;
    const double* Fy = sm + L::FY + (el * NCV + c) * NN;
    double bx = 0.0, by = 0.0;
#pragma unroll
    for (int q = 0; q < P1; ++q) {
      bx = fma(sDTW[i * (P1 + 1) + q], Fx[j * P1 + q], bx);
      by = fma(sDTW[j * (P1 + 1) + q], Fy[q * P1 + i], by);
    }
    if (i == P) bx += GF[(FR * P1 + j) * NCV + c];
    if (i == 0) bx -= GF[(FL * P1 + j) * NCV + c];
    bx -= op.sx * (0.5 * LF[(FR * P1 + j) * NCV + c]) * sD[P * (P1 + 1) + i];
    bx -= op.sx * (0.5 * LF[(FL * P1 + j) * NCV + c]) * sD[i];
    if (j == P) by += GF[(FT * P1 + i) * NCV + c];
    if (j == 0) by -= GF[(FB * P1 + i) * NCV + c];
    by -= op.sy * (0.5 * LF[(FT * P1 + i) * NCV + c]) * sD[P * (P1 + 1) + j];
    by -= op.sy * (0.5 * LF[(FB * P1 + i) * NCV + c]) * sD[j];
    const double fv = -bx * sW[i] + -by * sWy[j];
    const long long g = nidx(op, c, ey, ex, j, i);
    const double out = accumulate ? facc[c] + fv : fv;
    fm[g] = out;
    bad |= !isfinite(out);
  }
  if (bad && status) atomicMin(status, (int)(op.e0 + eg));
}

}  // namespace

int launch2_visc(Ctx* c, const Op2DDev& op, const double* u, double* f, int m_first, int m_count, int accumulate) {
  if (op.problem != SISDC_NS2D) return SISDC_OK;
  if (op.nc != 4) return c->fail(SISDC_ERR_ARG, "NS2D needs four fields");
  // P = 7: warp-per-element tensor-core kernel (ops2d.cu); SISDC_VISC_LINE=1 keeps the line formulation (A/B)
  const char* vl = getenv("SISDC_VISC_LINE");   // read per call: the GPU test compares the two kernels
  const bool line_only = vl && vl[0] == '1';
  if (op.p1 == 8 && !line_only && ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(f)) & 15) == 0 &&
      (op.ns & 1) == 0)
    return launch2_visc8(c, op, u, f, m_first, m_count, accumulate);
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
