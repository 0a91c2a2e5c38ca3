// Cluster-resident Jacobi-PCG for the implicit substep (M + a B[C]) x = M rhs.
//
// Replaces the reference's SuperLU solve + defect iteration
// (dgsem.py:492-533) by the pinned PCG of oracle/cg.py (Chronopoulos-Gear
// form: the Hestenes-Stiefel iterates with ONE fused reduction per iteration,
// (gamma, delta, rho) = ((r,u), (w,u), (r,r)) with u = D^-1 r, w = A u).
//
// The whole solve runs in ONE launch: a thread-block cluster of K <= 16 CTAs
// (one per SM) owns the elements in contiguous blocks, one thread per node.
// x, r, u, w, p, s and the Jacobi reciprocal live in registers; u (read by
// the element contraction) and the element fluxes q live in shared memory.
//
// Inter-CTA traffic is push-only (sm_90+/sm_100a DSMEM):
//  * the reduction: warps shuffle-reduce, warp 0 pre-reduces the CTA and
//    writes it with st.async into a slot of every CTA of the cluster; each
//    store completes a transaction count on the RECEIVER's mbarrier.  After
//    its own mbarrier phase completes a CTA sums the K slots in rank order
//    -> bitwise-identical scalars everywhere, no cluster barrier.
//  * the face halo: boundary nodes push w with the partials (r0, w0 once with
//    the setup reduction); the receiver advances the neighbours' s and r
//    itself, s' = fma(beta, s, w), r' = fma(-alpha, s', r), u' = r' dinv, with
//    exactly the owner's operations, so u's halo needs no extra exchange.
// One mbarrier wait per iteration; slot/halo buffers alternate by parity.
#include <cooperative_groups.h>
#include <string>
#include <type_traits>
#include "sisdc_dev.cuh"
#include "sisdc_host.h"

namespace cg = cooperative_groups;

namespace sisdc {

// fused stage rhs (sdc.py:218-237): x0 = rhs = base + dt W f_old (+ g) + dt_m conv(conv_in) - h,
// computed in the CG prologue with k_stage_rhs's exact operations (bitwise)
struct CgStage {
  const double* base;
  const double* conv_in;
  const double* f_old;
  const double* g;
  const double* h;
  double* conv_out;
  double dt_m, dt, gl, gr;   // gl / gr: Dirichlet outside states at conv_in's time
  int M;
  double w[MAXM];
};

struct CgArgs {
  int stage;        // 1: x0 from the fused stage rhs (sg), else x0 = rhs
  CgStage sg;
  Op1DDev op;
  CoefDev coef;
  double a;
  const double* rhs;
  double* x;
  double rtol2;
  int maxit, E, K;
  int* status;
  int* log_it;
  double* log_margin;
  int log_cap;
  long long* timing;   // diagnostics: clock64 stamps of CTA 0 (nullable)
  // grid mode (levels beyond one cluster: K > 16 CTAs of a cooperative launch, CL = false): halo and
  // reduction exchange through global memory, one grid barrier per exchange.  Layout (doubles):
  // HXD [K][4 P1] | HU0 [K][2 P1] | HRWS [2][K][8 P1] | slots [2][K][NVS]
  double* gws;
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async(uint32_t ra, double v, uint32_t rm) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
               :: "r"(ra), "d"(v), "r"(rm) : "memory");
}
__device__ __forceinline__ void st_async2(uint32_t ra, double v0, double v1, uint32_t rm) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               :: "r"(ra), "d"(v0), "d"(v1), "r"(rm) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(m) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(m), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
               :: "r"(m), "r"(parity) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum_j a[j] b[j] with three interleaved accumulators (shorter FMA chain)
template <int P1>
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int j = 0; j < P1; j += 3) {
    s0 = fma(a[j], b[j], s0);
    if (j + 1 < P1) s1 = fma(a[j + 1], b[j + 1], s1);
    if (j + 2 < P1) s2 = fma(a[j + 2], b[j + 2], s2);
  }
  return (s0 + s1) + s2;
}

constexpr int NVS = 6;   // setup reduction: gamma, delta, rho, (b,b), #nonzero b, pad
constexpr int NVL = 4;   // loop reduction:  gamma, delta, rho, pad

template <int P1>
struct CgShared {
  unsigned long long* mbar;   // [0],[1] reduction parity 0/1, [2] x0 halo, [3] u0 halo
  double* st;
  double* Xs;     // x0 (setup only)
  double* Ub;     // u, read by the element contraction
  double* Q;      // element fluxes
  double* Cs;     // coefficient: own nodes + [NL] left halo node P, [NL+1] right halo node 0
  double* HXD;    // halo (x0, dinv) pairs [2 sides][P1][2]
  double* HX;     // halo x0 [2][P1]
  double* HD;     // halo dinv [2][P1]
  double* HU0;    // halo u0 [2][P1]
  double* HU;     // halo u formed locally [2][P1]
  double* HRWS;   // pushed halo (r, w, s, pad) [2 parity][2 sides][P1][4]
  double* slots;  // reduction slots [2 parity][16 ranks][NVS]
  double* wbuf;   // per-thread partials [NVS][blockDim] (structure of arrays)
  double* bcast;  // reduced scalars [NVS]
  double* HQ;     // halo face fluxes q: [0] left element node P, [1] right element node 0
};

// nodes per element padded to an even count: elements start 16-byte aligned
__host__ __device__ constexpr int padded(int p1) { return p1 + (p1 & 1); }

template <int P1>
__device__ __forceinline__ CgShared<P1> carve(double* sm, int E, int nt) {
  CgShared<P1> s;
  const int NL = E * P1, NLP = E * padded(P1);
  double* q = sm;
  s.mbar = reinterpret_cast<unsigned long long*>(q); q += 4;
  s.HXD = q; q += 4 * P1;          // 16-byte aligned (v2 stores)
  s.HRWS = q; q += 16 * P1;        // 16-byte aligned
  s.slots = q; q += 2 * 16 * NVS;  // 16-byte aligned (NVS even)
  s.Xs = q; q += NLP;              // padded element layout, 16-byte aligned
  s.Ub = q; q += NLP;
  s.Q = q; q += NLP;
  s.wbuf = q; q += NVS * nt;
  s.bcast = q; q += 8;
  s.st = q; q += TabOff::size(P1);
  s.Cs = q; q += NL + 2;
  s.HX = q; q += 2 * P1;
  s.HD = q; q += 2 * P1;
  s.HU0 = q; q += 2 * P1;
  s.HU = q; q += 2 * P1;
  s.HQ = q; q += 2;
  return s;
}
static size_t cg_smem_bytes(int p1, int E, int nt) {
  return sizeof(double) * (4 + 4 * p1 + 16 * p1 + 2 * 16 * NVS + 3 * E * padded(p1) + NVS * nt + 8 +
                           TabOff::size(p1) + E * p1 + 2 + 8 * p1 + 2);
}

template <bool CL, int P1, bool DIR>
__global__ void __launch_bounds__(384) k_cg1d(CgArgs A) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = P1 - 1;
  const Op1DDev& op = A.op;
  int rank = 0;
  if constexpr (CL) rank = (int)cg::this_cluster().block_rank();
  const bool GM = !CL && A.K > 1;   // grid mode
  if (GM) rank = blockIdx.x;
  cg::grid_group grid = cg::this_grid();
  double* const gHXD = A.gws;
  double* const gHU0 = gHXD + (size_t)A.K * 4 * P1;
  double* const gHRWS = gHU0 + (size_t)A.K * 2 * P1;
  double* const gSLOT = gHRWS + (size_t)2 * A.K * 8 * P1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int P1P = padded(P1);
  const CgShared<P1> s = carve<P1>(sm, A.E, blockDim.x);
  const int K = A.K;
  const int e0 = rank * A.E;
  const int e1 = min(op.ne, e0 + A.E);
  const int nl = (e1 - e0) * P1, NL = A.E * P1;
  const int L = threadIdx.x, el = L / P1, i = L - el * P1;
  const bool own = L < nl;
  const bool first = el == 0, last = (el + 1) * P1 >= nl;
  const int ob = el * P1P, oL = ob + i;   // element base / node slot in the padded layout
  const bool helper = wid == 0;            // warp 0 rebuilds the halo element values
  const int egL = wrap(e0 - 1, op.ne), egR = wrap(e1, op.ne);
  const int rL = egL / A.E, rR = egR / A.E;
  uint32_t mb[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) mb[j] = sa(&s.mbar[j]);
  if constexpr (CL) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) mbar_init(mb[j]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  pdl_launch_dependents();
  const bool stamp = A.timing != nullptr && rank == 0 && threadIdx.x == 0;
  if (stamp) A.timing[0] = clock64();
  for (int t = threadIdx.x; t < TabOff::size(P1); t += blockDim.x) s.st[t] = op.tab[t];   // constant tables
  if constexpr (CL) cg::this_cluster().sync();   // mbarriers initialised cluster-wide (overlaps the predecessor)
  pdl_wait();   // everything below may read the predecessor's output
  double ci = 0.0, x = 0.0;
  if (A.stage) {   // x0 = the stage rhs of this substep, conv(conv_in) as conv_node (ops1d.cu)
    const CgStage& g = A.sg;
    const size_t gi = (size_t)e0 * P1 + L;
    if (own) s.Ub[oL] = g.conv_in[gi];   // staging (s.Ub is rewritten with u0 after the setup barriers)
    __syncthreads();
    if (own) {
      const double* ue = s.Ub + ob;
      const double* DTWs = s.st + TabOff::DTW(P1);
      double v = 0.0;
#pragma unroll 4
      for (int k = 0; k < P1; ++k) v = fma(DTWs[i * P1 + k], flux(op, ue[k]), v);
      const int eg = e0 + el;
      if (i == P) {
        const double nb = (DIR && eg == op.ne - 1) ? g.gr
                          : (last ? g.conv_in[(size_t)wrap(eg + 1, op.ne) * P1] : s.Ub[ob + P1P]);
        v -= rusanov(op, ue[P], nb);
      }
      if (i == 0) {
        const double nb = (DIR && eg == 0) ? g.gl
                          : (first ? g.conv_in[(size_t)wrap(eg - 1, op.ne) * P1 + P] : s.Ub[ob - P1P + P]);
        v += rusanov(op, nb, ue[0]);
      }
      const double cv = v * s.st[TabOff::minv(P1) + i];
      if (g.conv_out) g.conv_out[gi] = cv;
      double q = 0.0;
      if (g.f_old) {
        double acc = 0.0;
        for (int j = 0; j < g.M; ++j) acc = fma(g.w[j], g.f_old[(size_t)j * op.n + gi], acc);
        q = g.dt * acc;
      }
      if (g.g) q = q + g.g[gi];
      double rr = (g.base[gi] + q) + g.dt_m * cv;
      if (g.h) rr = rr - g.h[gi];
      x = rr;
    }
  } else if (own) {
    x = A.rhs[(size_t)e0 * P1 + L];   // x0 = rhs
  }
  if (own) {
    ci = coef_at(op, A.coef, e0 + el, i);
    s.Cs[L] = ci;
    s.Xs[oL] = x;
  }
  if (L == 0) s.Cs[NL] = coef_at(op, A.coef, egL, P);
  if (L == 1) s.Cs[NL + 1] = coef_at(op, A.coef, egR, 0);
  __syncthreads();

  const double* D = s.st + TabOff::D(P1);
  const double* DTW = s.st + TabOff::DTW(P1);
  const double mi = s.st[TabOff::m(P1) + i];
  const double sc = op.s, mu0 = op.mu0, a = A.a;
  const double cP = s.Cs[min(el * P1 + P, NL - 1)], c0 = s.Cs[min(el * P1, NL - 1)];
  // Dirichlet outer faces (dgsem.py:282-289): outside value 0 in the operator (the
  // boundary data moves to the right-hand side), one-sided q and C, lift weight 1
  // (DIR: a separate instantiation, so the periodic kernel is unchanged)
  const bool dirL = DIR && e0 + el == 0;
  const bool dirR = DIR && e0 + el == op.ne - 1;
  const double cR = dirR ? cP : (last ? s.Cs[NL + 1] : s.Cs[min((el + 1) * P1, NL - 1)]);
  const double cL = dirL ? c0 : (first ? s.Cs[NL] : s.Cs[min(max(el * P1 - 1, 0), NL - 1)]);
  double dg = 1.0;
  if (own) {   // Jacobi diagonal diag(M + a B[C]) (closed form of dgsem.py:414-490)
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < P1; ++k) d = fma(s.st[TabOff::D2W(P1) + i * P1 + k], s.Cs[el * P1 + k], d);
    d = sc * d;
    if (i == P) d += dirR ? mu0 * cP - 2.0 * sc * cP * D[P * P1 + P] : mu0 * (0.5 * (cP + cR)) - sc * cP * D[P * P1 + P];
    if (i == 0) d += dirL ? mu0 * c0 + 2.0 * sc * c0 * D[0] : mu0 * (0.5 * (cL + c0)) + sc * c0 * D[0];
    dg = mi + a * d;
  }
  const double dinv = 1.0 / dg;
  // per-node face constants of the SIP operator (dgsem.py:290-308)
  const double muR = mu0 * (0.5 * (cP + cR)), muL = mu0 * (0.5 * (cL + c0));
  const double kR = sc * ((dirR ? 1.0 : 0.5) * cP), kL = sc * ((dirL ? 1.0 : 0.5) * c0);
  const double DPi = D[P * P1 + i], D0i = D[i];

  // ---- push targets (boundary nodes) and reduction targets (warp 0 lanes)
  const bool pushL = own && first, pushR = own && last;   // first elem -> left nb's right side, last -> right nb's left
  uint32_t tL[4] = {0, 0, 0, 0}, tR[4] = {0, 0, 0, 0};    // remote: HXD, HU0, HRWS parity 0, HRWS parity 1
  uint32_t mL[4] = {0, 0, 0, 0}, mR[4] = {0, 0, 0, 0};
  uint32_t rslot[2] = {0, 0}, rmb[2] = {0, 0};
  if constexpr (CL) {
    if (pushL) {
      tL[0] = mapa(sa(s.HXD + 2 * (P1 + i)), rL);
      tL[1] = mapa(sa(s.HU0 + P1 + i), rL);
      tL[2] = mapa(sa(s.HRWS + 4 * (P1 + i)), rL);
      tL[3] = mapa(sa(s.HRWS + 8 * P1 + 4 * (P1 + i)), rL);
#pragma unroll
      for (int j = 0; j < 4; ++j) mL[j] = mapa(mb[j], rL);
    }
    if (pushR) {
      tR[0] = mapa(sa(s.HXD + 2 * i), rR);
      tR[1] = mapa(sa(s.HU0 + i), rR);
      tR[2] = mapa(sa(s.HRWS + 4 * i), rR);
      tR[3] = mapa(sa(s.HRWS + 8 * P1 + 4 * i), rR);
#pragma unroll
      for (int j = 0; j < 4; ++j) mR[j] = mapa(mb[j], rR);
    }
    if (wid < 5 && lane < K) {   // the reducing warps (csum: at most 5 quantities)
      rslot[0] = mapa(sa(s.slots + rank * NVS), lane);
      rslot[1] = mapa(sa(s.slots + (16 + rank) * NVS), lane);
      rmb[0] = mapa(mb[0], lane);
      rmb[1] = mapa(mb[1], lane);
    }
  }
  // halo bytes riding on a reduction's mbarrier: (r0, w0) pairs with the setup
  // reduction, then w alone per iteration (the receiver advances the
  // neighbours' r and s itself, see the loop)
  uint32_t halo_rws_bytes = 2u * P1 * 16u;

  // Cluster sum of NV values into buffer `par` (with the (r,w,s) halo pushed
  // by the caller on the same mbarrier); identical bits in every CTA.
  // Every thread parks its NR partials in shared memory (structure of
  // arrays); each quantity is summed in a fixed order (per lane over the
  // warps, then across the lanes), the CTA totals are pushed to every CTA
  // (NV slots, NR <= NV real values), and after the K totals have arrived
  // they are summed in rank order and broadcast through shared memory.
  //  * P1 < 9: warp 0 does all of it, the NR quantities interleaved, remote
  //    stores in pairs.
  //  * PARRED (P1 >= 9): warp j reduces quantity j (j, j + nred, ... with
  //    fewer warps) and pushes it itself; the pad slots are not pushed.
  //    Measured on the cfg2 fine level: 1.78 -> 1.61 us per iteration.  At
  //    P1 = 5 the single-value pushes (twice the mbarrier transactions) cost
  //    more than the parallel sums save (1.70 -> 2.08 us), hence the split.
  // Same operations in the same order per quantity either way (bitwise).
  // idle(): warp 0 work placed in the shadow of the cluster wait (before the
  // final broadcast barrier)
  constexpr bool PARRED = P1 >= 9;
#ifndef SISDC_CG1_GATHER
#define SISDC_CG1_GATHER 1
#endif
  constexpr bool GATHER = SISDC_CG1_GATHER;
  auto csum = [&](auto& v, auto nr_tag, auto nv_tag, int par, uint32_t& phase, auto&& idle) {
    constexpr int NR = decltype(nr_tag)::value;
    constexpr int NV = decltype(nv_tag)::value;
    constexpr int MAXW = 12;   // <= 384 threads
    const int nt = blockDim.x;
#pragma unroll
    for (int j = 0; j < NR; ++j) s.wbuf[j * nt + threadIdx.x] = v[j];
    __syncthreads();
    // pairwise tree over the <= 12 values of this lane, then the warp sum
    auto qsum = [&](int j) {
      double e[MAXW];
#pragma unroll
      for (int m = 0; m < MAXW; ++m) e[m] = (lane + 32 * m < nt) ? s.wbuf[j * nt + lane + 32 * m] : 0.0;
#pragma unroll
      for (int w2 = 1; w2 < MAXW; w2 *= 2)
#pragma unroll
        for (int m = 0; m + w2 < MAXW; m += 2 * w2) e[m] += e[m + w2];
      return warp_sum(e[0]);
    };
    if constexpr (PARRED) {
      const int nred = min(NR, nt >> 5);   // reducing warps
      if (wid < nred) {
        for (int j = wid; j < NR; j += nred) {
          const double tj = qsum(j);
          if constexpr (CL) {
            if (lane < K) st_async((par ? rslot[1] : rslot[0]) + 8 * j, tj, (par ? rmb[1] : rmb[0]));
          } else {
            if (lane == 0) s.bcast[j] = tj;
          }
        }
        if constexpr (CL) {
          if (wid == 0) {   // the NV - NR pad slots are never read: not pushed
            if (lane == 0) mbar_expect((par ? mb[1] : mb[0]), 8u * K * NR + halo_rws_bytes);
            idle();
          }
          mbar_wait((par ? mb[1] : mb[0]), phase);
          const double* slots = s.slots + par * 16 * NVS;
          for (int j = wid; j < NR; j += nred) {   // K <= 16 slots: 4 butterfly levels
            double q = lane < K ? slots[lane * NVS + j] : 0.0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
            if (lane == 0) s.bcast[j] = q;
          }
        } else {
          if (wid == 0) idle();
        }
      }
    } else if (GATHER && CL && min(NR, nt >> 5) > 1) {
      // P1 < 9 variant: parallel sums, totals gathered to warp 0 through shared
      // memory and a named barrier of the reducing warps, paired pushes by warp
      // 0 (the transaction count of a single reducing warp), parallel receives
      const int nred = min(NR, nt >> 5);
      if (wid < nred) {
        for (int j = wid; j < NR; j += nred) {
          const double tj = qsum(j);
          if (lane == 0) s.wbuf[j * nt] = tj;   // region j is read by this warp only
        }
        asm volatile("bar.sync 1, %0;" ::"r"(nred * 32) : "memory");
        if (wid == 0) {
          double t[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) t[j] = j < NR ? s.wbuf[j * nt] : 0.0;
          if (lane < K)
#pragma unroll
            for (int j = 0; j < NV; j += 2) st_async2((par ? rslot[1] : rslot[0]) + 8 * j, t[j], t[j + 1], (par ? rmb[1] : rmb[0]));
          if (lane == 0) mbar_expect((par ? mb[1] : mb[0]), 8u * K * NV + halo_rws_bytes);
          idle();
        }
        mbar_wait((par ? mb[1] : mb[0]), phase);
        const double* slots = s.slots + par * 16 * NVS;
        for (int j = wid; j < NR; j += nred) {   // K <= 16 slots: 4 butterfly levels
          double q = lane < K ? slots[lane * NVS + j] : 0.0;
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
          if (lane == 0) s.bcast[j] = q;
        }
      }
    } else if (wid == 0) {
      double t[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) t[j] = 0.0;
#pragma unroll
      for (int j = 0; j < NR; ++j) t[j] = qsum(j);
      if constexpr (CL) {
        const double* slots = s.slots + par * 16 * NVS;
        if (lane < K)
#pragma unroll
          for (int j = 0; j < NV; j += 2) st_async2((par ? rslot[1] : rslot[0]) + 8 * j, t[j], t[j + 1], (par ? rmb[1] : rmb[0]));
        if (lane == 0) mbar_expect((par ? mb[1] : mb[0]), 8u * K * NV + halo_rws_bytes);
        idle();
        mbar_wait((par ? mb[1] : mb[0]), phase);
#pragma unroll
        for (int j = 0; j < NR; ++j) {   // K <= 16 slots: 4 butterfly levels
          double q = lane < K ? slots[lane * NVS + j] : 0.0;
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
          t[j] = q;
        }
      } else {
        idle();
      }
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < NR; ++j) s.bcast[j] = t[j];
    }
    if constexpr (CL) phase ^= 1;
    __syncthreads();
    if (GM) {   // CTA totals -> global slots, grid barrier (also publishes the halo), sum in rank order
      double* slots = gSLOT + (size_t)par * K * NVS;
      if (threadIdx.x < NR) slots[(size_t)rank * NVS + threadIdx.x] = s.bcast[threadIdx.x];
      __threadfence();
      grid.sync();
      if (wid == 0) {
#pragma unroll
        for (int j = 0; j < NR; ++j) {   // lane-strided over the ranks, then the butterfly: one fixed order everywhere
          double q = 0.0;
          for (int m = lane; m < K; m += 32) q += __ldcg(slots + (size_t)m * NVS + j);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
          if (lane == 0) s.bcast[j] = q;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = s.bcast[j];
  };

  // w = A v on own nodes: v = own shared vector, hv = halo values [left P1][right P1]
  // element rows of D and D^T W for this node, in registers
  double Dr[P1], DTr[P1];
#pragma unroll
  for (int j = 0; j < P1; ++j) {
    Dr[j] = D[i * P1 + j];
    DTr[j] = DTW[i * P1 + j];
  }
  // sum_j row[j] e[j] over a padded (16-byte aligned) element with double2 loads
  auto erow = [&](const double (&row)[P1], const double* e) -> double {
    const double2* e2 = reinterpret_cast<const double2*>(e);
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int j2 = 0; j2 < P1P / 2; ++j2) {
      const double2 t = e2[j2];
      g0 = fma(row[2 * j2], t.x, g0);
      if (2 * j2 + 1 < P1) g1 = fma(row[2 * j2 + 1], t.y, g1);
    }
    return g0 + g1;
  };
  auto matvec = [&](const double* v, const double* hv) -> double {
    if (own) s.Q[oL] = ci * (sc * erow(Dr, v + ob));
    __syncthreads();
    if (!own) return 0.0;
    double B = erow(DTr, s.Q + ob);
    const double pn = dirR ? 0.0 : (last ? hv[P1] : v[ob + P1P]);
    const double pp = dirL ? 0.0 : (first ? hv[P] : v[ob - P1P + P]);
    const double jr = v[ob + P] - pn;
    const double jl = pp - v[ob];
    if (i == P) {
      const double qn = dirR ? s.Q[ob + P] : (last ? cR * (sc * dot3<P1>(D, hv + P1)) : s.Q[ob + P1P]);
      B += -(0.5 * (s.Q[ob + P] + qn)) + muR * jr;
    }
    if (i == 0) {
      const double qp = dirL ? s.Q[ob] : (first ? cL * (sc * dot3<P1>(D + P * P1, hv)) : s.Q[ob - P1P + P]);
      B -= -(0.5 * (qp + s.Q[ob])) + muL * jl;
    }
    B -= (kR * jr) * DPi;
    B -= (kL * jl) * D0i;
    return fma(a, B, mi * v[oL]);
  };

  // ---- setup 1: halo (x0, dinv) -> r0 = b - A x0, u0 = D^-1 r0
  if constexpr (CL) {
    if (threadIdx.x == 0) mbar_expect(mb[2], 2u * P1 * 16u);
    if (pushL) st_async2(tL[0], x, dinv, mL[2]);
    if (pushR) st_async2(tR[0], x, dinv, mR[2]);
    mbar_wait(mb[2], 0);
  } else if (GM) {   // my last element is the right neighbour's left halo, my first the left one's right halo
    if (own && last) { double* g = gHXD + (size_t)rR * 4 * P1; g[2 * i] = x; g[2 * i + 1] = dinv; }
    if (own && first) { double* g = gHXD + (size_t)rL * 4 * P1; g[2 * (P1 + i)] = x; g[2 * (P1 + i) + 1] = dinv; }
    __threadfence();
    grid.sync();
    if (threadIdx.x < 4 * P1) s.HXD[threadIdx.x] = __ldcg(gHXD + (size_t)rank * 4 * P1 + threadIdx.x);
    __syncthreads();
  } else {
    if (own && last) { s.HXD[2 * i] = x; s.HXD[2 * i + 1] = dinv; }
    if (own && first) { s.HXD[2 * (P1 + i)] = x; s.HXD[2 * (P1 + i) + 1] = dinv; }
    __syncthreads();
  }
  if (helper && lane < 2 * P1) {
    s.HX[lane] = s.HXD[2 * lane];
    s.HD[lane] = s.HXD[2 * lane + 1];
  }
  // b = M rhs (+ a M D(0; t): the Dirichlet data of the affine SIP, dgsem.py:517-529)
  const double b0 = mi * x;
  double bi = b0;
  if (dirL) bi += a * ((i == 0 ? mu0 * c0 * op.gl : 0.0) + sc * c0 * op.gl * D0i);
  if (dirR) bi += a * ((i == P ? mu0 * cP * op.gr : 0.0) - sc * cP * op.gr * DPi);
  double r = bi - matvec(s.Xs, s.HX);
  double u = r * dinv;
  // ---- setup 2: halo u0 -> w0 = A u0
  if (own) s.Ub[oL] = u;
  if constexpr (CL) {
    if (threadIdx.x == 0) mbar_expect(mb[3], 2u * P1 * 8u);
    if (pushL) st_async(tL[1], u, mL[3]);
    if (pushR) st_async(tR[1], u, mR[3]);
    mbar_wait(mb[3], 0);
  } else if (GM) {
    if (own && last) gHU0[(size_t)rR * 2 * P1 + i] = u;
    if (own && first) gHU0[(size_t)rL * 2 * P1 + P1 + i] = u;
    __threadfence();
    grid.sync();
    if (threadIdx.x < 2 * P1) s.HU0[threadIdx.x] = __ldcg(gHU0 + (size_t)rank * 2 * P1 + threadIdx.x);
  } else {
    if (own && last) s.HU0[i] = u;
    if (own && first) s.HU0[P1 + i] = u;
  }
  __syncthreads();
  if (stamp) A.timing[1] = clock64();
  double w = matvec(s.Ub, s.HU0);
  double p = 0.0, sv = 0.0;   // p_{-1} = s_{-1} = 0
  // push (r0, w0) with the setup reduction (parity 0; s_{-1} = 0 is implied),
  // then w alone with every loop reduction: one mbarrier transaction per
  // boundary node instead of two
  auto push_rws = [&](int par, bool setup) {
    if constexpr (CL) {
      if (setup) {
        if (pushL) st_async2((par ? tL[3] : tL[2]), r, w, (par ? mL[1] : mL[0]));
        if (pushR) st_async2((par ? tR[3] : tR[2]), r, w, (par ? mR[1] : mR[0]));
      } else {
        if (pushL) st_async((par ? tL[3] : tL[2]) + 8, w, (par ? mL[1] : mL[0]));
        if (pushR) st_async((par ? tR[3] : tR[2]) + 8, w, (par ? mR[1] : mR[0]));
      }
    } else if (GM) {   // published by the grid barrier of the reduction that follows
      if (own && last) { double* h = gHRWS + ((size_t)par * K + rR) * 8 * P1; h[4 * i] = r; h[4 * i + 1] = w; }
      if (own && first) {
        double* h = gHRWS + ((size_t)par * K + rL) * 8 * P1;
        h[4 * (P1 + i)] = r;
        h[4 * (P1 + i) + 1] = w;
      }
    } else {
      double* h = s.HRWS + par * 8 * P1;
      if (own && last) { h[4 * i] = r; h[4 * i + 1] = w; h[4 * i + 2] = sv; }
      if (own && first) { h[4 * (P1 + i)] = r; h[4 * (P1 + i) + 1] = w; h[4 * (P1 + i) + 2] = sv; }
    }
  };
  push_rws(0, true);
  uint32_t ph0 = 0, ph1 = 0;   // mbarrier phases of the two reduction buffers (scalars: no local array)
  double v6[NVS] = {own ? r * u : 0.0, own ? w * u : 0.0, own ? r * r : 0.0, own ? bi * bi : 0.0,
                    (own && b0 != 0.0) ? 1.0 : 0.0, 0.0};   // b == 0 test on M rhs (dgsem.py:509-511)
  if (stamp) A.timing[2] = clock64();
  csum(v6, std::integral_constant<int, 5>{}, std::integral_constant<int, NVS>{}, 0, ph0, [] {});
  halo_rws_bytes = 2u * P1 * 8u;
  if (stamp) A.timing[3] = clock64();
  double gamma = v6[0], rho = v6[2];
  const double thr = A.rtol2 * v6[3];
  if (v6[4] == 0.0) {   // b == 0 -> zeros (dgsem.py:510-511)
    if (own) A.x[(size_t)e0 * P1 + L] = 0.0;
    return;
  }
  double alpha = gamma / v6[1], beta = 0.0;
  double rgamma, ralpha;   // formed by warp 0 inside each loop reduction
  double hr = 0.0, hs = 0.0;   // helper lanes: the neighbours' r and s at halo node `lane`
  int k = 0;
  bool ok = true;
  while (rho > thr) {
    if (k >= A.maxit) { ok = false; break; }
    const int par = k & 1;          // halo data from the previous reduction
    // neighbour u_{k+1} from its pushed (r, w, s): the owner's exact operations
    if (helper) {   // warp 0 rebuilds the neighbours' u: their s and r advanced here, w pushed
      if (lane < 2 * P1) {
        const double* h = GM ? gHRWS + ((size_t)par * K + rank) * 8 * P1 + 4 * lane : s.HRWS + par * 8 * P1 + 4 * lane;
        const double h0 = GM ? __ldcg(h) : h[0], h1 = GM ? __ldcg(h + 1) : h[1];   // L1 may hold the line of two iterations ago
        if (k == 0) {   // r0 from the setup push, s_{-1} = 0
          hr = h0;
          hs = 0.0;
        }
        hs = fma(beta, hs, h1);
        hr = fma(-alpha, hs, hr);
        s.HU[lane] = hr * s.HD[lane];
      }
    }
    p = fma(beta, p, u);
    sv = fma(beta, sv, w);
    x = fma(alpha, p, x);
    r = fma(-alpha, sv, r);
    u = r * dinv;
    if (own) s.Ub[oL] = u;
    const bool sub = stamp && k == 5;
    if (sub) A.timing[70] = clock64();
    __syncthreads();
    if (sub) A.timing[71] = clock64();
    w = matvec(s.Ub, s.HU);
    if (sub) A.timing[72] = clock64();
    push_rws(par ^ 1, false);
    double v4[NVL] = {own ? r * u : 0.0, own ? w * u : 0.0, own ? r * r : 0.0, 0.0};
    // 1 / alpha and 1 / gamma (needed by the scalar recurrence below) are
    // formed once, by warp 0 while it waits for the cluster's partials, and
    // broadcast with the sums: the other warps skip the two reciprocal
    // sequences (same operations on the same values: bitwise)
    uint32_t phv = par ? ph0 : ph1;   // buffer par ^ 1
    csum(v4, std::integral_constant<int, 3>{}, std::integral_constant<int, NVL>{}, par ^ 1, phv, [&] {
      if (lane == 0) {
        s.bcast[3] = 1.0 / alpha;
        s.bcast[4] = 1.0 / gamma;
      }
    });
    if (par) ph0 = phv; else ph1 = phv;
    ralpha = s.bcast[3];
    rgamma = s.bcast[4];
    if (sub) A.timing[73] = clock64();
    ++k;
    if (stamp && k < 60) A.timing[4 + k] = clock64();
    rho = v4[2];
    if (rho <= thr) break;
    const double gn = v4[0];
    beta = __dmul_rn(gn, rgamma);   // one division on the critical path
    alpha = gn / __dsub_rn(v4[1], __dmul_rn(beta, __dmul_rn(gn, ralpha)));
    gamma = gn;
    if (sub) A.timing[74] = clock64();
  }
  if (own) A.x[(size_t)e0 * P1 + L] = x;
  if (stamp) { A.timing[64] = clock64(); A.timing[65] = k; }
  if (rank == 0 && threadIdx.x == 0) {
    int idx = atomicAdd(&A.status[2], 1);
    if (idx < A.log_cap) {
      A.log_it[idx] = ok ? k : -1;
      A.log_margin[idx] = thr > 0.0 ? sqrt(rho / thr) : 0.0;
    }
    if (!ok) atomicAdd(&A.status[1], 1);
  }
}

// Partition: one thread per node, at most 384 nodes per CTA and 16 CTAs (one cluster).
// Returns -1 when the level needs more: the caller falls back to the grid mode.
static int choose_partition(const Ctx* c, int ne, int p1, int& K, int& E) {
  int want = c->cluster_ctas > 0 ? c->cluster_ctas : (ne * p1 + 287) / 288;   // ~288 nodes per CTA
  K = want < 1 ? 1 : (want > 16 ? 16 : want);
  if (K > ne) K = ne;
  for (;;) {
    E = (ne + K - 1) / K;
    K = (ne + E - 1) / E;   // no empty CTA
    if (E * p1 <= 384 || K >= 16 || K >= ne) break;
    ++K;
  }
  return E * p1 <= 384 ? 0 : -1;
}

// resident blocks of the non-cluster instantiation (grid mode: cooperative launch)
template <int P1, bool DIR>
static int cg_grid_capacity(Ctx* c, int threads, size_t smem, int* cap) {
  int per_sm = 0, sms = 0;
  cudaError_t e = cudaFuncSetAttribute(k_cg1d<false, P1, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg1d<false, P1, DIR>, threads, smem);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  if (e != cudaSuccess) return c->cuda(e, "cg1d grid occupancy");
  *cap = per_sm * sms;
  return SISDC_OK;
}

template <int P1, bool DIR>
static int launch_cg_t(Ctx* c, CgArgs& A, int threads, size_t smem) {
  static bool attr_done[2] = {false, false};
  if (A.gws != nullptr) {   // grid mode: K > 16 blocks of a cooperative launch
    int cap = 0;
    if (int rc = cg_grid_capacity<P1, DIR>(c, threads, smem, &cap)) return rc;
    if (A.K > cap || A.K > CG1G_MAXK)
      return c->fail(SISDC_ERR_UNSUPPORTED, "implicit_solve: level too large for the grid-mode CG (" +
                                                std::to_string(A.K) + " blocks of 384 nodes, " +
                                                std::to_string(cap < CG1G_MAXK ? cap : CG1G_MAXK) + " resident)");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(A.K);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cg1d<false, P1, DIR>, A);
    if (e != cudaSuccess) return c->cuda(e, "cg1d grid-mode launch");
    return c->after_launch("cg1d (grid mode)");
  }
  if (A.K == 1) {
    if (!attr_done[0]) {
      cudaFuncSetAttribute(k_cg1d<false, P1, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_done[0] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = c->pdl;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cg1d<false, P1, DIR>, A);
    if (e != cudaSuccess) return c->cuda(e, "cg1d launch");
    return c->after_launch("cg1d");
  }
  if (!attr_done[1]) {
    cudaFuncSetAttribute(k_cg1d<true, P1, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_cg1d<true, P1, DIR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_done[1] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(A.K);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = A.K;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlap launch + prologue with the predecessor
  at[1].val.programmaticStreamSerializationAllowed = c->pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_cg1d<true, P1, DIR>, A);
  if (e != cudaSuccess) return c->cuda(e, "cg1d cluster launch");
  return c->after_launch("cg1d");
}

int launch_cg1d(Ctx* c, const Op1DDev& op, CoefDev k, double a, const double* rhs, double* x,
                const StageFuse* sf) {
  const int p1 = op.p1;
  int K, E;
  bool grid_mode = false;
  if (choose_partition(c, op.ne, p1, K, E)) {
    // beyond one cluster (16 CTAs x 384 nodes): the same kernel in grid mode, ~384 nodes per block
    E = 384 / p1;
    K = (op.ne + E - 1) / E;
    E = (op.ne + K - 1) / K;   // balanced, no empty block
    K = (op.ne + E - 1) / E;
    grid_mode = true;
  }
  int threads = ((E * p1 + 31) / 32) * 32;
  if (threads < 64) threads = 64;
  size_t smem = cg_smem_bytes(p1, E, threads);
  CgArgs A{};
  A.op = op; A.coef = k; A.a = a; A.rhs = rhs; A.x = x;
  A.gws = grid_mode ? c->d_cg1g : nullptr;
  if (sf) {
    if (sf->M > MAXM) return c->fail(SISDC_ERR_ARG, "too many collocation nodes");
    A.stage = 1;
    A.sg.base = sf->base; A.sg.conv_in = sf->conv_in; A.sg.f_old = sf->f_old; A.sg.g = sf->g; A.sg.h = sf->h;
    A.sg.conv_out = sf->conv_out; A.sg.dt_m = sf->dt_m; A.sg.dt = sf->dt; A.sg.gl = sf->gl; A.sg.gr = sf->gr;
    A.sg.M = sf->M;
    for (int j = 0; j < sf->M; ++j) A.sg.w[j] = (sf->f_old && sf->w_row) ? sf->w_row[j] : 0.0;
  }
  A.rtol2 = c->rtol * c->rtol; A.maxit = c->maxit; A.E = E; A.K = K;
  A.status = c->d_status; A.log_it = c->d_log_it; A.log_margin = c->d_log_margin; A.log_cap = c->log_cap;
  A.timing = c->d_timing;
  switch (p1) {
    case 2: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<2, true>(c, A, threads, smem) : launch_cg_t<2, false>(c, A, threads, smem);
    case 3: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<3, true>(c, A, threads, smem) : launch_cg_t<3, false>(c, A, threads, smem);
    case 4: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<4, true>(c, A, threads, smem) : launch_cg_t<4, false>(c, A, threads, smem);
    case 5: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<5, true>(c, A, threads, smem) : launch_cg_t<5, false>(c, A, threads, smem);
    case 6: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<6, true>(c, A, threads, smem) : launch_cg_t<6, false>(c, A, threads, smem);
    case 7: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<7, true>(c, A, threads, smem) : launch_cg_t<7, false>(c, A, threads, smem);
    case 8: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<8, true>(c, A, threads, smem) : launch_cg_t<8, false>(c, A, threads, smem);
    case 9: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<9, true>(c, A, threads, smem) : launch_cg_t<9, false>(c, A, threads, smem);
    case 10: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<10, true>(c, A, threads, smem) : launch_cg_t<10, false>(c, A, threads, smem);
    case 11: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<11, true>(c, A, threads, smem) : launch_cg_t<11, false>(c, A, threads, smem);
    case 12: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<12, true>(c, A, threads, smem) : launch_cg_t<12, false>(c, A, threads, smem);
    case 13: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<13, true>(c, A, threads, smem) : launch_cg_t<13, false>(c, A, threads, smem);
    case 14: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<14, true>(c, A, threads, smem) : launch_cg_t<14, false>(c, A, threads, smem);
    case 15: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<15, true>(c, A, threads, smem) : launch_cg_t<15, false>(c, A, threads, smem);
    case 16: return A.op.bc == SISDC_DIRICHLET ? launch_cg_t<16, true>(c, A, threads, smem) : launch_cg_t<16, false>(c, A, threads, smem);
    default: return c->fail(SISDC_ERR_UNSUPPORTED, "degree outside 1..15");
  }
}

}  // namespace sisdc
