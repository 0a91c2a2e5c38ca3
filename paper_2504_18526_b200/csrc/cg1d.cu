// Cluster-resident Jacobi-PCG for the implicit substep (M + a B[C]) x = M rhs.
//
// Replaces the reference's SuperLU solve + defect iteration
// (dgsem.py:492-533) by the pinned PCG of oracle/cg.py.  The whole solve runs
// in ONE launch: a thread-block cluster of K <= 16 CTAs (one per SM) owns the
// elements in contiguous blocks, one thread per node.  The iterate x, the
// residual r, the Jacobi diagonal and the node's operator rows live in
// registers; the search direction p and the element fluxes q live in shared
// memory.
//
// Inter-CTA traffic is push-only and barrier-free (sm_90+/sm_100a DSMEM):
//  * dot products: every warp shuffle-reduces its partial and writes it with
//    st.async into a slot of every CTA of the cluster; the store completes a
//    transaction count on the RECEIVER's mbarrier.  A CTA waits on its own
//    mbarrier until all K*nw partials have landed, then every warp sums the
//    slots in one fixed order -> bitwise-identical totals everywhere.
//  * face halo: the boundary element's (p_k, z_{k+1}) are pushed with the
//    r.z partials; the receiver forms p_{k+1} = fma(beta_k, p_k, z_{k+1})
//    exactly as the owner does.
// No cluster barrier (and no release fence waiting on remote stores) sits on
// the iteration's critical path: two mbarrier waits per iteration.
#include <cooperative_groups.h>
#include <type_traits>
#include "sisdc_dev.cuh"
#include "sisdc_host.h"

namespace cg = cooperative_groups;

namespace sisdc {

struct CgArgs {
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

template <int P1>
struct CgShared {
  double* st;
  double* Pb[2];
  double* Q;
  double* Cs;    // own nodes + [NL] = C(left halo, node P), [NL+1] = C(right halo, node 0)
  double* HX;    // halo x0 [2][P1]
  double* HPZ;   // halo (p_k, z_{k+1}) pairs [2][P1][2]
  double* HP;    // halo p_k values formed locally [2][P1]
  double* slotA;
  double* slotB;
  double* wpart;              // per-warp partials [32][4]
  unsigned long long* mbar;   // [0] A, [1] B, [2] X
};

template <int P1>
__device__ __forceinline__ CgShared<P1> carve(double* sm, int E, int K, int nw) {
  CgShared<P1> s;
  const int NL = E * P1;
  double* q = sm;
  s.mbar = reinterpret_cast<unsigned long long*>(q); q += 4;
  s.st = q; q += TabOff::size(P1);
  s.Pb[0] = q; q += NL;
  s.Pb[1] = q; q += NL;
  s.Q = q; q += NL;
  s.Cs = q; q += NL + 2;
  s.HX = q; q += 2 * P1;
  q += (q - sm) & 1;   // 16-byte alignment for v2 stores
  s.HPZ = q; q += 4 * P1;
  s.HP = q; q += 2 * P1;
  s.slotB = q; q += 16 * 4;   // 16-byte aligned: receives v2 stores, [rank][NV]
  s.slotA = q; q += 16;
  s.wpart = q; q += 32 * 4;
  return s;
}
static size_t cg_smem_bytes(int p1, int E, int K, int nw) {
  return sizeof(double) * (4 + TabOff::size(p1) + 4 * E * p1 + 2 + 2 * p1 + 1 + 4 * p1 + 2 * p1 + 64 + 16 + 128);
}

template <bool CL, int P1>
__global__ void __launch_bounds__(512) k_cg1d(CgArgs A) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = P1 - 1;
  const Op1DDev& op = A.op;
  int rank = 0;
  if constexpr (CL) rank = (int)cg::this_cluster().block_rank();
  const int nw = (blockDim.x + 31) >> 5;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const CgShared<P1> s = carve<P1>(sm, A.E, A.K, nw);
  const int K = A.K;
  const int e0 = rank * A.E;
  const int e1 = min(op.ne, e0 + A.E);
  const int nl = (e1 - e0) * P1, NL = A.E * P1;
  const int L = threadIdx.x, el = L / P1, i = L - el * P1;
  const bool own = L < nl;
  const bool first = el == 0, last = (el + 1) * P1 >= nl;
  const int egL = wrap(e0 - 1, op.ne), egR = wrap(e1, op.ne);
  const int rL = egL / A.E, rR = egR / A.E;
  const uint32_t mA = sa(&s.mbar[0]), mB = sa(&s.mbar[1]), mX = sa(&s.mbar[2]);
  if (threadIdx.x == 0) {
    mbar_init(mA);
    mbar_init(mB);
    mbar_init(mX);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = threadIdx.x; t < TabOff::size(P1); t += blockDim.x) s.st[t] = op.tab[t];
  double ci = 0.0, rhs = 0.0;
  if (own) {
    ci = coef_at(op, A.coef, e0 + el, i);
    rhs = A.rhs[(size_t)e0 * P1 + L];
    s.Cs[L] = ci;
    s.Pb[1][L] = rhs;
  }
  if (L == 0) s.Cs[NL] = coef_at(op, A.coef, egL, P);
  if (L == 1) s.Cs[NL + 1] = coef_at(op, A.coef, egR, 0);
  if constexpr (CL) cg::this_cluster().sync();   // mbarriers initialised cluster-wide
  else __syncthreads();
  // remote addresses this thread pushes to
  // boundary element threads: first element -> left neighbour's right halo, last -> right neighbour's left halo
  const bool pushL = own && first, pushR = own && last;
  uint32_t hxL = 0, hxR = 0, hpzL = 0, hpzR = 0, mBL = 0, mBR = 0, mXL = 0, mXR = 0;
  if constexpr (CL) {
    if (pushL) {
      hxL = mapa(sa(s.HX + P1 + i), rL);
      hpzL = mapa(sa(s.HPZ + 2 * (P1 + i)), rL);
      mBL = mapa(mB, rL);
      mXL = mapa(mX, rL);
    }
    if (pushR) {
      hxR = mapa(sa(s.HX + i), rR);
      hpzR = mapa(sa(s.HPZ + 2 * i), rR);
      mBR = mapa(mB, rR);
      mXR = mapa(mX, rR);
    }
  }
  uint32_t phA = 0, phB = 0;
  const uint32_t halo_bytes = 2u * P1 * 16u;
  // remote slot / mbarrier addresses for warp 0's lanes (lane r pushes to CTA r)
  uint32_t raA = 0, raB2 = 0, raB4 = 0, rmA = 0, rmB = 0;
  if constexpr (CL) {
    if (wid == 0 && lane < K) {
      raA = mapa(sa(s.slotA + rank), lane);
      raB2 = mapa(sa(s.slotB + 2 * rank), lane);
      raB4 = mapa(sa(s.slotB + 4 * rank), lane);
      rmA = mapa(mA, lane);
      rmB = mapa(mB, lane);
    }
  }

  // Cluster sum of NV values: warp shuffles, CTA pre-reduction by warp 0, one
  // st.async per (CTA, destination CTA) completing on the receiver's mbarrier,
  // then every warp sums the K slots in rank order (identical bits everywhere).
  auto csum = [&](auto& v, auto nv_tag, bool useA) {
    constexpr int NV = decltype(nv_tag)::value;
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < NV; ++j) s.wpart[wid * 4 + j] = v[j];
    __syncthreads();
    double* slots = useA ? s.slotA : s.slotB;
    if (wid == 0) {
      double t[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) t[j] = warp_sum(lane < nw ? s.wpart[lane * 4 + j] : 0.0);
      if constexpr (CL) {
        if (lane < K) {
          if constexpr (NV == 1) st_async(raA, t[0], rmA);
          else {
            const uint32_t ra = NV == 2 ? raB2 : raB4;
#pragma unroll
            for (int j = 0; j < NV; j += 2) st_async2(ra + 8 * j, t[j], t[j + 1], rmB);
          }
        }
      } else {
        if (lane == 0)
#pragma unroll
          for (int j = 0; j < NV; ++j) slots[j] = t[j];
      }
    }
    if constexpr (CL) {
      const uint32_t mb = useA ? mA : mB;
      if (threadIdx.x == 0) mbar_expect(mb, 8u * K * NV + (useA ? 0u : halo_bytes));
      mbar_wait(mb, useA ? phA : phB);
      if (useA) phA ^= 1; else phB ^= 1;
    } else {
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = warp_sum(lane < K ? slots[lane * NV + j] : 0.0);
  };

  const double* D = s.st + TabOff::D(P1);
  const double* DTW = s.st + TabOff::DTW(P1);
  const double mi = s.st[TabOff::m(P1) + i];
  const double sc = op.s, mu0 = op.mu0, a = A.a;
  const double cR = last ? s.Cs[NL + 1] : s.Cs[min((el + 1) * P1, NL - 1)];
  const double cL = first ? s.Cs[NL] : s.Cs[max(el * P1 - 1, 0)];
  const double cP = s.Cs[min(el * P1 + P, NL - 1)], c0 = s.Cs[min(el * P1, NL - 1)];
  double dg = 1.0;
  if (own) {   // Jacobi diagonal diag(M + a B[C]) (closed form of dgsem.py:414-490)
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < P1; ++k) d = fma(s.st[TabOff::D2W(P1) + i * P1 + k], s.Cs[el * P1 + k], d);
    d = sc * d;
    if (i == P) d += mu0 * (0.5 * (cP + cR)) - sc * cP * D[P * P1 + P];
    if (i == 0) d += mu0 * (0.5 * (cL + c0)) + sc * c0 * D[0];
    dg = mi + a * d;
  }
  const double dinv = 1.0 / dg;   // Jacobi: z = r * dinv
  // per-node face constants of the SIP operator (dgsem.py:290-308)
  const double muR = mu0 * (0.5 * (cP + cR)), muL = mu0 * (0.5 * (cL + c0));
  const double kR = sc * (0.5 * cP), kL = sc * (0.5 * c0);
  const double DPi = D[P * P1 + i], D0i = D[i];

  // A v on own nodes; halo element values of v in hv[0..P1) (left), hv[P1..2P1) (right)
  auto matvec = [&](const double* v, const double* hv) -> double {
    if (own) {
      const double* ve = v + el * P1;
      s.Q[L] = ci * (sc * dot3<P1>(D + i * P1, ve));
    }
    __syncthreads();
    if (!own) return 0.0;
    const int b = el * P1;
    double B = dot3<P1>(DTW + i * P1, s.Q + b);
    const double pn = last ? hv[P1] : v[b + P1];
    const double pp = first ? hv[P] : v[b - 1];
    const double jr = v[b + P] - pn;
    const double jl = pp - v[b];
    if (i == P) {
      const double qn = last ? cR * (sc * dot3<P1>(D, hv + P1)) : s.Q[b + P1];
      B += -(0.5 * (s.Q[b + P] + qn)) + muR * jr;
    }
    if (i == 0) {
      const double qp = first ? cL * (sc * dot3<P1>(D + P * P1, hv)) : s.Q[b - 1];
      B -= -(0.5 * (qp + s.Q[b])) + muL * jl;
    }
    B -= (kR * jr) * DPi;
    B -= (kL * jl) * D0i;
    return fma(a, B, mi * v[L]);
  };

  // ---- r = b - A x0: exchange the x0 halo
  const double* hx;
  if constexpr (CL) {
    if (threadIdx.x == 0) mbar_expect(mX, 2u * P1 * 8u);
    if (pushL) st_async(hxL, rhs, mXL);
    if (pushR) st_async(hxR, rhs, mXR);
    mbar_wait(mX, 0);
    hx = s.HX;
  } else {
    // single CTA, periodic: halo elements are this CTA's last / first element
    if (L < 2 * P1) {
      const int side = L / P1, j = L - side * P1;
      s.HX[L] = s.Pb[1][(side ? 0 : (nl - P1)) + j];
    }
    __syncthreads();
    hx = s.HX;
  }
  double x = rhs;
  const double ax = matvec(s.Pb[1], hx);
  const double b = mi * rhs;
  double r = b - ax;
  double z = r * dinv;
  if (own) s.Pb[0][L] = z;   // p_0 = z_0 = fma(0, p_{-1} = 0, z_0)
  // halo push (p_{-1} = 0, z_0) with the setup reduction
  auto push_halo = [&](double pk, double zk) {
    if constexpr (CL) {
      if (pushL) st_async2(hpzL, pk, zk, mBL);
      if (pushR) st_async2(hpzR, pk, zk, mBR);
    } else {
      if (L < nl && (first || last)) {
        // local halo: my first element is my own right halo, last element my left halo
        if (first) { s.HPZ[2 * (P1 + i)] = pk; s.HPZ[2 * (P1 + i) + 1] = zk; }
        if (last) { s.HPZ[2 * i] = pk; s.HPZ[2 * i + 1] = zk; }
      }
    }
  };
  push_halo(0.0, z);
  double v4[4] = {own ? r * z : 0.0, own ? r * r : 0.0, own ? b * b : 0.0, (own && b != 0.0) ? 1.0 : 0.0};
  csum(v4, std::integral_constant<int, 4>{}, false);
  double rz = v4[0], rr = v4[1];
  const double thr = A.rtol2 * v4[2];
  if (v4[3] == 0.0) {   // b == 0 -> zeros (dgsem.py:510-511)
    if (own) A.x[(size_t)e0 * P1 + L] = 0.0;
    return;
  }
  int k = 0;
  double beta = 0.0;
  bool ok = true;
  while (rr > thr) {
    if (k >= A.maxit) { ok = false; break; }
    double* pc = s.Pb[k & 1];
    double* po = s.Pb[(k + 1) & 1];
    // neighbour p_k = fma(beta_{k-1}, p_{k-1}, z_k) from the pushed pairs
    if (L < 2 * P1) s.HP[L] = fma(beta, s.HPZ[2 * L], s.HPZ[2 * L + 1]);
    // (matvec's first __syncthreads orders HP before its use)
    const double ap = matvec(pc, s.HP);
    const double pk = own ? pc[L] : 0.0;
    double v1[1] = {pk * ap};
    csum(v1, std::integral_constant<int, 1>{}, true);
    const double alpha = rz / v1[0];
    x = fma(alpha, pk, x);
    r = fma(-alpha, ap, r);
    z = r * dinv;
    push_halo(pk, z);
    double v2[2] = {own ? r * z : 0.0, own ? r * r : 0.0};
    csum(v2, std::integral_constant<int, 2>{}, false);
    beta = v2[0] / rz;
    rz = v2[0];
    rr = v2[1];
    ++k;
    if (rr <= thr) break;
    if (own) po[L] = fma(beta, pk, z);
    __syncthreads();
  }
  if (own) A.x[(size_t)e0 * P1 + L] = x;
  if (rank == 0 && threadIdx.x == 0) {
    int idx = atomicAdd(&A.status[2], 1);
    if (idx < A.log_cap) {
      A.log_it[idx] = ok ? k : -1;
      A.log_margin[idx] = thr > 0.0 ? sqrt(rr / thr) : 0.0;
    }
    if (!ok) atomicAdd(&A.status[1], 1);
  }
}

// Partition: one thread per node, at most 512 nodes per CTA and 16 CTAs.
static int choose_partition(const Ctx* c, int ne, int p1, int& K, int& E) {
  int want = c->cluster_ctas > 0 ? c->cluster_ctas : (ne * p1 + 287) / 288;   // ~288 nodes per CTA
  K = want < 1 ? 1 : (want > 16 ? 16 : want);
  if (K > ne) K = ne;
  for (;;) {
    E = (ne + K - 1) / K;
    K = (ne + E - 1) / E;   // no empty CTA
    if (E * p1 <= 512 || K >= 16 || K >= ne) break;
    ++K;
  }
  return E * p1 <= 512 ? 0 : -1;
}

template <int P1>
static int launch_cg_t(Ctx* c, CgArgs& A, int threads, size_t smem) {
  static bool attr_done[2] = {false, false};
  if (A.K == 1) {
    if (!attr_done[0]) {
      cudaFuncSetAttribute(k_cg1d<false, P1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_done[0] = true;
    }
    k_cg1d<false, P1><<<1, threads, smem, c->stream>>>(A);
    return c->after_launch("cg1d");
  }
  if (!attr_done[1]) {
    cudaFuncSetAttribute(k_cg1d<true, P1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_cg1d<true, P1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_done[1] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(A.K);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = A.K;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_cg1d<true, P1>, A);
  if (e != cudaSuccess) return c->cuda(e, "cg1d cluster launch");
  return c->after_launch("cg1d");
}

int launch_cg1d(Ctx* c, const Op1DDev& op, CoefDev k, double a, const double* rhs, double* x) {
  const int p1 = op.p1;
  int K, E;
  if (choose_partition(c, op.ne, p1, K, E))
    return c->fail(SISDC_ERR_UNSUPPORTED, "implicit_solve: level too large for the cluster-resident CG "
                                          "(more than 16 CTAs x 512 nodes)");
  int threads = ((E * p1 + 31) / 32) * 32;
  if (threads < 64) threads = 64;
  const int nw = threads / 32;
  size_t smem = cg_smem_bytes(p1, E, K, nw);
  CgArgs A{};
  A.op = op; A.coef = k; A.a = a; A.rhs = rhs; A.x = x;
  A.rtol2 = c->rtol * c->rtol; A.maxit = c->maxit; A.E = E; A.K = K;
  A.status = c->d_status; A.log_it = c->d_log_it; A.log_margin = c->d_log_margin; A.log_cap = c->log_cap;
  switch (p1) {
    case 2: return launch_cg_t<2>(c, A, threads, smem);
    case 3: return launch_cg_t<3>(c, A, threads, smem);
    case 4: return launch_cg_t<4>(c, A, threads, smem);
    case 5: return launch_cg_t<5>(c, A, threads, smem);
    case 6: return launch_cg_t<6>(c, A, threads, smem);
    case 7: return launch_cg_t<7>(c, A, threads, smem);
    case 8: return launch_cg_t<8>(c, A, threads, smem);
    case 9: return launch_cg_t<9>(c, A, threads, smem);
    case 10: return launch_cg_t<10>(c, A, threads, smem);
    case 11: return launch_cg_t<11>(c, A, threads, smem);
    case 12: return launch_cg_t<12>(c, A, threads, smem);
    case 13: return launch_cg_t<13>(c, A, threads, smem);
    case 14: return launch_cg_t<14>(c, A, threads, smem);
    case 15: return launch_cg_t<15>(c, A, threads, smem);
    case 16: return launch_cg_t<16>(c, A, threads, smem);
    default: return c->fail(SISDC_ERR_UNSUPPORTED, "degree outside 1..15");
  }
}

}  // namespace sisdc
