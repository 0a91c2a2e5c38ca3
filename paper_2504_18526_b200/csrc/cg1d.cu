// Cluster-resident Jacobi-PCG for the implicit substep (M + a B[C]) x = M rhs.
//
// Replaces the reference's SuperLU solve + defect iteration
// (dgsem.py:492-533) by the pinned PCG of oracle/cg.py.  The whole solve runs
// in ONE launch: a thread-block cluster of K <= 16 CTAs (one per SM) owns the
// elements in contiguous blocks, every CG vector lives in shared memory, the
// face halo of the search direction is read from the neighbour CTA through
// distributed shared memory, and the dot products are reduced by pushing
// per-CTA partials into every CTA's shared memory followed by one hardware
// cluster barrier.  Two cluster barriers per iteration:
//   A: p.Ap          B: (r.z, r.r)
// The neighbour's new search direction is recomputed from its z and previous
// p with the same fused multiply-add the owner uses (bitwise identical), so no
// third barrier is needed after the p update.  All reductions run in a fixed
// order, identical in every CTA: the iteration is deterministic.
#include <cooperative_groups.h>
#include <climits>
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

struct CgSmem {
  double *st, *X, *R, *Z, *AP, *Pb[2], *DG, *C, *Q, *H, *slotA, *slotB, *wscr, *bc;
};

__device__ __forceinline__ CgSmem carve(double* sm, int p1, int E) {
  CgSmem s;
  const int NL = E * p1;
  s.st = sm;
  double* q = sm + TabOff::size(p1);
  s.X = q; q += NL;
  s.R = q; q += NL;
  s.Z = q; q += NL;
  s.AP = q; q += NL;
  s.Pb[0] = q; q += NL;
  s.Pb[1] = q; q += NL;
  s.DG = q; q += NL;
  s.C = q; q += NL + 2;   // + C at left-halo node P, right-halo node 0
  s.Q = q; q += NL;
  s.H = q; q += 4;        // halo: pL, qL, pR, qR
  s.slotA = q; q += 16 * 4;
  s.slotB = q; q += 16 * 4;
  s.wscr = q; q += 32 * 4;
  s.bc = q; q += 8;
  return s;
}
static size_t cg_smem_bytes(int p1, int E) { return sizeof(double) * (TabOff::size(p1) + 9 * E * p1 + 2 + 4 + 128 + 128 + 8); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum NV values over the whole cluster (or CTA); identical bits in every CTA.
template <int NV, bool CL>
__device__ __forceinline__ void cluster_sum(double (&v)[NV], const CgSmem& s, double* slots, int K, int rank) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) s.wscr[wid * 4 + j] = v[j];
  __syncthreads();
  if (wid == 0) {
    double t[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) t[j] = warp_sum(lane < nw ? s.wscr[lane * 4 + j] : 0.0);
    if constexpr (CL) {
      if (lane < K) {
        double* dst = cg::this_cluster().map_shared_rank(slots, lane);
#pragma unroll
        for (int j = 0; j < NV; ++j) dst[rank * 4 + j] = t[j];
      }
    } else {
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) s.bc[j] = t[j];
    }
  }
  if constexpr (CL) {
    cg::this_cluster().sync();
    if (wid == 0) {
      double t[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) t[j] = warp_sum(lane < K ? slots[lane * 4 + j] : 0.0);
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) s.bc[j] = t[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = s.bc[j];
}

template <bool CL>
__device__ __forceinline__ double* remote(double* p, int r) {
  if constexpr (CL) return cg::this_cluster().map_shared_rank(p, r);
  else return p;
}

// Fetch the halo element values of the search direction into s.H and compute
// the neighbour face fluxes q.  mode 0: value = src0 (direct);
// mode 1: value = fma(beta, src1, src0) (neighbour's p_{k} from z_k, p_{k-1}).
template <bool CL>
__device__ __forceinline__ void halo_fetch(const CgArgs& A, const CgSmem& s, int rank, int e0, int e1,
                                           double* own0, double* own1, int mode, double beta) {
  const Op1DDev& op = A.op;
  const int p1 = op.p1, P = p1 - 1;
  const double* D = s.st + TabOff::D(p1);
  int side = (int)threadIdx.x - ((int)blockDim.x - 2);   // last two threads
  if (side < 0) return;
  int eg = side == 0 ? wrap(e0 - 1, op.ne) : wrap(e1, op.ne);
  int r = eg / A.E, el = eg - r * A.E;
  const double* s0 = remote<CL>(own0, r) + el * p1;
  const double* s1 = mode ? remote<CL>(own1, r) + el * p1 : nullptr;
  int row = side == 0 ? P : 0;   // face node of the neighbour element
  double g = 0.0, pf = 0.0;
  for (int j = 0; j < p1; ++j) {
    double pj = mode ? fma(beta, s1[j], s0[j]) : s0[j];
    g = fma(D[row * p1 + j], pj, g);
    if (j == row) pf = pj;
  }
  double cf = s.C[A.E * p1 + side];
  s.H[2 * side] = pf;
  s.H[2 * side + 1] = cf * (op.s * g);
}

// Ap = m p + a B[C] p on own nodes; returns the thread's partial p.Ap
__device__ __forceinline__ double matvec(const CgArgs& A, const CgSmem& s, const double* pv, int nl) {
  const Op1DDev& op = A.op;
  const int p1 = op.p1, P = p1 - 1, NL = A.E * p1;
  const double* D = s.st + TabOff::D(p1);
  const double* DTW = s.st + TabOff::DTW(p1);
  const double* ms = s.st + TabOff::m(p1);
  for (int L = threadIdx.x; L < nl; L += blockDim.x) {
    int el = L / p1, i = L - el * p1;
    const double* pe = pv + el * p1;
    double g = 0.0;
#pragma unroll 4
    for (int j = 0; j < p1; ++j) g = fma(D[i * p1 + j], pe[j], g);
    s.Q[L] = s.C[L] * (op.s * g);
  }
  __syncthreads();
  double part = 0.0;
  for (int L = threadIdx.x; L < nl; L += blockDim.x) {
    int el = L / p1, i = L - el * p1, b = el * p1;
    double B = 0.0;
#pragma unroll 4
    for (int k = 0; k < p1; ++k) B = fma(DTW[i * p1 + k], s.Q[b + k], B);
    const bool last = (b + p1 >= nl), first = (b == 0);
    double pn = last ? s.H[2] : pv[b + p1], qn = last ? s.H[3] : s.Q[b + p1], cn = last ? s.C[NL + 1] : s.C[b + p1];
    double pp = first ? s.H[0] : pv[b - 1], qp = first ? s.H[1] : s.Q[b - 1], cp = first ? s.C[NL] : s.C[b - 1];
    double jr = pv[b + P] - pn;
    double jl = pp - pv[b];
    if (i == P) B += -(0.5 * (s.Q[b + P] + qn)) + (op.mu0 * (0.5 * (s.C[b + P] + cn))) * jr;
    if (i == 0) B -= -(0.5 * (qp + s.Q[b])) + (op.mu0 * (0.5 * (cp + s.C[b]))) * jl;
    B -= (op.s * ((0.5 * s.C[b + P]) * jr)) * D[P * p1 + i];
    B -= (op.s * ((0.5 * s.C[b]) * jl)) * D[i];
    double ap = fma(A.a, B, ms[i] * pv[L]);
    s.AP[L] = ap;
    part = fma(pv[L], ap, part);
  }
  return part;
}

template <bool CL>
__global__ void __launch_bounds__(1024) k_cg1d(CgArgs A) {
  extern __shared__ double sm[];
  const Op1DDev& op = A.op;
  const int p1 = op.p1, P = p1 - 1;
  int rank = 0;
  if constexpr (CL) rank = (int)cg::this_cluster().block_rank();
  const CgSmem s = carve(sm, p1, A.E);
  const int e0 = rank * A.E;
  const int e1 = min(op.ne, e0 + A.E);
  const int nl = (e1 - e0) * p1, NL = A.E * p1;
  load_tab(s.st, op.tab, p1);
  __syncthreads();
  const double* ms = s.st + TabOff::m(p1);
  const double* D = s.st + TabOff::D(p1);
  const double* D2W = s.st + TabOff::D2W(p1);
  // ---- setup: x0 = rhs, coefficient, Jacobi diagonal, zero p_{-1}
  for (int L = threadIdx.x; L < NL; L += blockDim.x) {
    int el = L / p1, i = L - el * p1;
    bool own = L < nl;
    s.X[L] = own ? A.rhs[(size_t)e0 * p1 + L] : 0.0;
    s.C[L] = own ? coef_at(op, A.coef, e0 + el, i) : 0.0;
    s.Pb[1][L] = 0.0;
  }
  if (threadIdx.x == 0) s.C[NL] = coef_at(op, A.coef, wrap(e0 - 1, op.ne), P);
  if (threadIdx.x == 1) s.C[NL + 1] = coef_at(op, A.coef, wrap(e1, op.ne), 0);
  __syncthreads();
  for (int L = threadIdx.x; L < nl; L += blockDim.x) {
    int el = L / p1, i = L - el * p1, b = el * p1;
    double d = 0.0;
#pragma unroll 4
    for (int k = 0; k < p1; ++k) d = fma(D2W[i * p1 + k], s.C[b + k], d);
    d = op.s * d;
    if (i == P) {
      double cn = (b + p1 >= nl) ? s.C[NL + 1] : s.C[b + p1];
      d += op.mu0 * (0.5 * (s.C[b + P] + cn)) - op.s * s.C[b + P] * D[P * p1 + P];
    }
    if (i == 0) {
      double cp = (b == 0) ? s.C[NL] : s.C[b - 1];
      d += op.mu0 * (0.5 * (cp + s.C[b])) + op.s * s.C[b] * D[0];
    }
    s.DG[L] = ms[i] + A.a * d;
  }
  if constexpr (CL) cg::this_cluster().sync(); else __syncthreads();
  // r = b - A x0 (halo of x0 read directly: stable after the barrier)
  halo_fetch<CL>(A, s, rank, e0, e1, s.X, nullptr, 0, 0.0);
  __syncthreads();
  matvec(A, s, s.X, nl);
  double v4[4] = {0.0, 0.0, 0.0, 0.0};
  for (int L = threadIdx.x; L < nl; L += blockDim.x) {
    int i = L % p1;
    double b = ms[i] * A.rhs[(size_t)e0 * p1 + L];
    double r = b - s.AP[L];
    double z = r / s.DG[L];
    s.R[L] = r;
    s.Z[L] = z;
    s.Pb[0][L] = z;   // p_0 = fma(0, p_{-1} = 0, z_0)
    v4[0] = fma(r, z, v4[0]);
    v4[1] = fma(r, r, v4[1]);
    v4[2] = fma(b, b, v4[2]);
    v4[3] += (b != 0.0) ? 1.0 : 0.0;
  }
  cluster_sum<4, CL>(v4, s, s.slotB, A.K, rank);
  double rz = v4[0], rr = v4[1];
  const double thr = A.rtol2 * v4[2];
  if (v4[3] == 0.0) {   // b == 0 -> zeros (dgsem.py:510-511)
    for (int L = threadIdx.x; L < nl; L += blockDim.x) A.x[(size_t)e0 * p1 + L] = 0.0;
    if constexpr (CL) cg::this_cluster().sync();
    return;
  }
  int k = 0;
  double beta = 0.0;
  bool ok = true;
  while (rr > thr) {
    if (k >= A.maxit) { ok = false; break; }
    double* pc = s.Pb[k & 1];
    double* po = s.Pb[(k + 1) & 1];
    // halo p_k of the neighbours = fma(beta_{k-1}, p_{k-1}, z_k)
    halo_fetch<CL>(A, s, rank, e0, e1, s.Z, po, 1, beta);
    double v1[1] = {matvec(A, s, pc, nl)};
    cluster_sum<1, CL>(v1, s, s.slotA, A.K, rank);
    const double alpha = rz / v1[0];
    double v2[2] = {0.0, 0.0};
    for (int L = threadIdx.x; L < nl; L += blockDim.x) {
      double p = pc[L];
      s.X[L] = fma(alpha, p, s.X[L]);
      double r = fma(-alpha, s.AP[L], s.R[L]);
      double z = r / s.DG[L];
      s.R[L] = r;
      s.Z[L] = z;
      v2[0] = fma(r, z, v2[0]);
      v2[1] = fma(r, r, v2[1]);
    }
    cluster_sum<2, CL>(v2, s, s.slotB, A.K, rank);
    beta = v2[0] / rz;
    rz = v2[0];
    rr = v2[1];
    ++k;
    if (rr <= thr) break;
    for (int L = threadIdx.x; L < nl; L += blockDim.x) po[L] = fma(beta, pc[L], s.Z[L]);
    __syncthreads();
  }
  for (int L = threadIdx.x; L < nl; L += blockDim.x) A.x[(size_t)e0 * p1 + L] = s.X[L];
  if (rank == 0 && threadIdx.x == 0) {
    int idx = atomicAdd(&A.status[2], 1);
    if (idx < A.log_cap) {
      A.log_it[idx] = ok ? k : -1;
      A.log_margin[idx] = thr > 0.0 ? sqrt(rr / thr) : 0.0;
    }
    if (!ok) atomicAdd(&A.status[1], 1);
  }
  // keep every CTA's shared memory alive until remote readers are done
  if constexpr (CL) cg::this_cluster().sync();
}

// Cluster size: about 576 nodes per CTA (one thread per node), at most 16
// CTAs (non-portable cluster), enough CTAs for the vectors to fit in 200 KB.
static void choose_partition(const Ctx* c, int ne, int p1, int& K, int& E) {
  K = c->cluster_ctas > 0 ? c->cluster_ctas : (ne * p1 + 575) / 576;
  K = K < 1 ? 1 : (K > 16 ? 16 : K);
  if (K > ne) K = ne;
  for (;;) {
    E = (ne + K - 1) / K;
    K = (ne + E - 1) / E;   // no empty CTA
    if (cg_smem_bytes(p1, E) <= 200 * 1024 || K >= 16 || K >= ne) break;
    ++K;
  }
}

int launch_cg1d(Ctx* c, const Op1DDev& op, CoefDev k, double a, const double* rhs, double* x) {
  const int p1 = op.p1;
  int K, E;
  choose_partition(c, op.ne, p1, K, E);
  size_t smem = cg_smem_bytes(p1, E);
  if (smem > 227 * 1024)
    return c->fail(SISDC_ERR_UNSUPPORTED, "implicit_solve: level too large for the cluster-resident CG "
                                          "(n_elem*(P+1) beyond 16 CTAs of shared memory)");
  CgArgs A{};
  A.op = op; A.coef = k; A.a = a; A.rhs = rhs; A.x = x;
  A.rtol2 = c->rtol * c->rtol; A.maxit = c->maxit; A.E = E; A.K = K;
  A.status = c->d_status; A.log_it = c->d_log_it; A.log_margin = c->d_log_margin; A.log_cap = c->log_cap;
  int threads = E * p1;
  threads = threads > 1024 ? 1024 : ((threads + 31) / 32) * 32;
  if (threads < 64) threads = 64;
  if (K == 1) {
    cudaError_t e = cudaFuncSetAttribute(k_cg1d<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return c->cuda(e, "cg1d smem attribute");
    k_cg1d<false><<<1, threads, smem, c->stream>>>(A);
    return c->after_launch("cg1d");
  }
  cudaError_t e = cudaFuncSetAttribute(k_cg1d<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return c->cuda(e, "cg1d smem attribute");
  e = cudaFuncSetAttribute(k_cg1d<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return c->cuda(e, "cg1d cluster attribute");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(K);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = K;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k_cg1d<true>, A);
  if (e != cudaSuccess) return c->cuda(e, "cg1d cluster launch");
  return c->after_launch("cg1d");
}

}  // namespace sisdc
