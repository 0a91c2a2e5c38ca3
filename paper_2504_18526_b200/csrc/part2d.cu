// Element-row partitioned 2-D operators (BASELINE configs 4-5 across GPUs).
//
// The global nex x ney mesh is cut into contiguous blocks of element rows, one
// per rank.  A partition stores its rows with one ghost row on
// each side, (ncomp, rows + 2, nex, P+1, P+1); the 2-D kernels read y-neighbours
// of their boundary rows from the ghost rows (Op2DDev::row0 / ynb), so every
// kernel is unchanged except for addressing.  Before a face-coupled operator
// runs, the ghost rows of its face-coupled inputs are refreshed by the halo
// exchange:
//   * ranks on different GPUs: NCCL send/recv of the boundary rows (one
//     contiguous nex*(P+1)^2 run per field and side) inside one NCCL group on
//     the operator's stream, so it orders with the kernels and needs no host
//     synchronisation;
//   * partitions driven by one process (the single-GPU emulation of R ranks,
//     and the 1-rank case): one copy kernel over all local partitions.
// The implicit solve is the split Chronopoulos-Gear PCG (ops2d.cu k2p_*): per
// iteration phase A, halo(u), phase B, a fixed-order reduction, one NCCL
// allreduce of three doubles, and the scalar recurrences on the device.  The
// host polls the convergence flag one batch behind the launches; inside a
// CUDA-graph capture a fixed-length batch is recorded instead (kernels return
// at once after convergence), so partitioned slabs replay as graphs too.
// Elementwise work (defects, transfers, copies) runs over the concatenated
// storage of the local partitions unchanged.
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <new>
#include <nccl.h>
#include "abi_internal.h"

using namespace sisdc;

// ------------------------------------------------------------------ NCCL
// resolved at run time from the libnccl.so.2 already loaded by the host
// process (torch), so the library itself links without NCCL
namespace {
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*groupStart)();
  ncclResult_t (*groupEnd)();
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*errorString)(ncclResult_t);
  bool ok = false;
};

NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.ok ? &api : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
#define SISDC_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); if (!api.field) return nullptr;
  SISDC_SYM(getUniqueId, "ncclGetUniqueId");
  SISDC_SYM(commInitRank, "ncclCommInitRank");
  SISDC_SYM(commDestroy, "ncclCommDestroy");
  SISDC_SYM(groupStart, "ncclGroupStart");
  SISDC_SYM(groupEnd, "ncclGroupEnd");
  SISDC_SYM(send, "ncclSend");
  SISDC_SYM(recv, "ncclRecv");
  SISDC_SYM(allReduce, "ncclAllReduce");
  SISDC_SYM(errorString, "ncclGetErrorString");
#undef SISDC_SYM
  api.ok = true;
  return &api;
}
}  // namespace

struct sisdc_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

namespace {

int nccl_fail(Ctx* c, ncclResult_t r, const char* what) {
  NcclApi* api = nccl();
  return c->fail(SISDC_ERR_CUDA, std::string(what) + ": " + (api ? api->errorString(r) : "NCCL unavailable"));
}

// rows of global rank q when ney rows are split over nranks
void rank_rows(int ney, int nranks, int q, int* begin, int* count) {
  const int base = ney / nranks, rem = ney % nranks;
  *count = base + (q < rem ? 1 : 0);
  *begin = q * base + (q < rem ? q : rem);
}

// refresh the ghost rows of mcount node vectors (stride mstride) of a state
// (nc = ncomp, scalar = false) or of a scalar field (nc = 1, scalar = true)
int halo(sisdc_op1d* op, const double* vec_c, int mcount, long long mstride, bool scalar) {
  Ctx* c = C(op);
  double* vec = const_cast<double*>(vec_c);   // ghost rows are scratch of every operator input
  const int nc = scalar ? 1 : op->dev2.nc;
  const int np = (int)op->parts.size();
  if (!op->comm) {
    Op2DDev ops[MAXPART];
    double* base[MAXPART];
    for (int p = 0; p < np; ++p) {
      ops[p] = op->parts[p].dev;
      base[p] = vec + (scalar ? op->parts[p].offc : op->parts[p].off);
    }
    return launch2p_halo(c, np, ops, base, nc, mcount, mstride);
  }
  NcclApi* api = nccl();
  if (!api) return c->fail(SISDC_ERR_UNSUPPORTED, "NCCL is not available in this process");
  const Part2D& P = op->parts[0];
  const int R = op->comm->nranks, q = op->comm->rank;
  const int prev = (q + R - 1) % R, next = (q + 1) % R;
  const size_t row = (size_t)P.dev.nex * P.dev.p1 * P.dev.p1;
  // packed exchange (one contiguous buffer per side: 2 sends + 2 receives) when the rows can be moved
  // with 16-byte copies; per-(vector, field) messages otherwise
  const bool packed = op->d_hsend && mcount <= HALO_MAXVEC && (row & 1) == 0 && (P.dev.nn & 1) == 0 &&
                      (mstride & 1) == 0 && (reinterpret_cast<uintptr_t>(vec) & 15) == 0;
  if (packed) {
    const size_t cnt = (size_t)mcount * nc * row;   // one side
    if (int rc = launch2p_halo_pack(c, P.dev, vec, op->d_hsend, nc, mcount, mstride, 0)) return rc;
    // first owned rows -> prev (its top ghost rows), last owned rows -> next (its bottom ghost rows); the
    // k-th send to a peer pairs with its k-th receive from us (1 rank: self; 2 ranks: prev == next)
    ncclResult_t r = api->groupStart();
    if (r == ncclSuccess) r = api->send(op->d_hsend, cnt, ncclDouble, prev, op->comm->comm, c->stream);
    if (r == ncclSuccess) r = api->send(op->d_hsend + cnt, cnt, ncclDouble, next, op->comm->comm, c->stream);
    if (r == ncclSuccess) r = api->recv(op->d_hrecv, cnt, ncclDouble, next, op->comm->comm, c->stream);
    if (r == ncclSuccess) r = api->recv(op->d_hrecv + cnt, cnt, ncclDouble, prev, op->comm->comm, c->stream);
    const ncclResult_t r2 = api->groupEnd();
    if (r != ncclSuccess) return nccl_fail(c, r, "halo send/recv");
    if (r2 != ncclSuccess) return nccl_fail(c, r2, "halo group");
    ++c->launches;
    return launch2p_halo_pack(c, P.dev, vec, op->d_hrecv, nc, mcount, mstride, 1);
  }
  ncclResult_t r = api->groupStart();
  for (int m = 0; m < mcount && r == ncclSuccess; ++m)
    for (int f = 0; f < nc && r == ncclSuccess; ++f) {
      double* b = vec + m * mstride + f * P.dev.nn;
      // first owned row -> prev's top ghost; last owned row -> next's bottom ghost.  Issue order =
      // dgsem2d.halo_schedule (NCCL pairs the k-th send to a peer with its k-th receive from us;
      // correct for 1 rank (self), 2 ranks (prev == next) and more), tested over gloo on CPU
      r = api->send(b + row, row, ncclDouble, prev, op->comm->comm, c->stream);
      if (r == ncclSuccess) r = api->send(b + (size_t)P.dev.ney * row, row, ncclDouble, next, op->comm->comm, c->stream);
      if (r == ncclSuccess) r = api->recv(b + (size_t)(P.dev.ney + 1) * row, row, ncclDouble, next, op->comm->comm, c->stream);
      if (r == ncclSuccess) r = api->recv(b, row, ncclDouble, prev, op->comm->comm, c->stream);
    }
  const ncclResult_t r2 = api->groupEnd();
  if (r != ncclSuccess) return nccl_fail(c, r, "halo send/recv");
  if (r2 != ncclSuccess) return nccl_fail(c, r2, "halo group");
  ++c->launches;
  return SISDC_OK;
}

int halo_coef(sisdc_op1d* op, const CoefDev& k) {
  if (k.kind == SISDC_COEF_SI) return halo(op, k.ptr, 1, 0, false);
  if (k.kind == SISDC_COEF_FIELD) return halo(op, k.ptr, 1, 0, true);
  return SISDC_OK;
}

CoefDev coef_part(const CoefDev& k, const Part2D& P) {
  CoefDev r = k;
  if (k.kind == SISDC_COEF_SI) r.ptr = k.ptr + P.off;
  if (k.kind == SISDC_COEF_FIELD) r.ptr = k.ptr + P.offc;
  return r;
}

inline const double* at(const double* p, long long o) { return p ? p + o : nullptr; }
inline double* at(double* p, long long o) { return p ? p + o : nullptr; }

}  // namespace

// ghost rows of a per-element scalar field (one value per element: the frozen artificial viscosity).
// The element "nodes" are 1 x 1, so the exchange runs on copies of the partition descriptors with
// p1 = 1 (row = nex values, field stride = nys * nex).
int part2_halo_elem(sisdc_op1d* op, double* v) {
  Ctx* c = C(op);
  const int np = (int)op->parts.size();
  Op2DDev ops[MAXPART];
  double* base[MAXPART];
  long long offe = 0;
  for (int p = 0; p < np; ++p) {
    ops[p] = op->parts[p].dev;
    ops[p].p1 = 1;
    ops[p].nn = (long long)ops[p].nys * ops[p].nex;
    base[p] = v + offe;
    offe += ops[p].nn;
  }
  if (!op->comm) return launch2p_halo(c, np, ops, base, 1, 1, 0);
  NcclApi* api = nccl();
  if (!api) return c->fail(SISDC_ERR_UNSUPPORTED, "NCCL is not available in this process");
  const int R = op->comm->nranks, q = op->comm->rank;
  const int prev = (q + R - 1) % R, next = (q + 1) % R;
  const size_t row = (size_t)ops[0].nex;
  double* b = base[0];
  ncclResult_t r = api->groupStart();
  if (r == ncclSuccess) r = api->send(b + row, row, ncclDouble, prev, op->comm->comm, c->stream);
  if (r == ncclSuccess) r = api->send(b + (size_t)ops[0].ney * row, row, ncclDouble, next, op->comm->comm, c->stream);
  if (r == ncclSuccess) r = api->recv(b + (size_t)(ops[0].ney + 1) * row, row, ncclDouble, next, op->comm->comm, c->stream);
  if (r == ncclSuccess) r = api->recv(b, row, ncclDouble, prev, op->comm->comm, c->stream);
  const ncclResult_t r2 = api->groupEnd();
  if (r != ncclSuccess) return nccl_fail(c, r, "nu_art halo send/recv");
  if (r2 != ncclSuccess) return nccl_fail(c, r2, "nu_art halo group");
  ++c->launches;
  return SISDC_OK;
}

// ------------------------------------------------------ entry points
int part2_conv(sisdc_op1d* op, const double* u, double* out) {
  if (int rc = halo(op, u, 1, 0, false)) return rc;
  for (const Part2D& P : op->parts)
    if (int rc = launch2_conv(C(op), P.dev, u + P.off, out + P.off)) return rc;
  return SISDC_OK;
}

int part2_sip(sisdc_op1d* op, CoefDev k, const double* u, double* out) {
  if (int rc = halo(op, u, 1, 0, false)) return rc;
  if (int rc = halo_coef(op, k)) return rc;
  for (const Part2D& P : op->parts)
    if (int rc = launch2_sip(C(op), P.dev, coef_part(k, P), u + P.off, out + P.off)) return rc;
  return SISDC_OK;
}

int part2_coef_field(sisdc_op1d* op, CoefDev k, double* out) {
  if (int rc = halo_coef(op, k)) return rc;
  for (const Part2D& P : op->parts)
    if (int rc = launch2_coef(C(op), P.dev, coef_part(k, P), out + P.offc)) return rc;
  return SISDC_OK;
}

int part2_eval_nodes(sisdc_op1d* op, int mode, int scheme, int M, int m_first, int m_count, const double* u0,
                     const double* u, const double* conv_prev, const double* dts, double* f, double* h1, double* h2) {
  if (M > 16 || m_first < 0 || m_count < 1 || m_first + m_count > M) return C(op)->fail(SISDC_ERR_ARG, "bad node range");
  const long long ns = op->n_total;
  // u_m for the evaluated nodes and u_{m-1} (SI coefficient, conv of the previous node)
  if (mode != 0) {
    if (m_first == 0) {
      if (int rc = halo(op, u0, 1, 0, false)) return rc;
      if (int rc = halo(op, u, m_count, ns, false)) return rc;
    } else if (int rc = halo(op, u + (m_first - 1) * ns, m_count + 1, ns, false)) {
      return rc;
    }
  } else if (int rc = halo(op, u + m_first * ns, m_count, ns, false)) {
    return rc;
  }
  for (const Part2D& P : op->parts)
    if (int rc = launch2_node_eval(C(op), P.dev, mode, scheme, M, m_first, m_count, u0 + P.off, u + P.off,
                                   at(conv_prev, P.off), dts, f + P.off, at(h1, P.off), at(h2, P.off)))
      return rc;
  return SISDC_OK;
}

int part2_stage(sisdc_op1d* op, const double* base, const double* conv_in, double dt_m, const double* f_old, int M,
                const double* w_row, double dt, const double* g, const double* h, double* rhs, double* conv_out) {
  if (int rc = halo(op, conv_in, 1, 0, false)) return rc;
  for (const Part2D& P : op->parts)
    if (int rc = launch2_stage(C(op), P.dev, base + P.off, conv_in + P.off, dt_m, at(f_old, P.off), M, w_row, dt,
                               at(g, P.off), at(h, P.off), rhs + P.off, at(conv_out, P.off)))
      return rc;
  return SISDC_OK;
}

namespace {
// sums of the local partitions (fixed order) -> allreduced sums at d_red + 4
int reduce_all(sisdc_op1d* op, int mode, int fsetup = 0) {
  Ctx* c = C(op);
  const int np = (int)op->parts.size();
  Op2DDev ops[MAXPART];
  double* ws[MAXPART];
  for (int p = 0; p < np; ++p) {
    ops[p] = op->parts[p].dev;
    ws[p] = op->parts[p].ws;
  }
  if (!op->comm) return launch2p_reduce(c, np, ws, ops, op->parts[0].G, mode, op->d_red + 4, fsetup);
  if (int rc = launch2p_reduce(c, np, ws, ops, op->parts[0].G, mode, op->d_red, fsetup)) return rc;
  NcclApi* api = nccl();
  if (!api) return c->fail(SISDC_ERR_UNSUPPORTED, "NCCL is not available in this process");
  const ncclResult_t r = api->allReduce(op->d_red, op->d_red + 4, 3, ncclDouble, ncclSum, op->comm->comm, c->stream);
  if (r != ncclSuccess) return nccl_fail(c, r, "CG allreduce");
  ++c->launches;
  return SISDC_OK;
}

// ucur: which u buffer holds this iteration's u (the other the previous one); -1 setup
int phase_all(sisdc_op1d* op, int phase, const CoefDev& k, double a, const double* rhs, double* x, int ucur = -1) {
  for (const Part2D& P : op->parts)
    if (int rc = launch2p_phase(C(op), phase, P.dev, coef_part(k, P), a, rhs + P.off, x + P.off, P.ws, P.G, op->d_sc,
                                ucur))
      return rc;
  return SISDC_OK;
}

int halo_u(sisdc_op1d* op, int which) {
  Ctx* c = C(op);
  const int np = (int)op->parts.size();
  if (!op->comm) {
    Op2DDev ops[MAXPART];
    double* base[MAXPART];
    for (int p = 0; p < np; ++p) {
      ops[p] = op->parts[p].dev;
      base[p] = cg2p_U(ops[p], op->parts[p].ws, which);
    }
    return launch2p_halo(c, np, ops, base, ops[0].nc, 1, 0);
  }
  // one local partition: its workspace u has the storage layout of a state
  const Part2D& P = op->parts[0];
  return halo(op, cg2p_U(P.dev, P.ws, which) - P.off, 1, 0, false);
}

// ghost rows of CG workspace vectors of every local partition: the (r, s, w) triple of parity par
// (three consecutive state-sized vectors: one halo call) or, dinv = true, the Jacobi reciprocal (one
// field).  Partitions differ in size, so bases and strides are per partition (mstride -1).
int halo_ws(sisdc_op1d* op, bool dinv, int par, int nvec = 3) {
  Ctx* c = C(op);
  const int np = (int)op->parts.size();
  auto vec = [&](const Part2D& P) { return dinv ? P.ws + cg2p_dinv_off(P.dev) : cg2p_RSW(P.dev, P.ws, par); };
  if (!op->comm) {
    Op2DDev ops[MAXPART];
    double* base[MAXPART];
    for (int p = 0; p < np; ++p) {
      ops[p] = op->parts[p].dev;
      base[p] = vec(op->parts[p]);
    }
    return launch2p_halo(c, np, ops, base, dinv ? 1 : ops[0].nc, dinv ? 1 : nvec, -1);
  }
  const Part2D& P = op->parts[0];   // one local partition: halo() adds P.off / P.offc back
  return halo(op, vec(P) - (dinv ? P.offc : P.off), dinv ? 1 : nvec, P.dev.n, dinv);
}

// fused iteration j (P = 7): the (r, s, w) of parity j & 1 get their ghost rows, then ONE pass per
// partition does update + matvec (k2_cgf single-pass mode) and writes parity (j + 1) & 1.
// Overlap (partitions of >= 3 bands driven through a communicator; SISDC_PART_OVERLAP, below): only the first and the last band
// of a partition read ghost rows, so the halo exchange and those two bands run on the operator's second
// stream while the interior bands run on the main stream; the two launches split the partition's G
// blocks (and block-partial slots) in proportion to their work and are co-resident.  Fork after the
// previous iteration's scalar kernel, join before the reduction.
struct StreamSwap {   // launch on another stream for a scope (Ctx is single-threaded)
  Ctx* c;
  cudaStream_t saved;
  StreamSwap(Ctx* c_, cudaStream_t s) : c(c_), saved(c_->stream) { c->stream = s; }
  ~StreamSwap() { c->stream = saved; }
};

// SISDC_PART_OVERLAP: 1 always, 0 never; unset: only with a communicator of more than one rank.  On ONE
// GPU there is no transfer to hide and the two co-resident launches cost ~8% (cfg4 fine solve 8.07 ->
// 8.74 ms, in-process partition; 442 -> 494 ms per eager cfg4 step through one NCCL rank), so single-GPU
// runs keep the single launch unless asked.
int overlap_mode() {
  const char* v = getenv("SISDC_PART_OVERLAP");   // read per solve: tests toggle it
  return !v ? -1 : v[0] == '0' ? 0 : 1;
}

int iterate_fused(sisdc_op1d* op, int j, const CoefDev& k, double a, const double* rhs, double* x) {
  Ctx* c = C(op);
  const int par = j & 1;
  const int om = overlap_mode();
  bool split = (om == 1 || (om < 0 && op->comm != nullptr && op->nranks > 1)) && op->halo_stream != nullptr;
  for (const Part2D& P : op->parts) split = split && cg2p_bands(P.dev) >= 3 && P.G >= 8;
  if (!split) {
    if (int rc = halo_ws(op, false, par)) return rc;
    for (const Part2D& P : op->parts)
      if (int rc = launch2p_fpass(c, P.dev, coef_part(k, P), a, rhs + P.off, x + P.off, P.ws, P.G, op->d_sc, par))
        return rc;
  } else {
    cudaError_t e = cudaEventRecord(op->ev_fork, c->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(op->halo_stream, op->ev_fork, 0);
    if (e != cudaSuccess) return c->cuda(e, "halo fork");
    auto edge_blocks = [](const Part2D& P) {   // the edge launch's share of the G blocks: 2 of nb bands
      const int nb = cg2p_bands(P.dev);
      int ge = (5 * P.G + nb) / (2 * nb);   // 1.25 x its share: it starts late by the halo's latency
      return ge < 1 ? 1 : ge > P.G - 1 ? P.G - 1 : ge;
    };
    {
      StreamSwap sw(c, op->halo_stream);
      if (int rc = halo_ws(op, false, par)) return rc;
      for (const Part2D& P : op->parts) {
        const int ge = edge_blocks(P);
        if (int rc = launch2p_fpass(c, P.dev, coef_part(k, P), a, rhs + P.off, x + P.off, P.ws, P.G, op->d_sc, par, 2,
                                    P.G - ge, ge))
          return rc;
      }
    }
    e = cudaEventRecord(op->ev_join, op->halo_stream);
    if (e != cudaSuccess) return c->cuda(e, "halo join");
    for (const Part2D& P : op->parts)
      if (int rc = launch2p_fpass(c, P.dev, coef_part(k, P), a, rhs + P.off, x + P.off, P.ws, P.G, op->d_sc, par, 1, 0,
                                  P.G - edge_blocks(P)))
        return rc;
    e = cudaStreamWaitEvent(c->stream, op->ev_join, 0);
    if (e != cudaSuccess) return c->cuda(e, "halo join");
  }
  if (int rc = reduce_all(op, 1)) return rc;
  return launch2p_scalar(c, 2, op->d_red + 4, op->d_sc);
}

// iteration j: u_prev in buffer j & 1 (the setup's u0 in buffer 0), u_new in the other
int iterate(sisdc_op1d* op, int j, const CoefDev& k, double a, const double* rhs, double* x) {
  if (cg2p_fused(op->parts[0].dev)) return iterate_fused(op, j, k, a, rhs, x);
  const int ucur = (j + 1) & 1;
  if (int rc = phase_all(op, P2_UPDATE, k, a, rhs, x, ucur)) return rc;
  if (int rc = halo_u(op, ucur)) return rc;
  if (int rc = phase_all(op, P2_MATVEC, k, a, rhs, x, ucur)) return rc;
  if (int rc = reduce_all(op, 1)) return rc;
  return launch2p_scalar(C(op), 2, op->d_red + 4, op->d_sc);
}
}  // namespace

int part2_solve(sisdc_op1d* op, CoefDev k, double a, const double* rhs, double* x) {
  Ctx* c = C(op);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cap);
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(rhs)) & 15))
    return c->fail(SISDC_ERR_ARG, "2-D implicit solve: rhs and x must be 16-byte aligned");
  // coefficient source and rhs (x0 = rhs feeds the first matvec)
  if (int rc = halo_coef(op, k)) return rc;
  if (int rc = halo(op, rhs, 1, 0, false)) return rc;
  if (int rc = phase_all(op, P2_INIT, k, a, rhs, x)) return rc;
  if (int rc = phase_all(op, P2_DINV, k, a, rhs, x)) return rc;
  if (cg2p_fused(op->parts[0].dev))   // the fused pass rebuilds the neighbour rows' u = r dinv: dinv ghost rows, once
    if (int rc = halo_ws(op, true, 0)) return rc;
  // fused levels: the two setup matvecs as single passes of the fused pipeline (k2_cgf MODE 1 / 2; u0 = r0 dinv
  // is rebuilt on chip, so only r0's ghost rows travel); SISDC_PART_FSETUP=0 keeps the split kernels (A/B)
  const char* fsv = getenv("SISDC_PART_FSETUP");
  const bool fsetup = cg2p_fused(op->parts[0].dev) && !(fsv && fsv[0] == '0');
  if (fsetup) {
    for (const Part2D& P : op->parts)
      if (int rc = launch2p_fsetup(c, 1, P.dev, coef_part(k, P), a, rhs + P.off, x + P.off, P.ws, P.G, op->d_sc)) return rc;
    if (int rc = reduce_all(op, 0, 1)) return rc;
    if (int rc = launch2p_scalar(c, 0, op->d_red + 4, op->d_sc)) return rc;
    if (int rc = halo_ws(op, false, 0, 1)) return rc;   // r0
    for (const Part2D& P : op->parts)
      if (int rc = launch2p_fsetup(c, 2, P.dev, coef_part(k, P), a, rhs + P.off, x + P.off, P.ws, P.G, op->d_sc)) return rc;
    if (int rc = reduce_all(op, 2)) return rc;
    if (int rc = launch2p_scalar(c, 1, op->d_red + 4, op->d_sc)) return rc;
  } else {
    if (int rc = phase_all(op, P2_RESID, k, a, rhs, x)) return rc;
    if (int rc = reduce_all(op, 0)) return rc;
    if (int rc = launch2p_scalar(c, 0, op->d_red + 4, op->d_sc)) return rc;
    if (int rc = phase_all(op, P2_U0, k, a, rhs, x)) return rc;
    if (int rc = halo_u(op, 0)) return rc;
    if (int rc = phase_all(op, P2_MATVEC, k, a, rhs, x)) return rc;
    if (int rc = reduce_all(op, 1)) return rc;
    if (int rc = launch2p_scalar(c, 1, op->d_red + 4, op->d_sc)) return rc;
  }
  if (capturing) {
    // inside a CUDA-graph capture the host cannot poll: a fixed number of iterations is recorded (kernels
    // after convergence return at once: device-side convergence), and the closing scalar kernel latches a
    // failure if the batch was too short (SISDC_PART_CAPTURE_ITERS, default 32; cfg4 / cfg5 solves take 6-25)
    static const int cap_iters = [] {
      const char* v = getenv("SISDC_PART_CAPTURE_ITERS");
      const int n = v ? atoi(v) : 32;
      return n > 0 ? n : 32;
    }();
    for (int j = 0; j < cap_iters; ++j)
      if (int rc = iterate(op, j, k, a, rhs, x)) return rc;
    return launch2p_scalar(c, 3, op->d_red + 4, op->d_sc);
  }
  // iterations in batches of B; the flag of batch j-1 is read while batch j runs
  constexpr int B = 2;
  const int max_batches = c->maxit / B + 3;
  for (int j = 0; j < max_batches; ++j) {
    for (int i = 0; i < B; ++i)
      if (int rc = iterate(op, j * B + i, k, a, rhs, x)) return rc;
    cudaError_t e = cudaMemcpyAsync(op->h_done + (j & 1), &op->d_sc->done, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaEventRecord(op->ev[j & 1], c->stream);
    if (e != cudaSuccess) return c->cuda(e, "CG convergence flag");
    if (j > 0) {
      e = cudaEventSynchronize(op->ev[(j - 1) & 1]);
      if (e != cudaSuccess) return c->cuda(e, "CG convergence flag");
      if (op->h_done[(j - 1) & 1]) return SISDC_OK;
    }
  }
  cudaError_t e = cudaEventSynchronize(op->ev[(max_batches - 1) & 1]);
  if (e != cudaSuccess) return c->cuda(e, "CG convergence flag");
  return SISDC_OK;   // the scalar kernel latched the failure (status[1]) at maxit
}

void part2_destroy(sisdc_op1d* op) {
  for (Part2D& P : op->parts) cudaFree(P.ws);
  op->parts.clear();
  cudaFree(op->d_red);
  cudaFree(op->d_sc);
  if (op->h_done) cudaFreeHost(op->h_done);
  for (cudaEvent_t& e : op->ev)
    if (e) cudaEventDestroy(e);
  if (op->ev_fork) cudaEventDestroy(op->ev_fork);
  if (op->ev_join) cudaEventDestroy(op->ev_join);
  if (op->halo_stream) cudaStreamDestroy(op->halo_stream);
  cudaFree(op->d_hsend);
  cudaFree(op->d_hrecv);
}

// ------------------------------------------------------------------ ABI
extern "C" {

int sisdc_nccl_unique_id(unsigned char* id) {
  if (!id) return SISDC_ERR_ARG;
  NcclApi* api = nccl();
  if (!api) return SISDC_ERR_UNSUPPORTED;
  ncclUniqueId u;
  if (api->getUniqueId(&u) != ncclSuccess) return SISDC_ERR_CUDA;
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return SISDC_OK;
}

int sisdc_comm_create(sisdc_ctx* x, const unsigned char* id, int nranks, int rank, sisdc_comm** out) {
  if (!x || !id || !out || nranks < 1 || rank < 0 || rank >= nranks) return SISDC_ERR_ARG;
  *out = nullptr;
  NcclApi* api = nccl();
  if (!api) return x->c.fail(SISDC_ERR_UNSUPPORTED, "NCCL is not available in this process");
  sisdc_comm* cm = new (std::nothrow) sisdc_comm();
  if (!cm) return SISDC_ERR_ARG;
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  cudaSetDevice(x->c.device);
  const ncclResult_t r = api->commInitRank(&cm->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete cm;
    return nccl_fail(&x->c, r, "ncclCommInitRank");
  }
  cm->nranks = nranks;
  cm->rank = rank;
  *out = cm;
  return SISDC_OK;
}

void sisdc_comm_destroy(sisdc_comm* cm) {
  if (!cm) return;
  NcclApi* api = nccl();
  if (api && cm->comm) api->commDestroy(cm->comm);
  delete cm;
}

int sisdc_op2d_create_part(sisdc_ctx* x, const sisdc_op2d_desc* d, int nranks, int first_rank, int nlocal,
                           sisdc_comm* comm, sisdc_op1d** out) {
  if (!x || !d || !out) return SISDC_ERR_ARG;
  *out = nullptr;
  Ctx& c = x->c;
  if (nranks < 1 || nlocal < 1 || nlocal > MAXPART || first_rank < 0 || first_rank + nlocal > nranks)
    return c.fail(SISDC_ERR_ARG, "bad partition counts");
  if (nranks > d->ney) return c.fail(SISDC_ERR_ARG, "more ranks than element rows");
  if (comm && (comm->nranks != nranks || comm->rank != first_rank || nlocal != 1))
    return c.fail(SISDC_ERR_ARG, "an NCCL communicator drives exactly one local partition (its own rank)");
  if (!comm && nlocal != nranks) return c.fail(SISDC_ERR_ARG, "without a communicator every partition must be local");
  sisdc_op1d* op = nullptr;
  if (int rc = op2d_create_impl(x, d, false, &op)) return rc;
  op->comm = comm;
  op->nranks = nranks;
  Op2DDev& g = op->dev2;
  // P = 3 partitions iterate with the fused 2 x 2-tile pass when every rank's block has an even number of
  // element rows and nex is even (the same decision on every rank: rank_rows is deterministic)
  g.fused_sub2 = g.p1 == 4 && d->nex % 2 == 0 ? 1 : 0;
  for (int q = 0; q < nranks && g.fused_sub2; ++q) {
    int rb = 0, rcnt = 0;
    rank_rows(d->ney, nranks, q, &rb, &rcnt);
    if (rcnt % 2 != 0) g.fused_sub2 = 0;
  }
  const long long nnod = (long long)g.p1 * g.p1;
  long long off = 0, offc = 0;
  for (int l = 0; l < nlocal; ++l) {
    Part2D P;
    P.rank = first_rank + l;
    int rb = 0, rcnt = 0;
    rank_rows(d->ney, nranks, P.rank, &rb, &rcnt);
    P.row_begin = rb;
    P.dev = g;
    P.dev.ney = rcnt;
    P.dev.nys = rcnt + 2;
    P.dev.row0 = 1;
    P.dev.e0 = (long long)rb * g.nex;
    P.dev.nn = (long long)P.dev.nys * g.nex * nnod;
    P.dev.n = P.dev.nn * g.nc;
    P.off = off;
    P.offc = offc;
    off += P.dev.n;
    offc += P.dev.nn;
    op->parts.push_back(P);
  }
  op->n_total = off;
  op->nn_total = offc;
  cudaError_t e = cudaSuccess;
  for (Part2D& P : op->parts) {
    P.dev.ns = off;
    int rc = cg2p_blocks(&c, P.dev, &P.G);
    if (rc) { sisdc_op1d_destroy(op); return rc; }
  }
  // one block count for all partitions (the reduction walks G slots of each)
  int G = op->parts[0].G;
  for (const Part2D& P : op->parts) G = P.G < G ? P.G : G;
  for (Part2D& P : op->parts) {
    P.G = G;
    if (e == cudaSuccess) e = cudaMalloc(&P.ws, cg2p_ws_doubles(P.dev, G) * sizeof(double));
  }
  if (e == cudaSuccess) e = cudaMalloc(&op->d_red, 8 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&op->d_sc, sizeof(CgPScal));
  if (e == cudaSuccess) e = cudaMemset(op->d_sc, 0, sizeof(CgPScal));
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&op->h_done), 2 * sizeof(int), cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&op->ev[0], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&op->ev[1], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&op->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&op->halo_stream, cudaStreamNonBlocking);
  if (comm) {   // packed NCCL halo buffers (both sides of up to HALO_MAXVEC node vectors)
    const size_t hb = 2 * (size_t)HALO_MAXVEC * g.nc * g.nex * nnod * sizeof(double);
    if (e == cudaSuccess) e = cudaMalloc(&op->d_hsend, hb);
    if (e == cudaSuccess) e = cudaMalloc(&op->d_hrecv, hb);
  }
  if (e != cudaSuccess) {
    const int rc = c.cuda(e, "partition workspace");
    sisdc_op1d_destroy(op);
    return rc;
  }
  *out = op;
  return SISDC_OK;
}

int sisdc_op2d_part_layout(const sisdc_op1d* op, int cap, int* row_begin, int* row_count, int64_t* offset,
                           int* nparts) {
  if (!op || !nparts) return SISDC_ERR_ARG;
  *nparts = (int)op->parts.size();
  for (int p = 0; p < *nparts && p < cap; ++p) {
    if (row_begin) row_begin[p] = op->parts[p].row_begin;
    if (row_count) row_count[p] = op->parts[p].dev.ney;
    if (offset) offset[p] = op->parts[p].off;
  }
  return SISDC_OK;
}

int sisdc_halo_exchange(sisdc_op1d* op, double* vec, int mcount, int64_t mstride, int scalar_field) {
  if (!op || !vec || mcount < 1) return SISDC_ERR_ARG;
  if (!op->parted()) return C(op)->fail(SISDC_ERR_ARG, "not a partitioned operator");
  return halo(op, vec, mcount, mstride, scalar_field != 0);
}

}  // extern "C"
