// Internal definitions of the opaque ABI handles, shared by abi.cu and
// part2d.cu (element-row partitioned 2-D operators).
#pragma once
#include <vector>
#include "sisdc_dev.cuh"
#include "sisdc_dev2d.cuh"
#include "sisdc_host.h"

struct sisdc_ctx {
  sisdc::Ctx c;
};

struct sisdc_comm;   // NCCL communicator (part2d.cu)
constexpr int HALO_MAXVEC = 17;   // node vectors of one packed halo exchange (M + 1 <= 17)

// one element-row partition of a 2-D operator (ghost-row storage)
struct Part2D {
  sisdc::Op2DDev dev;
  long long off = 0;    // offset of the partition in a state vector of the operator
  long long offc = 0;   // offset in a scalar (coefficient) field
  int row_begin = 0;    // first owned global element row
  int rank = 0;         // global rank that owns it
  double* ws = nullptr; // split-CG workspace (cg2p_ws_doubles)
  int G = 0;            // blocks of the split-CG kernels
};

struct sisdc_op1d {   // dimension-tagged operator handle (1-D or 2-D)
  sisdc_ctx* ctx;
  int dim = 1;
  sisdc_op1d_desc desc;
  sisdc::Op1DDev dev;
  sisdc::Op2DDev dev2;
  double* d_tab = nullptr;
  double* d_cgws = nullptr;   // 2-D CG workspace (allocated at creation: graph-safe)
  int cg_blocks = 0;
  std::vector<double> nodes, weights, D;
  std::vector<double> btab;    // Dirichlet trace table: (t, g_l, g_r) triples
  // partitioned 2-D operator (empty parts: single periodic domain)
  std::vector<Part2D> parts;
  sisdc_comm* comm = nullptr;  // NULL: every partition is local (in-process)
  int nranks = 1;
  long long n_total = 0, nn_total = 0;
  double* d_red = nullptr;           // [0..3] local partial sums, [4..7] allreduced sums
  sisdc::CgPScal* d_sc = nullptr;
  int* h_done = nullptr;             // pinned [2]
  cudaEvent_t ev[2] = {nullptr, nullptr};
  // halo / interior overlap of the fused split iteration: the halo and the two ghost-row bands run on
  // halo_stream while the interior bands run on the operator's stream (fork / join by events)
  cudaStream_t halo_stream = nullptr;
  double* d_hsend = nullptr;         // packed NCCL halo: [2 sides][HALO_MAXVEC][nc][row] send / receive buffers
  double* d_hrecv = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool parted() const { return !parts.empty(); }
  long long n() const { return dim == 1 ? (long long)dev.n * dev.nc : (parted() ? n_total : dev2.n); }
  bool cns() const { return dim == 1 && dev.problem == SISDC_CNS1D; }
  double* d_pinv = nullptr;   // 1-D CNS: element-block Jacobi inverses (n_elem x (3(P+1))^2)
  double* d_c9 = nullptr;     // 1-D CNS: materialised 3x3 coefficient per node (n x 9)
  double* d_cws = nullptr;    // 1-D CNS: [zero vector | D(0; t)] (2 x 3n), Dirichlet solves
};

struct sisdc_xfer {
  sisdc_ctx* ctx;
  int dim = 1;
  sisdc::XferDev dev;
  sisdc::Xfer2Dev dev2;
  double* d_tab = nullptr;
};

inline sisdc::Ctx* C(sisdc_op1d* op) { return &op->ctx->c; }
inline sisdc::CoefDev coef(sisdc_coef k) { return sisdc::CoefDev{k.kind, k.value, k.ptr}; }

// 2-D operator creation (abi.cu); alloc_cg = false skips the cooperative-CG workspace
int op2d_create_impl(sisdc_ctx* x, const sisdc_op2d_desc* d, bool alloc_cg, sisdc_op1d** out);
void part2_destroy(sisdc_op1d* op);
// partitioned OperatorContext entry points (part2d.cu)
int part2_conv(sisdc_op1d* op, const double* u, double* out);
int part2_sip(sisdc_op1d* op, sisdc::CoefDev k, const double* u, double* out);
int part2_coef_field(sisdc_op1d* op, sisdc::CoefDev k, double* out);
int part2_eval_nodes(sisdc_op1d* op, int mode, int scheme, int M, int m_first, int m_count, const double* u0,
                     const double* u, const double* conv_prev, const double* dts, double* f, double* h1, double* h2);
int part2_stage(sisdc_op1d* op, const double* base, const double* conv_in, double dt_m, const double* f_old, int M,
                const double* w_row, double dt, const double* g, const double* h, double* rhs, double* conv_out);
int part2_solve(sisdc_op1d* op, sisdc::CoefDev k, double a, const double* rhs, double* x);
// ghost rows of a per-element scalar (nys x nex per partition, partitions concatenated): the artificial viscosity
int part2_halo_elem(sisdc_op1d* op, double* v);
