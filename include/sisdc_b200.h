/*
 * sisdc_b200.h -- C ABI of the B200-native SI-MLSDC / DG-SEM sweep path.
 *
 * The reference (arXiv 2504.18526, package `sisdc`, pure Python/numpy) has
 * no native boundary: its hot path is the duck-typed OperatorContext
 * protocol (pkg/src/sisdc/integrators.py:29-60) implemented by
 * DGOperator (pkg/src/sisdc/dgsem.py:117-571) and driven by the sweeper
 * (sdc.py) and the multilevel engine (mlsdc.py, transfer.py).  This header
 * is the boundary a maintainer binds (ctypes in this repo, see
 * INTEGRATION.md): plain pointers, sizes and PODs, no torch types.
 *
 * Conventions
 *  - Every state is a DEVICE pointer to float64 in the reference layout
 *    (ncomp, n_elem, P+1), C order (dgsem.py:12-13); node arrays (M, N).
 *  - All calls are asynchronous and ordered on the context's current
 *    stream (sisdc_ctx_set_stream).  Only the *_read/status calls sync.
 *  - Every export returns SISDC_OK or an error code; the message is in
 *    sisdc_ctx_last_error().  No C++ exception crosses the ABI.
 *  - Device-side failures (non-finite rhs, CG non-convergence) are latched
 *    in device flags and reported by sisdc_ctx_status(), so a whole slab
 *    can run (or be replayed from a CUDA graph) without host syncs.
 */
#ifndef SISDC_B200_H
#define SISDC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SISDC_ABI_VERSION 2

enum sisdc_status {
  SISDC_OK = 0,
  SISDC_ERR_ARG = 1,          /* bad argument (reference: ValueError)            */
  SISDC_ERR_CUDA = 2,         /* CUDA runtime error                              */
  SISDC_ERR_NONFINITE = 3,    /* dgsem.py:348-351 non-finite rhs (SolverError)   */
  SISDC_ERR_NOCONV = 4,       /* dgsem.py:530-533 stalled solve (SolverError)    */
  SISDC_ERR_UNSUPPORTED = 5   /* configuration outside the built path            */
};

enum sisdc_problem {
  SISDC_CONVDIFF = 0, SISDC_BURGERS = 1,        /* 1-D, problems.py:25-82               */
  SISDC_EULER2D = 2,                            /* 2-D Euler (+ isotropic nu Laplacian)  */
  SISDC_ADVECTION2D = 3, SISDC_BURGERS2D = 4,   /* 2-D scalar (cross-dimension checks)   */
  SISDC_CNS1D = 5,                              /* 1-D CompressibleFlow, problems.py:160-240 */
  SISDC_NS2D = 6                                /* 2-D compressible Navier-Stokes: Stokes stress +
                                                   Fourier heat flux (desc nu = eta, prandtl)  */
};
enum sisdc_bc { SISDC_PERIODIC = 0, SISDC_DIRICHLET = 1 };       /* Mesh1D.bc         */
enum sisdc_scheme { SISDC_EULER = 0, SISDC_SI1 = 1, SISDC_SI2 = 2 }; /* integrators.py:26 */

/* Coefficient descriptor: the reference's opaque coefficient object
 * (integrators.py:46-55; kinds dgsem.py:229-239), evaluated on the fly. */
enum sisdc_coef_kind {
  SISDC_COEF_NONE = 0,
  SISDC_COEF_CONST = 1,     /* python float                                      */
  SISDC_COEF_FIELD = 2,     /* (n_elem, P+1) scalar field at ptr                 */
  SISDC_COEF_SI = 3,        /* (value/2) A_c(u_b)^2 + A_d + nu_art, u_b = ptr,
                               value = dt_m (dgsem.py:356-396, scheme si1/si2)    */
  SISDC_COEF_PHYS = 4,      /* physical A_d + nu_art (dgsem.py:313-326); systems:
                               A_d(u_b), u_b = ptr                               */
  SISDC_COEF_MATRIX = 5     /* (n_elem, P+1, ncomp, ncomp) matrix field at ptr
                               (dgsem.py:229-239 kind "matrix"; 1-D CNS only)    */
};
typedef struct { int kind; double value; const double* ptr; } sisdc_coef;

typedef struct sisdc_ctx sisdc_ctx;
typedef struct sisdc_op1d sisdc_op1d;
typedef struct sisdc_xfer sisdc_xfer;

/* Mesh1D (dgsem.py:72-106) + problem (problems.py) + DGOperator options. */
typedef struct {
  int n_elem;
  int degree;        /* P, 1..15                         */
  int ncomp;         /* 1 for the scalar problems         */
  int bc;            /* SISDC_PERIODIC / SISDC_DIRICHLET  */
  int problem;       /* sisdc_problem                     */
  double x_left, x_right;
  double speed;      /* ConvectionDiffusion.speed         */
  double nu;         /* physical viscosity (0 => None)    */
  double penalty;    /* DGOperator penalty_const (2.0)    */
  /* SISDC_CNS1D (ncomp 3, periodic): CompressibleFlow(gamma, R_gas, eta, Pr),
   * problems.py:171-187; the implicit system is non-symmetric, so its solve is
   * the pinned Jacobi-BiCGStab of oracle/cg.py (replaces splu, dgsem.py:503-533) */
  double gamma, eta, prandtl;
} sisdc_op1d_desc;

/* 2-D tensor-product DG-SEM on a uniform periodic nex x ney mesh of
 * [x_left,x_right] x [y_bottom,y_top] (BASELINE configs 3-5; the reference is
 * 1-D only).  State layout (ncomp, ney, nex, P+1 [y], P+1 [x]).  Every
 * operator entry point below accepts a 2-D handle; the SI coefficient is the
 * isotropic (dt_m/2) lambda(u_b)^2 + nu (SISDC_NS2D: + eta/rho_b max(4/3,
 * gamma/Pr)), lambda = |v| + c. */
typedef struct {
  int nex, ney;
  int degree;        /* P, 1..8                                   */
  int ncomp;         /* 4 for Euler/NS, 1 for the scalar problems  */
  int problem;       /* SISDC_EULER2D / SISDC_NS2D / SISDC_ADVECTION2D / SISDC_BURGERS2D */
  double x_left, x_right, y_bottom, y_top;
  double gamma;      /* ideal gas                                  */
  double nu;         /* EULER2D: isotropic kinematic viscosity (0 => Euler);
                        NS2D: dynamic viscosity eta                  */
  double ax, ay;     /* advection velocity (SISDC_ADVECTION2D)     */
  double penalty;    /* SIP penalty constant (2.0)                 */
  double prandtl;    /* NS2D Prandtl number (ABI version 2, appended) */
} sisdc_op2d_desc;

/* ----------------------------------------------------------- context */
int  sisdc_abi_version(void);
/* sizeof of the by-pointer / by-value PODs, for bindings to check their
 * mirrors: 0 sisdc_op1d_desc, 1 sisdc_op2d_desc, 2 sisdc_coef (-1 otherwise) */
int  sisdc_struct_size(int which);
int  sisdc_ctx_create(int device, sisdc_ctx** out);
void sisdc_ctx_destroy(sisdc_ctx* ctx);
const char* sisdc_ctx_last_error(const sisdc_ctx* ctx);
int  sisdc_ctx_set_stream(sisdc_ctx* ctx, void* cuda_stream);
int  sisdc_ctx_synchronize(sisdc_ctx* ctx);
/* CG pins (oracle/cg.py): rtol on ||r||_2 <= rtol ||b||_2, maxit; cluster_ctas
 * = 0 picks the cluster size automatically (1..16). */
int  sisdc_ctx_set_cg(sisdc_ctx* ctx, double rtol, int maxit, int cluster_ctas);
/* Latched device status (syncs): first non-finite element (-1 if none),
 * number of CG failures, number of solves logged since the last reset. */
int  sisdc_ctx_status(sisdc_ctx* ctx, int* nonfinite_elem, int* cg_failures, int* n_solves);
int  sisdc_ctx_reset_status(sisdc_ctx* ctx);          /* failure flags; async, capturable */
int  sisdc_ctx_reset_log(sisdc_ctx* ctx);             /* flags + CG log counter */
/* Copy the per-solve CG log (iterations, ||r||/(rtol||b||)) (syncs). */
int  sisdc_ctx_cg_log(sisdc_ctx* ctx, int cap, int* iters, double* margins, int* n_out);
/* Diagnostics: clock64 stamps of the last implicit solve's CTA 0 (setup
 * milestones [0..3], end of iteration k at [4+k], end [64], iterations [65]);
 * needs SISDC_CG_TIMING=1 in the environment when the context is created. */
int  sisdc_ctx_debug_timing(sisdc_ctx* ctx, long long* out, int cap);
/* Number of kernels this context has launched (host-side counter). */
int64_t sisdc_ctx_launch_count(const sisdc_ctx* ctx);
int  sisdc_copy(sisdc_ctx* ctx, double* dst, const double* src, int64_t n);  /* D2D, async */
/* out = coef4[0] v0 + coef4[1] v1 + coef4[2] v2 + coef4[3] v3 (NULL terms
 * skipped; coef4 host), async: the vector updates of the non-incremental
 * sweep (sdc.py:245-284). */
int  sisdc_lincomb(sisdc_ctx* ctx, int64_t n, const double* coef4, const double* v0, const double* v1,
                   const double* v2, const double* v3, double* out);

/* ------------------------------------------------------ DG operator */
int  sisdc_op1d_create(sisdc_ctx* ctx, const sisdc_op1d_desc* desc, sisdc_op1d** out);
/* 2-D operator: returns the same opaque handle type (dimension-tagged). */
int  sisdc_op2d_create(sisdc_ctx* ctx, const sisdc_op2d_desc* desc, sisdc_op1d** out);
void sisdc_op1d_destroy(sisdc_op1d* op);
/* Host copies of the element tables: GLL nodes/weights (P+1), D ((P+1)^2). */
int  sisdc_op1d_tables(const sisdc_op1d* op, double* nodes, double* weights, double* D);
/* Per-element artificial viscosity nu_art (device, n_elem; partitioned 2-D operators: storage rows,
 * ghost rows included) or NULL (DGOperator.nu_art, frozen per slab by begin_slab, dgsem.py:563-571). */
int  sisdc_op1d_set_nu_art(sisdc_op1d* op, const double* nu_art);
/* Dirichlet trace data (problem.boundary_state(t), dgsem.py:212-216,282-284):
 * register the outside states g_l(t_j), g_r(t_j) for n times (merged into the
 * operator's table); gl, gr are (n, ncomp) row-major (ncomp = 3 for CNS).  Every entry point that takes a time t (or node times)
 * on a Dirichlet operator looks its data up here and fails with
 * SISDC_ERR_ARG for an unregistered time. */
int  sisdc_op1d_set_boundary(sisdc_op1d* op, int n, const double* times, const double* gl, const double* gr);
/* smooth_start (dgsem.py:574-589): out = u with every interior interface's
 * two traces replaced by their mean (the periodic wrap too), for M node vectors;
 * the MLSDC presmoothing hook of the coarse-to-fine solution transfer
 * (mlsdc.py:139-140). */
int  sisdc_smooth_start(sisdc_op1d* op, int M, const double* u, double* out);
/* Persson-Peraire modal sensor (dgsem.py:537-559) -> nu_art (device, n_elem).
 * 2-D operators: the tensor-product generalisation (modes with max(k, l) = P, h = max(dx, dy)), one value
 * per element of the storage ((rows + 2) x nex per partition, ghost rows exchanged here). */
int  sisdc_persson_viscosity(sisdc_op1d* op, const double* u, double kappa_s, double c_s, double* nu_art);

/* OperatorContext methods (integrators.py:37-60, dgsem.py:205-352). */
int  sisdc_apply_convection(sisdc_op1d* op, const double* u, double t, double* out);
int  sisdc_apply_diffusion(sisdc_op1d* op, sisdc_coef c, const double* u, double t, double* out);
int  sisdc_eval_rhs(sisdc_op1d* op, const double* u, double t, double* out);
int  sisdc_coef_field(sisdc_op1d* op, sisdc_coef c, double* out);   /* materialise (n_elem*(P+1)) */
/* (M + a B[C]) x = M rhs by the pinned Jacobi-PCG (replaces splu, dgsem.py:503-533). */
int  sisdc_implicit_solve(sisdc_op1d* op, sisdc_coef c, double a, const double* rhs, double t, double* x);

/* ------------------------------------------ fused sweep-stage kernels */
/* rhs = base + dt*sum_i w_row[i] f_old[i] (+ g_m) + dt_m*conv(conv_in) - h_old
 * (sdc.py:218,231,235,237 and predictor sdc.py:144-151); f_old (M,N) may be
 * NULL (no quadrature), g_m / h_old may be NULL; conv_out (nullable)
 * receives conv(conv_in). */
int  sisdc_stage_rhs(sisdc_op1d* op, const double* base, const double* conv_in, double dt_m,
                     const double* f_old, int M, const double* w_row, double dt,
                     const double* g_m, const double* h_old, double t,
                     double* rhs, double* conv_out);
/* sisdc_stage_rhs followed by sisdc_implicit_solve (coefficient k, shift a,
 * the stage's convection at t_conv, the solve at t_solve): x = S(rhs).  On a
 * 1-D operator the stage is computed inside the CG launch's prologue (one
 * launch per substep half instead of two; same arithmetic); elsewhere it runs
 * as the two calls, with the rhs in rhs_scratch. */
int  sisdc_stage_solve(sisdc_op1d* op, sisdc_coef k, double a, const double* base, const double* conv_in,
                       double dt_m, const double* f_old, int M, const double* w_row, double dt,
                       const double* g_m, const double* h_old, double t_conv, double t_solve,
                       double* rhs_scratch, double* conv_out, double* x);
/* Node caches f, h1, h2 for nodes m_first..m_first+m_count-1 (sdc.py:77-119):
 * f = eval_rhs(u_m); h1 = dt_m (conv(u_{m-1}) + D[C_m] u_m);
 * h2 = dt_m (conv(u_m) + D[C_m] u_m) with C_m the scheme's coefficient frozen
 * at u_{m-1}.  conv_prev (nullable): m_count vectors with the node stride, conv_prev[j] = conv(u_{m_first+j-1})
 * as the stage kernels left it (one batched launch per sweep instead of one per node).
 * dts = the M substep sizes (host).  h2 may be NULL (euler/si1). */
int  sisdc_node_caches(sisdc_op1d* op, int scheme, int M, int m_first, int m_count,
                       const double* u0, const double* u, const double* conv_prev,
                       const double* dts, double t0, const double* times,
                       double* f, double* h1, double* h2);
/* f[m] = eval_rhs(u[m]) for m < M (mlsdc.py:68-77 fresh evaluations). */
int  sisdc_eval_rhs_nodes(sisdc_op1d* op, int M, const double* u, const double* times, double* f);
/* out = u - prev - dt * W f (+ add), prev = (u0, u_0..u_{M-2}); incremental
 * form with W = w_nn, or nonincremental with prev = u0 and W = w_0n
 * (sdc.py:304-319; mlsdc.py:68-101).  add (M,N) nullable, sign applied:
 * out = sign*(defect) + add. */
int  sisdc_collocation_defect(sisdc_op1d* op, int M, const double* W, double dt, int incremental,
                              const double* u0, const double* u, const double* f,
                              double sign, const double* add, double* out);

/* ------------------------------------- space-time p-transfers (transfer.py) */
/* It (Mf x Mc) = Lagrange(tau_c -> tau_f), Pt (Mc x Mf); Isp ((Pf+1) x (Pc+1)),
 * Psp ((Pc+1) x (Pf+1)) (transfer.py:61-96,213-245).  The temporal restriction
 * is It^T; the spatial residual restriction Rsp ((Pc+1) x (Pf+1)) is given, or
 * NULL for the reference's Isp^T (transfer.py:243). */
/* 2-D: n_elem = nex*ney*ncomp element slabs, spatial matrices applied in x and y. */
int  sisdc_xfer2d_create(sisdc_ctx* ctx, int n_elem, int pc1, int pf1, int Mc, int Mf,
                         const double* It, const double* Pt, const double* Isp, const double* Psp,
                         const double* Rsp, sisdc_xfer** out);
int  sisdc_xfer_create(sisdc_ctx* ctx, int n_elem, int pc1, int pf1,
                       int Mc, int Mf, const double* It, const double* Pt,
                       const double* Isp, const double* Psp, const double* Rsp, sisdc_xfer** out);
void sisdc_xfer_destroy(sisdc_xfer* x);
/* Spatial apply of one state: dir 0 interp (c->f), 1 project (f->c), 2 restrict (f->c). */
int  sisdc_xfer_spatial(sisdc_xfer* x, int dir, const double* in, double* out);
/* Fine -> coarse space-time apply, spatial factor first (transfer.py:335-342):
 * out (Mc, Nc) = T S in (Mf, Nf); spatial_dir 1 project (P_sp) / 2 restrict (I_sp^T),
 * temporal_dir 1 project (P_t) / 2 restrict (I_t^T). */
int  sisdc_xfer_down(sisdc_xfer* x, int spatial_dir, int temporal_dir, const double* in, double* out);
/* FAS restriction (mlsdc.py:84-101 minus the coarse defect):
 * r = g_f - F_f(u_f) (g_f nullable, F with cached f, incremental/nonincremental W),
 * v = P_t(P_sp u_f), rr = R_t(R_sp r). */
int  sisdc_xfer_fas_restrict(sisdc_xfer* x, const double* Wf, double dt, int incremental,
                             const double* u0f, const double* uf, const double* ff, const double* gf,
                             double* v, double* rr);
/* uf (+)= I_sp(I_t(uc - vc)) ; vc nullable; accumulate 0 assigns
 * (transfer.py:344-352, mlsdc.py:125-126,134-142). */
int  sisdc_xfer_interp(sisdc_xfer* x, int accumulate, const double* uc, const double* vc, double* uf);

/* ------------------------------ element-row partitioned 2-D operators
 * (BASELINE north star: elements partitioned across the GPUs of one
 * box, NCCL only for the face halo and the CG allreduce).  The reference has no
 * parallel path; these calls have no reference counterpart.
 * A partitioned operator owns contiguous element-row blocks of the global
 * mesh `desc`; rank q of nranks owns rows [q*b + min(q,r), +b + (q<r)) with
 * b = ney/nranks, r = ney%nranks.  Its state vectors are the concatenation of
 * its local partitions, each stored (ncomp, rows+2, nex, P+1, P+1) with one
 * ghost row on either side (the neighbours' boundary rows, refreshed by the
 * operator itself before every face-coupled kernel).  Every OperatorContext,
 * sweep-stage and transfer entry point above accepts it unchanged (transfers
 * with n_elem = the storage element slabs, ghost rows included).
 *  - comm == NULL: all nranks partitions are local to this process
 *    (nlocal == nranks, first_rank 0): halo exchange and allreduce are device
 *    copies / fixed-order sums (one GPU emulating nranks ranks).
 *  - comm != NULL: one local partition, rank = comm's rank; halo exchange by
 *    NCCL send/recv, the CG dot products by one NCCL allreduce per iteration.
 * The partitioned implicit solve polls its convergence flag on the host once
 * per two iterations and therefore cannot be captured in a CUDA graph. */
typedef struct sisdc_comm sisdc_comm;
/* NCCL unique id (128 bytes) made on rank 0 and broadcast by the caller. */
int  sisdc_nccl_unique_id(unsigned char* id128);
int  sisdc_comm_create(sisdc_ctx* ctx, const unsigned char* id128, int nranks, int rank, sisdc_comm** out);
void sisdc_comm_destroy(sisdc_comm* comm);
int  sisdc_op2d_create_part(sisdc_ctx* ctx, const sisdc_op2d_desc* global_desc, int nranks, int first_rank,
                            int nlocal, sisdc_comm* comm, sisdc_op1d** out);
/* Local partitions: first global row, owned rows, offset in a state vector. */
int  sisdc_op2d_part_layout(const sisdc_op1d* op, int cap, int* row_begin, int* row_count, int64_t* offset,
                            int* nparts);
/* Refresh the ghost rows of mcount node vectors (stride mstride) of a state
 * (scalar_field 0) or of a scalar coefficient field (scalar_field 1). */
int  sisdc_halo_exchange(sisdc_op1d* op, double* vec, int mcount, int64_t mstride, int scalar_field);

#ifdef __cplusplus
}
#endif
#endif
