// Host-side internals shared by the ABI and the kernel launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include "../../include/sisdc_b200.h"

namespace sisdc {

struct Op1DDev;
struct CoefDev;
struct XferDev;
struct Op2DDev;
struct Xfer2Dev;

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int* d_status = nullptr;        // [0] first non-finite element (INT_MAX: none), [1] CG failures, [2] log count
  int* d_log_it = nullptr;        // per-solve CG iterations
  double* d_log_margin = nullptr; // per-solve ||r||/(rtol ||b||)
  int log_cap = 1 << 20;          // per-solve log entries kept (a long test session logs > 65k solves)
  long long* d_timing = nullptr;  // SISDC_CG_TIMING=1: CG clock64 stamps [66]
  double* d_cg1g = nullptr;       // grid-mode 1-D CG: halo / reduction exchange buffers (CG1G_DOUBLES)
  double rtol = 1e-14;
  int maxit = 1000;
  int cluster_ctas = 0;
  int pdl = 1;                    // programmatic dependent launch of the 1-D kernels (SISDC_PDL=0 disables)
  int64_t launches = 0;
  std::string err;

  int fail(int code, const std::string& msg) {
    err = msg;
    return code;
  }
  int cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SISDC_OK;
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return SISDC_ERR_CUDA;
  }
  int after_launch(const char* name) {
    ++launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      err = std::string("launch ") + name + ": " + cudaGetErrorString(e);
      return SISDC_ERR_CUDA;
    }
    return SISDC_OK;
  }
};

constexpr int CG1G_MAXK = 1024;                       // grid-mode 1-D CG: most blocks of one solve
constexpr size_t CG1G_DOUBLES = (size_t)CG1G_MAXK * (22 * 16 + 12);

int launch_apply_convection(Ctx* c, const Op1DDev& op, const double* u, double* out);
int launch_apply_diffusion(Ctx* c, const Op1DDev& op, CoefDev k, const double* u, double* out);
int launch_coef_field(Ctx* c, const Op1DDev& op, CoefDev k, double* out);
int launch_node_eval(Ctx* c, const Op1DDev& op, int mode, int scheme, int M, int m_first, int m_count,
                     const double* u0, const double* u, const double* conv_prev, const double* dts,
                     double* f, double* h1, double* h2, const double* bnd = nullptr);
int launch_stage_rhs(Ctx* c, const Op1DDev& op, const double* base, const double* conv_in, double dt_m,
                     const double* f_old, int M, const double* w_row, double dt, const double* g,
                     const double* h, double* rhs, double* conv_out);
int launch_defect(Ctx* c, int N, int M, const double* W, double dt, int incremental, const double* u0,
                  const double* u, const double* f, double sign, const double* add, double* out);
int launch_xfer_spatial(Ctx* c, const XferDev& x, int dir, const double* in, double* out);
int launch_fas_restrict(Ctx* c, const XferDev& x, const double* Wf, double dt, int incremental, const double* u0f,
                        const double* uf, const double* ff, const double* gf, double* v, double* rr);
int launch_xfer_down(Ctx* c, const XferDev& x, int sdir, int tdir, const double* in, double* out);
int launch_xfer_interp(Ctx* c, const XferDev& x, int accumulate, const double* uc, const double* vc, double* uf);
int launch_lincomb(Ctx* c, long long n, const double* coef, const double* const* v, double* out);
int launch_smooth_start(Ctx* c, const Op1DDev& op, int M, const double* u, double* out);
int launch_persson(Ctx* c, const Op1DDev& op, const double* u, double kappa, double cs, double* nu_art);
// stage rhs fused into the 1-D CG prologue (sisdc_stage_solve)
struct StageFuse {
  const double* base;
  const double* conv_in;
  const double* f_old;
  const double* w_row;
  const double* g;
  const double* h;
  double* conv_out;
  double dt_m, dt, gl, gr;
  int M;
};
int launch_cg1d(Ctx* c, const Op1DDev& op, CoefDev k, double a, const double* rhs, double* x,
                const StageFuse* sf = nullptr);
// 1-D compressible flow, 3 fields (cns1d.cu)
int cns_conv(Ctx* c, const Op1DDev& op, const double* u, double* out);
int cns_sip(Ctx* c, const Op1DDev& op, CoefDev k, const double* u, double* out);
int cns_coef(Ctx* c, const Op1DDev& op, CoefDev k, double* out);
int cns_node_eval(Ctx* c, const Op1DDev& op, int mode, int scheme, int M, int m_first, int m_count,
                  const double* u0, const double* u, const double* conv_prev, const double* dts, double* f,
                  double* h1, double* h2, const double* bnd = nullptr);   // bnd: (M, 12) Dirichlet states
int cns_stage(Ctx* c, const Op1DDev& op, const double* base, const double* conv_in, double dt_m,
              const double* f_old, int M, const double* w_row, double dt, const double* g, const double* h,
              double* rhs, double* conv_out);
int cns_solve(Ctx* c, const Op1DDev& op, CoefDev k, double a, const double* rhs, double* x, double* c9,
              double* pinv, const double* dbc = nullptr);
// 2-D (ops2d.cu)
int launch2_conv(Ctx* c, const Op2DDev& op, const double* u, double* out);
int launch2_sip(Ctx* c, const Op2DDev& op, CoefDev k, const double* u, double* out);
// NS2D physical viscous operator: f[m] (+)= visc(u[m]) for m in [m_first, m_first + m_count)
int launch2_visc(Ctx* c, const Op2DDev& op, const double* u, double* f, int m_first, int m_count, int accumulate);
int launch2_visc8(Ctx* c, const Op2DDev& op, const double* u, double* f, int m_first, int m_count, int accumulate);
int launch2_persson(Ctx* c, const Op2DDev& op, const double* u, double kappa, double cs, double* nu_art);
int launch2_coef(Ctx* c, const Op2DDev& op, CoefDev k, double* out);
int launch2_node_eval(Ctx* c, const Op2DDev& op, int mode, int scheme, int M, int m_first, int m_count,
                      const double* u0, const double* u, const double* conv_prev, const double* dts,
                      double* f, double* h1, double* h2);
int launch2_stage(Ctx* c, const Op2DDev& op, const double* base, const double* conv_in, double dt_m,
                  const double* f_old, int M, const double* w_row, double dt, const double* g,
                  const double* h, double* rhs, double* conv_out);
int launch2x_spatial(Ctx* c, const Xfer2Dev& x, int dir, const double* in, double* out);
int launch2x_down(Ctx* c, const Xfer2Dev& x, int sdir, int tdir, const double* in, double* out);
int launch2x_fas(Ctx* c, const Xfer2Dev& x, const double* Wf, double dt, int incremental, const double* u0f,
                 const double* uf, const double* ff, const double* gf, double* v, double* rr);
int launch2x_interp(Ctx* c, const Xfer2Dev& x, int accumulate, const double* uc, const double* vc, double* uf);
int launch2_cg(Ctx* c, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws, int nblocks);
int cg2_blocks(Ctx* c, const Op2DDev& op, int* nblocks);
size_t cg2_ws_doubles(const Op2DDev& op, int nblocks);
int set_cg2_tables(Ctx* c, int p1, const double* tab);
// partitioned (ghost-row) 2-D operators: split CG phases, reductions, halo (ops2d.cu)
struct CgPScal;
enum { P2_INIT = 0, P2_DINV, P2_RESID, P2_U0, P2_UPDATE, P2_MATVEC };
size_t cg2p_ws_doubles(const Op2DDev& op, int G);
bool cg2p_fused(const Op2DDev& op);
size_t cg2p_dinv_off(const Op2DDev& op);
double* cg2p_RSW(const Op2DDev& op, double* ws, int par);
int launch2p_fpass(Ctx* c, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws, int G,
                   const CgPScal* sc, int par, int bsel = 0, int slot0 = 0, int nblk = -1);
int cg2p_bands(const Op2DDev& op);
double* cg2p_U(const Op2DDev& op, double* ws, int which);
int cg2p_blocks(Ctx* c, const Op2DDev& op, int* G);
int launch2p_phase(Ctx* c, int phase, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x,
                   double* ws, int G, const CgPScal* sc, int ucur);
int launch2p_reduce(Ctx* c, int nparts, double* const* ws, const Op2DDev* ops, int G, int mode, double* out,
                    int fsetup = 0);
int launch2p_fsetup(Ctx* c, int mode, const Op2DDev& op, CoefDev k, double a, const double* rhs, double* x, double* ws,
                    int G, const CgPScal* sc);
int launch2p_scalar(Ctx* c, int mode, const double* tot, CgPScal* sc);
int launch2p_halo_pack(Ctx* c, const Op2DDev& op, double* vec, double* buf, int nc, int mcount, long long mstride,
                       int dir);
int launch2p_halo(Ctx* c, int nparts, const Op2DDev* ops, double* const* base, int nc, int mcount, long long mstride);

}  // namespace sisdc
