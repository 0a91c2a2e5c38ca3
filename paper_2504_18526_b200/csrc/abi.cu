// C ABI of libsisdc_b200.so: contexts, operators, transfers and the exported
// OperatorContext / sweep-stage entry points (include/sisdc_b200.h).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>
#include "sisdc_dev.cuh"
#include "sisdc_dev2d.cuh"
#include "sisdc_host.h"

using namespace sisdc;

#include "abi_internal.h"

namespace {

// ---------------------------------------------- host element tables
void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0;
  if (n == 0) { p = 1.0; dp = 0.0; return; }
  for (int k = 1; k < n; ++k) {
    double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    double d2 = d0 + (2 * k + 1) * p1;
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  p = p1; dp = d1;
}

// GLL nodes (roots of (1-x^2) P'_P) by Newton from Chebyshev-Lobatto guesses,
// weights 2/(P(P+1) P_P(x)^2)  (collocation.py:163-167)
void gll(int p1, std::vector<double>& x, std::vector<double>& w) {
  const int P = p1 - 1;
  x.assign(p1, 0.0); w.assign(p1, 0.0);
  x[0] = -1.0; x[P] = 1.0;
  for (int j = 1; j < P; ++j) {
    double z = -std::cos(M_PI * j / P);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre(P, z, p, dp);
      double d2 = (2.0 * z * dp - P * (P + 1) * p) / (1.0 - z * z);
      double step = dp / d2;
      z -= step;
      if (std::fabs(step) < 1e-16) break;
    }
    x[j] = z;
  }
  for (int j = 0; j < p1; ++j) {
    double p, dp;
    legendre(P, x[j], p, dp);
    w[j] = 2.0 / (P * (P + 1) * p * p);
  }
}

// barycentric D (dgsem.py:33-43)
std::vector<double> diff_matrix(const std::vector<double>& x) {
  int n = (int)x.size();
  std::vector<double> lam(n), D(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double pr = 1.0;
    for (int k = 0; k < n; ++k) if (k != j) pr *= (x[j] - x[k]);
    lam[j] = 1.0 / pr;
  }
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      D[i * n + j] = (lam[j] / lam[i]) / (x[i] - x[j]);
      s += D[i * n + j];
    }
    D[i * n + i] = -s;
  }
  return D;
}

bool invert(std::vector<double> A, int n, std::vector<double>& inv) {
  inv.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r) if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (A[piv * n + c] == 0.0) return false;
    for (int k = 0; k < n; ++k) { std::swap(A[c * n + k], A[piv * n + k]); std::swap(inv[c * n + k], inv[piv * n + k]); }
    double d = A[c * n + c];
    for (int k = 0; k < n; ++k) { A[c * n + k] /= d; inv[c * n + k] /= d; }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = A[r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) { A[r * n + k] -= f * A[c * n + k]; inv[r * n + k] -= f * inv[c * n + k]; }
    }
  }
  return true;
}

// Dirichlet trace data of time t from the operator's table (exact match);
// table rows (t, g_l[nc], g_r[nc])
int bc_at3(sisdc_op1d* op, double t, double* gl, double* gr) {
  const int nc = op->dim == 1 ? op->dev.nc : 1, st = 1 + 2 * nc;
  for (int c = 0; c < nc; ++c) gl[c] = gr[c] = 0.0;
  if (op->dim != 1 || op->dev.bc != SISDC_DIRICHLET) return SISDC_OK;
  for (size_t j = 0; j + st - 1 < op->btab.size(); j += st)
    if (op->btab[j] == t) {
      for (int c = 0; c < nc; ++c) { gl[c] = op->btab[j + 1 + c]; gr[c] = op->btab[j + 1 + nc + c]; }
      return SISDC_OK;
    }
  return C(op)->fail(SISDC_ERR_ARG, "no Dirichlet boundary data registered for t = " + std::to_string(t));
}
int bc_at(sisdc_op1d* op, double t, double& gl, double& gr) {
  double l[3], r[3];
  int rc = bc_at3(op, t, l, r);
  gl = l[0];
  gr = r[0];
  return rc;
}
// the operator with its boundary states at time t
int dev_at(sisdc_op1d* op, double t, Op1DDev& d) {
  d = op->dev;
  if (int rc = bc_at3(op, t, d.gl3, d.gr3)) return rc;
  d.gl = d.gl3[0];
  d.gr = d.gr3[0];
  return SISDC_OK;
}

int check_coef(Ctx* c, sisdc_coef k);
int check_coef_op(sisdc_op1d* op, sisdc_coef k) {
  if (k.kind == SISDC_COEF_MATRIX && !op->cns())
    return C(op)->fail(SISDC_ERR_UNSUPPORTED, "matrix-valued coefficients are built for the 1-D CNS problem only");
  if (op->cns() && (k.kind == SISDC_COEF_SI || k.kind == SISDC_COEF_PHYS) && !k.ptr)
    return C(op)->fail(SISDC_ERR_ARG, "CNS coefficients need the frozen state u_b");
  return check_coef(C(op), k);
}
int check_coef(Ctx* c, sisdc_coef k) {
  if (k.kind < SISDC_COEF_NONE || k.kind > SISDC_COEF_MATRIX) return c->fail(SISDC_ERR_ARG, "unknown coefficient kind");
  if ((k.kind == SISDC_COEF_FIELD || k.kind == SISDC_COEF_SI || k.kind == SISDC_COEF_MATRIX) && !k.ptr)
    return c->fail(SISDC_ERR_ARG, "coefficient needs a device pointer");
  return SISDC_OK;
}

}  // namespace

extern "C" {

int sisdc_abi_version(void) { return SISDC_ABI_VERSION; }

int sisdc_struct_size(int which) {
  switch (which) {
    case 0: return (int)sizeof(sisdc_op1d_desc);
    case 1: return (int)sizeof(sisdc_op2d_desc);
    case 2: return (int)sizeof(sisdc_coef);
    default: return -1;
  }
}

int sisdc_ctx_create(int device, sisdc_ctx** out) {
  if (!out) return SISDC_ERR_ARG;
  *out = nullptr;
  sisdc_ctx* x = new (std::nothrow) sisdc_ctx();
  if (!x) return SISDC_ERR_ARG;
  Ctx& c = x->c;
  c.device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&c.d_status, 4 * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&c.d_log_it, c.log_cap * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&c.d_log_margin, c.log_cap * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c.d_cg1g, CG1G_DOUBLES * sizeof(double));   // at creation: graph-safe
  if (e != cudaSuccess) {
    delete x;
    return SISDC_ERR_CUDA;
  }
  const char* pdl = getenv("SISDC_PDL");   // A/B switch for programmatic dependent launch
  if (pdl && pdl[0] == '0') c.pdl = 0;
  const char* tm = getenv("SISDC_CG_TIMING");
  if (e == cudaSuccess && tm && tm[0] == '1') {
    e = cudaMalloc(&c.d_timing, 80 * sizeof(long long));
    if (e == cudaSuccess) e = cudaMemset(c.d_timing, 0, 80 * sizeof(long long));
  }
  int init[4] = {INT_MAX, 0, 0, 0};
  cudaMemcpy(c.d_status, init, sizeof(init), cudaMemcpyHostToDevice);
  *out = x;
  return SISDC_OK;
}

void sisdc_ctx_destroy(sisdc_ctx* x) {
  if (!x) return;
  cudaFree(x->c.d_status);
  cudaFree(x->c.d_log_it);
  cudaFree(x->c.d_log_margin);
  cudaFree(x->c.d_timing);
  cudaFree(x->c.d_cg1g);
  delete x;
}

const char* sisdc_ctx_last_error(const sisdc_ctx* x) { return x ? x->c.err.c_str() : "null context"; }

int sisdc_ctx_set_stream(sisdc_ctx* x, void* stream) {
  if (!x) return SISDC_ERR_ARG;
  x->c.stream = (cudaStream_t)stream;
  return SISDC_OK;
}

int sisdc_ctx_synchronize(sisdc_ctx* x) {
  if (!x) return SISDC_ERR_ARG;
  return x->c.cuda(cudaStreamSynchronize(x->c.stream), "synchronize");
}

int sisdc_ctx_set_cg(sisdc_ctx* x, double rtol, int maxit, int cluster_ctas) {
  if (!x || !(rtol > 0.0) || maxit < 1 || cluster_ctas < 0 || cluster_ctas > 16) return SISDC_ERR_ARG;
  x->c.rtol = rtol;
  x->c.maxit = maxit;
  x->c.cluster_ctas = cluster_ctas;
  return SISDC_OK;
}

int sisdc_ctx_status(sisdc_ctx* x, int* nonfinite_elem, int* cg_failures, int* n_solves) {
  if (!x) return SISDC_ERR_ARG;
  int h[4];
  int rc = x->c.cuda(cudaStreamSynchronize(x->c.stream), "status sync");
  if (rc) return rc;
  rc = x->c.cuda(cudaMemcpy(h, x->c.d_status, sizeof(h), cudaMemcpyDeviceToHost), "status read");
  if (rc) return rc;
  if (nonfinite_elem) *nonfinite_elem = h[0] == INT_MAX ? -1 : h[0];
  if (cg_failures) *cg_failures = h[1];
  if (n_solves) *n_solves = h[2];
  return SISDC_OK;
}

int sisdc_ctx_reset_status(sisdc_ctx* x) {
  if (!x) return SISDC_ERR_ARG;
  k_reset_status<<<1, 32, 0, x->c.stream>>>(x->c.d_status, 0);   // kernel, so it is graph-capturable
  return x->c.after_launch("reset_status");
}

int sisdc_ctx_reset_log(sisdc_ctx* x) {
  if (!x) return SISDC_ERR_ARG;
  k_reset_status<<<1, 32, 0, x->c.stream>>>(x->c.d_status, 1);
  return x->c.after_launch("reset_log");
}

int sisdc_ctx_cg_log(sisdc_ctx* x, int cap, int* iters, double* margins, int* n_out) {
  if (!x || cap < 0) return SISDC_ERR_ARG;
  int n = 0;
  int rc = sisdc_ctx_status(x, nullptr, nullptr, &n);
  if (rc) return rc;
  if (n > x->c.log_cap) n = x->c.log_cap;
  int m = n < cap ? n : cap;
  if (m > 0 && iters) rc = x->c.cuda(cudaMemcpy(iters, x->c.d_log_it, m * sizeof(int), cudaMemcpyDeviceToHost), "log");
  if (!rc && m > 0 && margins)
    rc = x->c.cuda(cudaMemcpy(margins, x->c.d_log_margin, m * sizeof(double), cudaMemcpyDeviceToHost), "log");
  if (n_out) *n_out = n;
  return rc;
}

int sisdc_ctx_debug_timing(sisdc_ctx* x, long long* out, int cap) {
  if (!x || !out || cap < 0) return SISDC_ERR_ARG;
  if (!x->c.d_timing) return x->c.fail(SISDC_ERR_UNSUPPORTED, "set SISDC_CG_TIMING=1 before creating the context");
  int n = cap < 80 ? cap : 80;
  int rc = x->c.cuda(cudaStreamSynchronize(x->c.stream), "timing sync");
  if (!rc) rc = x->c.cuda(cudaMemcpy(out, x->c.d_timing, n * sizeof(long long), cudaMemcpyDeviceToHost), "timing");
  return rc;
}

int64_t sisdc_ctx_launch_count(const sisdc_ctx* x) { return x ? x->c.launches : -1; }

int sisdc_lincomb(sisdc_ctx* x, int64_t n, const double* coef4, const double* v0, const double* v1,
                  const double* v2, const double* v3, double* out) {
  if (!x || !coef4 || !out || n < 0) return SISDC_ERR_ARG;
  const double* v[4] = {v0, v1, v2, v3};
  return launch_lincomb(&x->c, n, coef4, v, out);
}

int sisdc_copy(sisdc_ctx* x, double* dst, const double* src, int64_t n) {
  if (!x || n < 0 || (n > 0 && (!dst || !src))) return SISDC_ERR_ARG;
  if (n == 0) return SISDC_OK;
  return x->c.cuda(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, x->c.stream), "copy");
}

// ------------------------------------------------------------ operators
int sisdc_op1d_create(sisdc_ctx* x, const sisdc_op1d_desc* d, sisdc_op1d** out) {
  if (!x || !d || !out) return SISDC_ERR_ARG;
  *out = nullptr;
  Ctx& c = x->c;
  if (!(d->x_right > d->x_left)) return c.fail(SISDC_ERR_ARG, "empty domain");
  if (d->n_elem < 1 || d->degree < 1) return c.fail(SISDC_ERR_ARG, "need at least one element and degree >= 1");
  if (d->degree + 1 > MAXP1) return c.fail(SISDC_ERR_UNSUPPORTED, "degree above 15");
  const bool cns = d->problem == SISDC_CNS1D;
  if (d->ncomp != (cns ? 3 : 1)) return c.fail(SISDC_ERR_ARG, "ncomp does not match the problem");
  if (cns && d->n_elem < 2) return c.fail(SISDC_ERR_UNSUPPORTED, "1-D compressible flow needs >= 2 elements");
  if (cns && !(d->gamma > 1.0)) return c.fail(SISDC_ERR_ARG, "gamma must exceed 1");
  if (cns && !(d->prandtl > 0.0)) return c.fail(SISDC_ERR_ARG, "Prandtl number must be positive");
  if (cns && d->eta < 0.0) return c.fail(SISDC_ERR_ARG, "viscosity must be nonnegative");
  if (d->bc != SISDC_PERIODIC && d->bc != SISDC_DIRICHLET) return c.fail(SISDC_ERR_ARG, "unknown boundary condition");
  if (d->problem != SISDC_CONVDIFF && d->problem != SISDC_BURGERS && !cns) return c.fail(SISDC_ERR_ARG, "unknown problem");
  if (d->nu < 0) return c.fail(SISDC_ERR_ARG, "diffusion coefficient must be nonnegative");
  sisdc_op1d* op = new (std::nothrow) sisdc_op1d();
  if (!op) return SISDC_ERR_ARG;
  op->ctx = x;
  op->desc = *d;
  const int p1 = d->degree + 1;
  gll(p1, op->nodes, op->weights);
  op->D = diff_matrix(op->nodes);
  const double dx = (d->x_right - d->x_left) / d->n_elem;
  std::vector<double> tab(TabOff::size(p1), 0.0);
  for (int i = 0; i < p1; ++i)
    for (int k = 0; k < p1; ++k) {
      tab[TabOff::D(p1) + i * p1 + k] = op->D[i * p1 + k];
      tab[TabOff::DTW(p1) + i * p1 + k] = op->D[k * p1 + i] * op->weights[k];
      tab[TabOff::D2W(p1) + i * p1 + k] = op->D[k * p1 + i] * op->D[k * p1 + i] * op->weights[k];
    }
  for (int i = 0; i < p1; ++i) {
    double m = 0.5 * dx * op->weights[i];
    tab[TabOff::w(p1) + i] = op->weights[i];
    tab[TabOff::m(p1) + i] = m;
    tab[TabOff::minv(p1) + i] = 1.0 / m;
  }
  std::vector<double> V(p1 * p1), Vi;
  for (int i = 0; i < p1; ++i)
    for (int k = 0; k < p1; ++k) { double p, dp; legendre(k, op->nodes[i], p, dp); V[i * p1 + k] = p; }
  invert(V, p1, Vi);
  for (int i = 0; i < p1 * p1; ++i) tab[TabOff::Vinv(p1) + i] = Vi[i];
  cudaError_t e = cudaMalloc(&op->d_tab, tab.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(op->d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    int rc = c.cuda(e, "op1d tables");
    delete op;
    return rc;
  }
  Op1DDev& v = op->dev;
  v.ne = d->n_elem; v.p1 = p1; v.n = d->n_elem * p1; v.problem = d->problem;
  v.dx = dx; v.s = 2.0 / dx; v.mu0 = d->penalty * p1 * p1 / dx;   // dgsem.py:137
  v.speed = d->speed; v.nu = d->nu; v.tab = op->d_tab; v.nu_art = nullptr;
  v.bc = d->bc; v.gl = 0.0; v.gr = 0.0;
  v.nc = d->ncomp; v.gamma = d->gamma; v.eta = d->eta; v.Pr = d->prandtl;
  if (cns) {
    const size_t nb = 3 * p1;
    e = cudaMalloc(&op->d_pinv, (size_t)d->n_elem * nb * nb * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&op->d_c9, (size_t)d->n_elem * p1 * 9 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&op->d_cws, (size_t)2 * 3 * d->n_elem * p1 * sizeof(double));
    if (e == cudaSuccess) e = cudaMemset(op->d_cws, 0, (size_t)3 * d->n_elem * p1 * sizeof(double));   // zero vector
    if (e != cudaSuccess) {
      int rc = c.cuda(e, "cns block-Jacobi workspace");
      cudaFree(op->d_tab);
      cudaFree(op->d_pinv);
      delete op;
      return rc;
    }
  }
  *out = op;
  return SISDC_OK;
}

}  // extern "C"

// 2-D operator: shared 1-D element tables + tensor-product kernels
int op2d_create_impl(sisdc_ctx* x, const sisdc_op2d_desc* d, bool alloc_cg, sisdc_op1d** out) {
  if (!x || !d || !out) return SISDC_ERR_ARG;
  *out = nullptr;
  Ctx& c = x->c;
  if (!(d->x_right > d->x_left) || !(d->y_top > d->y_bottom)) return c.fail(SISDC_ERR_ARG, "empty domain");
  if (d->nex < 1 || d->ney < 1 || d->degree < 1) return c.fail(SISDC_ERR_ARG, "need elements and degree >= 1");
  if (d->degree + 1 > 9) return c.fail(SISDC_ERR_UNSUPPORTED, "2-D degree above 8");
  const bool euler = d->problem == SISDC_EULER2D || d->problem == SISDC_NS2D;
  if (d->problem == SISDC_NS2D && !(d->prandtl > 0.0)) return c.fail(SISDC_ERR_ARG, "Prandtl number must be positive");
  if (!euler && d->problem != SISDC_ADVECTION2D && d->problem != SISDC_BURGERS2D)
    return c.fail(SISDC_ERR_ARG, "unknown 2-D problem");
  if ((euler && d->ncomp != 4) || (!euler && d->ncomp != 1)) return c.fail(SISDC_ERR_ARG, "ncomp does not match the problem");
  if (d->nu < 0) return c.fail(SISDC_ERR_ARG, "viscosity must be nonnegative");
  sisdc_op1d* op = new (std::nothrow) sisdc_op1d();
  if (!op) return SISDC_ERR_ARG;
  op->ctx = x;
  op->dim = 2;
  const int p1 = d->degree + 1;
  gll(p1, op->nodes, op->weights);
  op->D = diff_matrix(op->nodes);
  const double dx = (d->x_right - d->x_left) / d->nex, dy = (d->y_top - d->y_bottom) / d->ney;
  std::vector<double> tab(TabOff::size(p1), 0.0);
  for (int i = 0; i < p1; ++i)
    for (int k = 0; k < p1; ++k) {
      tab[TabOff::D(p1) + i * p1 + k] = op->D[i * p1 + k];
      tab[TabOff::DTW(p1) + i * p1 + k] = op->D[k * p1 + i] * op->weights[k];
      tab[TabOff::D2W(p1) + i * p1 + k] = op->D[k * p1 + i] * op->D[k * p1 + i] * op->weights[k];
    }
  for (int i = 0; i < p1; ++i) {
    tab[TabOff::w(p1) + i] = op->weights[i];
    tab[TabOff::m(p1) + i] = op->weights[i];
    tab[TabOff::minv(p1) + i] = 1.0 / op->weights[i];
  }
  {   // inverse Legendre Vandermonde (the modal sensor of the artificial viscosity)
    std::vector<double> V(p1 * p1), Vi;
    for (int i = 0; i < p1; ++i)
      for (int k = 0; k < p1; ++k) { double p, dp; legendre(k, op->nodes[i], p, dp); V[i * p1 + k] = p; }
    invert(V, p1, Vi);
    for (int i = 0; i < p1 * p1; ++i) tab[TabOff::Vinv(p1) + i] = Vi[i];
  }
  Op2DDev& v = op->dev2;
  v.nex = d->nex; v.ney = d->ney; v.p1 = p1; v.nc = d->ncomp;
  v.nys = d->ney; v.row0 = 0; v.e0 = 0;
  v.nn = (long long)d->nex * d->ney * p1 * p1;
  v.n = v.nn * d->ncomp;
  v.ns = v.n;
  v.problem = d->problem;
  v.dx = dx; v.dy = dy; v.sx = 2.0 / dx; v.sy = 2.0 / dy;
  v.mux = d->penalty * p1 * p1 / dx; v.muy = d->penalty * p1 * p1 / dy;
  v.gamma = d->gamma; v.nu = d->nu; v.ax = d->ax; v.ay = d->ay;
  v.pr = d->problem == SISDC_NS2D ? d->prandtl : 1.0;
  v.nsi = d->problem == SISDC_NS2D ? std::max(4.0 / 3.0, d->gamma / d->prandtl) : 0.0;
  v.nu_art = nullptr;
  v.fused_sub2 = 0;
  cudaError_t e = cudaMalloc(&op->d_tab, tab.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(op->d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    int rc = c.cuda(e, "op2d tables");
    delete op;
    return rc;
  }
  v.tab = op->d_tab;
  int rc = set_cg2_tables(&c, p1, tab.data());
  if (!rc && alloc_cg) rc = cg2_blocks(&c, v, &op->cg_blocks);
  if (rc) { cudaFree(op->d_tab); delete op; return rc; }
  if (!alloc_cg) {
    *out = op;
    return SISDC_OK;
  }
  const size_t ws = cg2_ws_doubles(v, op->cg_blocks);
  e = cudaMalloc(&op->d_cgws, ws * sizeof(double));
  if (e != cudaSuccess) {
    rc = c.cuda(e, "op2d CG workspace");
    cudaFree(op->d_tab);
    delete op;
    return rc;
  }
  *out = op;
  return SISDC_OK;
}

extern "C" {

int sisdc_op2d_create(sisdc_ctx* x, const sisdc_op2d_desc* d, sisdc_op1d** out) {
  return op2d_create_impl(x, d, true, out);
}

void sisdc_op1d_destroy(sisdc_op1d* op) {
  if (!op) return;
  if (op->parted()) part2_destroy(op);
  cudaFree(op->d_tab);
  cudaFree(op->d_cgws);
  cudaFree(op->d_pinv);
  cudaFree(op->d_c9);
  cudaFree(op->d_cws);
  delete op;
}

int sisdc_op1d_tables(const sisdc_op1d* op, double* nodes, double* weights, double* D) {
  if (!op) return SISDC_ERR_ARG;
  int p1 = op->dev.p1;
  if (nodes) std::memcpy(nodes, op->nodes.data(), p1 * sizeof(double));
  if (weights) std::memcpy(weights, op->weights.data(), p1 * sizeof(double));
  if (D) std::memcpy(D, op->D.data(), p1 * p1 * sizeof(double));
  return SISDC_OK;
}

int sisdc_op1d_set_nu_art(sisdc_op1d* op, const double* nu_art) {
  if (!op) return SISDC_ERR_ARG;
  op->dev.nu_art = nu_art;
  op->dev2.nu_art = nu_art;
  // partitioned 2-D operator: nu_art is stored per STORAGE row ((rows + 2) x nex per partition, the ghost
  // rows filled by sisdc_persson_viscosity's halo), partitions concatenated
  long long offe = 0;
  for (Part2D& P : op->parts) {
    P.dev.nu_art = nu_art ? nu_art + offe : nullptr;
    offe += (long long)P.dev.nys * P.dev.nex;
  }
  return SISDC_OK;
}

int sisdc_smooth_start(sisdc_op1d* op, int M, const double* u, double* out) {
  if (!op || !u || !out || M < 1) return SISDC_ERR_ARG;
  if (op->dim == 2) return C(op)->fail(SISDC_ERR_UNSUPPORTED, "smooth_start is built for 1-D meshes");
  return launch_smooth_start(C(op), op->dev, M, u, out);
}

int sisdc_persson_viscosity(sisdc_op1d* op, const double* u, double kappa_s, double c_s, double* nu_art) {
  if (!op || !u || !nu_art || !(kappa_s > 0)) return SISDC_ERR_ARG;
  if (op->dim == 2) {
    if (!op->parted()) return launch2_persson(C(op), op->dev2, u, kappa_s, c_s, nu_art);
    long long offe = 0;
    for (const Part2D& P : op->parts) {   // owned rows of every local partition, then the ghost rows
      if (int rc = launch2_persson(C(op), P.dev, u + P.off, kappa_s, c_s, nu_art + offe)) return rc;
      offe += (long long)P.dev.nys * P.dev.nex;
    }
    return part2_halo_elem(op, nu_art);
  }
  return launch_persson(C(op), op->dev, u, kappa_s, c_s, nu_art);
}

int sisdc_op1d_set_boundary(sisdc_op1d* op, int n, const double* times, const double* gl, const double* gr) {
  if (!op || n < 0 || (n > 0 && (!times || !gl || !gr))) return SISDC_ERR_ARG;
  const int nc = op->dim == 1 ? op->dev.nc : 1, st = 1 + 2 * nc;   // gl, gr: (n, ncomp)
  for (int j = 0; j < n; ++j) {
    bool found = false;
    for (size_t q = 0; q + st - 1 < op->btab.size(); q += st)
      if (op->btab[q] == times[j]) {
        for (int c = 0; c < nc; ++c) { op->btab[q + 1 + c] = gl[j * nc + c]; op->btab[q + 1 + nc + c] = gr[j * nc + c]; }
        found = true;
        break;
      }
    if (!found) {
      op->btab.push_back(times[j]);
      for (int c = 0; c < nc; ++c) op->btab.push_back(gl[j * nc + c]);
      for (int c = 0; c < nc; ++c) op->btab.push_back(gr[j * nc + c]);
    }
  }
  if (op->btab.size() > (size_t)st * 4096) op->btab.erase(op->btab.begin(), op->btab.end() - st * 1024);   // keep recent times
  return SISDC_OK;
}

int sisdc_apply_convection(sisdc_op1d* op, const double* u, double t, double* out) {
  if (!op || !u || !out) return SISDC_ERR_ARG;
  if (op->parted()) return part2_conv(op, u, out);
  if (op->dim == 2) return launch2_conv(C(op), op->dev2, u, out);
  if (op->cns()) {
    Op1DDev d;
    if (int rc = dev_at(op, t, d)) return rc;
    return cns_conv(C(op), d, u, out);
  }
  Op1DDev d;
  if (int rc = dev_at(op, t, d)) return rc;
  return launch_apply_convection(C(op), d, u, out);
}

int sisdc_apply_diffusion(sisdc_op1d* op, sisdc_coef k, const double* u, double t, double* out) {
  if (!op || !u || !out) return SISDC_ERR_ARG;
  if (int rc = check_coef_op(op, k)) return rc;
  if (k.kind == SISDC_COEF_NONE || (k.kind == SISDC_COEF_CONST && k.value == 0.0))
    return C(op)->cuda(cudaMemsetAsync(out, 0, op->n() * sizeof(double), C(op)->stream), "zero");
  if (op->parted()) return part2_sip(op, coef(k), u, out);
  if (op->dim == 2) return launch2_sip(C(op), op->dev2, coef(k), u, out);
  if (op->cns()) {
    Op1DDev d;
    if (int rc = dev_at(op, t, d)) return rc;
    return cns_sip(C(op), d, coef(k), u, out);
  }
  Op1DDev d;
  if (int rc = dev_at(op, t, d)) return rc;
  return launch_apply_diffusion(C(op), d, coef(k), u, out);
}

int sisdc_eval_rhs(sisdc_op1d* op, const double* u, double t, double* out) {
  if (!op || !u || !out) return SISDC_ERR_ARG;
  if (op->parted()) return part2_eval_nodes(op, 0, SISDC_SI2, 1, 0, 1, u, u, nullptr, nullptr, out, nullptr, nullptr);
  if (op->dim == 2)
    return launch2_node_eval(C(op), op->dev2, 0, SISDC_SI2, 1, 0, 1, u, u, nullptr, nullptr, out, nullptr, nullptr);
  if (op->cns()) {
    double bnd[12] = {};
    if (int rc = bc_at3(op, t, bnd, bnd + 3)) return rc;
    return cns_node_eval(C(op), op->dev, 0, SISDC_SI2, 1, 0, 1, u, u, nullptr, nullptr, out, nullptr, nullptr,
                         op->dev.bc == SISDC_DIRICHLET ? bnd : nullptr);
  }
  Op1DDev d;
  if (int rc = dev_at(op, t, d)) return rc;
  return launch_node_eval(C(op), d, 0, SISDC_SI2, 1, 0, 1, u, u, nullptr, nullptr, out, nullptr, nullptr);
}

int sisdc_coef_field(sisdc_op1d* op, sisdc_coef k, double* out) {
  if (!op || !out) return SISDC_ERR_ARG;
  if (int rc = check_coef_op(op, k)) return rc;
  if (op->parted()) return part2_coef_field(op, coef(k), out);
  if (op->dim == 2) return launch2_coef(C(op), op->dev2, coef(k), out);
  if (op->cns()) return cns_coef(C(op), op->dev, coef(k), out);   // (n_elem, P+1, 3, 3)
  return launch_coef_field(C(op), op->dev, coef(k), out);
}

int sisdc_implicit_solve(sisdc_op1d* op, sisdc_coef k, double a, const double* rhs, double t, double* x) {
  if (!op || !rhs || !x) return SISDC_ERR_ARG;
  if (int rc = check_coef_op(op, k)) return rc;
  if (a == 0.0) {   // dgsem.py:505-506
    if (x == rhs) return SISDC_OK;
    return sisdc_copy(op->ctx, x, rhs, op->n());
  }
  if (k.kind == SISDC_COEF_NONE) return C(op)->fail(SISDC_ERR_ARG, "cannot assemble a zero coefficient");
  if (op->parted()) return part2_solve(op, coef(k), a, rhs, x);
  if (op->dim == 2) return launch2_cg(C(op), op->dev2, coef(k), a, rhs, x, op->d_cgws, op->cg_blocks);
  if (op->cns()) {
    if (x == rhs) return C(op)->fail(SISDC_ERR_ARG, "implicit_solve: x must not alias rhs");
    Op1DDev d;
    if (int rc = dev_at(op, t, d)) return rc;
    const double* dbc = nullptr;
    if (d.bc == SISDC_DIRICHLET) {   // affine SIP: D(0; t) moves to the right-hand side (dgsem.py:517-529)
      double* zero = op->d_cws;
      double* out = op->d_cws + 3 * (size_t)d.n;
      if (int rc = cns_sip(C(op), d, coef(k), zero, out)) return rc;
      dbc = out;
    }
    return cns_solve(C(op), d, coef(k), a, rhs, x, op->d_c9, op->d_pinv, dbc);
  }
  Op1DDev d;
  if (int rc = dev_at(op, t, d)) return rc;
  return launch_cg1d(C(op), d, coef(k), a, rhs, x);
}

int sisdc_stage_solve(sisdc_op1d* op, sisdc_coef k, double a, const double* base, const double* conv_in,
                      double dt_m, const double* f_old, int M, const double* w_row, double dt, const double* g_m,
                      const double* h_old, double t_conv, double t_solve, double* rhs_scratch, double* conv_out,
                      double* x) {
  if (!op || !base || !conv_in || !x || M < 0 || M > MAXM || (f_old && !w_row)) return SISDC_ERR_ARG;
  if (int rc = check_coef_op(op, k)) return rc;
  const bool fuse = op->dim == 1 && !op->cns() && !op->parted() && a != 0.0 && k.kind != SISDC_COEF_NONE;
  if (!fuse) {   // stage rhs into the scratch vector, then the solve
    if (!rhs_scratch) return C(op)->fail(SISDC_ERR_ARG, "stage_solve needs a rhs scratch vector here");
    if (int rc = sisdc_stage_rhs(op, base, conv_in, dt_m, f_old, M, w_row, dt, g_m, h_old, t_conv, rhs_scratch,
                                 conv_out))
      return rc;
    return sisdc_implicit_solve(op, k, a, rhs_scratch, t_solve, x);
  }
  Op1DDev d;
  if (int rc = dev_at(op, t_solve, d)) return rc;
  StageFuse sf{};
  sf.base = base; sf.conv_in = conv_in; sf.f_old = f_old; sf.w_row = w_row; sf.g = g_m; sf.h = h_old;
  sf.conv_out = conv_out; sf.dt_m = dt_m; sf.dt = dt; sf.M = M;
  if (int rc = bc_at(op, t_conv, sf.gl, sf.gr)) return rc;
  return launch_cg1d(C(op), d, coef(k), a, nullptr, x, &sf);
}

int sisdc_stage_rhs(sisdc_op1d* op, const double* base, const double* conv_in, double dt_m, const double* f_old,
                    int M, const double* w_row, double dt, const double* g_m, const double* h_old, double t,
                    double* rhs, double* conv_out) {
  if (!op || !base || !conv_in || !rhs || M < 0 || M > MAXM || (f_old && !w_row)) return SISDC_ERR_ARG;
  if (op->parted()) return part2_stage(op, base, conv_in, dt_m, f_old, M, w_row, dt, g_m, h_old, rhs, conv_out);
  if (op->dim == 2) return launch2_stage(C(op), op->dev2, base, conv_in, dt_m, f_old, M, w_row, dt, g_m, h_old, rhs, conv_out);
  if (op->cns()) {
    Op1DDev d;
    if (int rc = dev_at(op, t, d)) return rc;
    return cns_stage(C(op), d, base, conv_in, dt_m, f_old, M, w_row, dt, g_m, h_old, rhs, conv_out);
  }
  Op1DDev d;
  if (int rc = dev_at(op, t, d)) return rc;
  return launch_stage_rhs(C(op), d, base, conv_in, dt_m, f_old, M, w_row, dt, g_m, h_old, rhs, conv_out);
}

int sisdc_node_caches(sisdc_op1d* op, int scheme, int M, int m_first, int m_count, const double* u0,
                      const double* u, const double* conv_prev, const double* dts, double t0, const double* times,
                      double* f, double* h1, double* h2) {
  if (!op || !u0 || !u || !dts || !f || !h1) return SISDC_ERR_ARG;
  if (scheme < SISDC_EULER || scheme > SISDC_SI2) return C(op)->fail(SISDC_ERR_ARG, "unknown scheme");
  if (op->parted()) return part2_eval_nodes(op, 1, scheme, M, m_first, m_count, u0, u, conv_prev, dts, f, h1, h2);
  if (op->dim == 2)
    return launch2_node_eval(C(op), op->dev2, 1, scheme, M, m_first, m_count, u0, u, conv_prev, dts, f, h1, h2);
  if (op->cns()) {
    if (op->dev.bc != SISDC_DIRICHLET)
      return cns_node_eval(C(op), op->dev, 1, scheme, M, m_first, m_count, u0, u, conv_prev, dts, f, h1, h2);
    if (!times) return C(op)->fail(SISDC_ERR_ARG, "Dirichlet node caches need the node times");
    if (M > MAXM) return C(op)->fail(SISDC_ERR_ARG, "too many collocation nodes");
    double bnd[12 * MAXM] = {};
    for (int m = m_first; m < m_first + m_count && m < M; ++m) {
      if (int rc = bc_at3(op, times[m], bnd + 12 * m, bnd + 12 * m + 3)) return rc;
      if (int rc = bc_at3(op, m == 0 ? t0 : times[m - 1], bnd + 12 * m + 6, bnd + 12 * m + 9)) return rc;
    }
    return cns_node_eval(C(op), op->dev, 1, scheme, M, m_first, m_count, u0, u, conv_prev, dts, f, h1, h2, bnd);
  }
  if (op->dev.bc == SISDC_DIRICHLET) {   // boundary data at t_m and t_{m-1} per node
    if (!times) return C(op)->fail(SISDC_ERR_ARG, "Dirichlet node caches need the node times");
    if (M > MAXM) return C(op)->fail(SISDC_ERR_ARG, "too many collocation nodes");
    double bnd[4 * MAXM] = {};
    for (int m = m_first; m < m_first + m_count && m < M; ++m) {
      if (int rc = bc_at(op, times[m], bnd[m], bnd[M + m])) return rc;
      if (int rc = bc_at(op, m == 0 ? t0 : times[m - 1], bnd[2 * M + m], bnd[3 * M + m])) return rc;
    }
    return launch_node_eval(C(op), op->dev, 1, scheme, M, m_first, m_count, u0, u, conv_prev, dts, f, h1, h2, bnd);
  }
  return launch_node_eval(C(op), op->dev, 1, scheme, M, m_first, m_count, u0, u, conv_prev, dts, f, h1, h2);
}

int sisdc_eval_rhs_nodes(sisdc_op1d* op, int M, const double* u, const double* times, double* f) {
  if (!op || !u || !f || M < 1 || M > MAXM) return SISDC_ERR_ARG;
  if (op->parted()) return part2_eval_nodes(op, 0, SISDC_SI2, M, 0, M, u, u, nullptr, nullptr, f, nullptr, nullptr);
  if (op->dim == 2) return launch2_node_eval(C(op), op->dev2, 0, SISDC_SI2, M, 0, M, u, u, nullptr, nullptr, f, nullptr, nullptr);
  if (op->cns()) {
    if (op->dev.bc != SISDC_DIRICHLET)
      return cns_node_eval(C(op), op->dev, 0, SISDC_SI2, M, 0, M, u, u, nullptr, nullptr, f, nullptr, nullptr);
    if (!times) return C(op)->fail(SISDC_ERR_ARG, "Dirichlet evaluations need the node times");
    double bnd[12 * MAXM] = {};
    for (int m = 0; m < M; ++m)
      if (int rc = bc_at3(op, times[m], bnd + 12 * m, bnd + 12 * m + 3)) return rc;
    return cns_node_eval(C(op), op->dev, 0, SISDC_SI2, M, 0, M, u, u, nullptr, nullptr, f, nullptr, nullptr, bnd);
  }
  if (op->dev.bc == SISDC_DIRICHLET) {
    if (!times) return C(op)->fail(SISDC_ERR_ARG, "Dirichlet evaluations need the node times");
    double bnd[4 * MAXM] = {};
    for (int m = 0; m < M; ++m)
      if (int rc = bc_at(op, times[m], bnd[m], bnd[M + m])) return rc;
    return launch_node_eval(C(op), op->dev, 0, SISDC_SI2, M, 0, M, u, u, nullptr, nullptr, f, nullptr, nullptr, bnd);
  }
  return launch_node_eval(C(op), op->dev, 0, SISDC_SI2, M, 0, M, u, u, nullptr, nullptr, f, nullptr, nullptr);
}

int sisdc_collocation_defect(sisdc_op1d* op, int M, const double* W, double dt, int incremental, const double* u0,
                             const double* u, const double* f, double sign, const double* add, double* out) {
  if (!op || !W || !u0 || !u || !f || !out || M < 1 || M > MAXM) return SISDC_ERR_ARG;
  return launch_defect(C(op), (int)op->n(), M, W, dt, incremental, u0, u, f, sign, add, out);
}

// ------------------------------------------------------------ transfers
int sisdc_xfer_create(sisdc_ctx* x, int n_elem, int pc1, int pf1, int Mc, int Mf,
                      const double* It, const double* Pt, const double* Isp, const double* Psp, const double* Rsp,
                      sisdc_xfer** out) {
  if (!x || !It || !Pt || !Isp || !Psp || !out) return SISDC_ERR_ARG;
  *out = nullptr;
  // pf1 up to 2 MAXP1: an h-transfer parent maps to its contiguous pair of children
  if (n_elem < 1 || pc1 < 1 || pf1 < pc1 || pf1 > 2 * MAXP1) return x->c.fail(SISDC_ERR_ARG, "bad element sizes");
  if (Mc < 1 || Mf < Mc || Mf > MAXM) return x->c.fail(SISDC_ERR_ARG, "bad node counts");
  sisdc_xfer* t = new (std::nothrow) sisdc_xfer();
  if (!t) return SISDC_ERR_ARG;
  t->ctx = x;
  XferDev& d = t->dev;
  d.ne = n_elem; d.pc = pc1; d.pf = pf1; d.Mc = Mc; d.Mf = Mf;
  std::vector<double> tab(xo_size(d));
  std::memcpy(tab.data() + xo_It(d), It, Mf * Mc * sizeof(double));
  std::memcpy(tab.data() + xo_Pt(d), Pt, Mf * Mc * sizeof(double));
  std::memcpy(tab.data() + xo_Isp(d), Isp, d.pf * d.pc * sizeof(double));
  std::memcpy(tab.data() + xo_Psp(d), Psp, d.pf * d.pc * sizeof(double));
  for (int i = 0; i < d.pc; ++i)   // restriction: given, or the reference's I_sp^T (transfer.py:243)
    for (int j = 0; j < d.pf; ++j) tab[xo_Rsp(d) + i * d.pf + j] = Rsp ? Rsp[i * d.pf + j] : Isp[j * d.pc + i];
  cudaError_t e = cudaMalloc(&t->d_tab, tab.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(t->d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    int rc = x->c.cuda(e, "xfer tables");
    delete t;
    return rc;
  }
  d.tab = t->d_tab;
  *out = t;
  return SISDC_OK;
}

int sisdc_xfer2d_create(sisdc_ctx* x, int n_elem, int pc1, int pf1, int Mc, int Mf, const double* It,
                        const double* Pt, const double* Isp, const double* Psp, const double* Rsp,
                        sisdc_xfer** out) {
  int rc = sisdc_xfer_create(x, n_elem, pc1, pf1, Mc, Mf, It, Pt, Isp, Psp, Rsp, out);
  if (rc) return rc;
  sisdc_xfer* t = *out;
  t->dim = 2;
  t->dev2.nslab = n_elem; t->dev2.pc = pc1; t->dev2.pf = pf1; t->dev2.Mc = Mc; t->dev2.Mf = Mf;
  t->dev2.tab = t->d_tab;
  return SISDC_OK;
}

void sisdc_xfer_destroy(sisdc_xfer* t) {
  if (!t) return;
  cudaFree(t->d_tab);
  delete t;
}

int sisdc_xfer_spatial(sisdc_xfer* t, int dir, const double* in, double* out) {
  if (!t || !in || !out || dir < 0 || dir > 2) return SISDC_ERR_ARG;
  if (t->dim == 2) return launch2x_spatial(&t->ctx->c, t->dev2, dir, in, out);
  return launch_xfer_spatial(&t->ctx->c, t->dev, dir, in, out);
}

int sisdc_xfer_down(sisdc_xfer* t, int spatial_dir, int temporal_dir, const double* in, double* out) {
  if (!t || !in || !out || spatial_dir < 1 || spatial_dir > 2 || temporal_dir < 1 || temporal_dir > 2)
    return SISDC_ERR_ARG;
  if (t->dim == 2) return launch2x_down(&t->ctx->c, t->dev2, spatial_dir, temporal_dir, in, out);
  return launch_xfer_down(&t->ctx->c, t->dev, spatial_dir, temporal_dir, in, out);
}

int sisdc_xfer_fas_restrict(sisdc_xfer* t, const double* Wf, double dt, int incremental, const double* u0f,
                            const double* uf, const double* ff, const double* gf, double* v, double* rr) {
  if (!t || !Wf || !u0f || !uf || !ff || !v || !rr) return SISDC_ERR_ARG;
  if (t->dim == 2) return launch2x_fas(&t->ctx->c, t->dev2, Wf, dt, incremental, u0f, uf, ff, gf, v, rr);
  return launch_fas_restrict(&t->ctx->c, t->dev, Wf, dt, incremental, u0f, uf, ff, gf, v, rr);
}

int sisdc_xfer_interp(sisdc_xfer* t, int accumulate, const double* uc, const double* vc, double* uf) {
  if (!t || !uc || !uf) return SISDC_ERR_ARG;
  if (t->dim == 2) return launch2x_interp(&t->ctx->c, t->dev2, accumulate, uc, vc, uf);
  return launch_xfer_interp(&t->ctx->c, t->dev, accumulate, uc, vc, uf);
}

}  // extern "C"
