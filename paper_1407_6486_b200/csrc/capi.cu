// extern "C" entry points (include/pintlab_b200.h), the SDC sweep and FAS
// orchestration, and the runtime bookkeeping (errors, launch statistics,
// per-kernel CUDA-event timing).
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "../../include/pintlab_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "mg.h"

namespace pl {

// ---------------------------------------------------------------------------
// errors

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return PL_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// launch statistics and per-kind event timing

static std::mutex g_stat_mu;
static long long g_launches[K_NUM_KINDS];
static double g_bytes[K_NUM_KINDS];

void count_launch(int kind, double alg_bytes) {
  std::lock_guard<std::mutex> lk(g_stat_mu);
  g_launches[kind] += 1;
  g_bytes[kind] += alg_bytes;
}

static unsigned g_time_mask = 0;     // kinds whose launches get event pairs
struct EvPair {
  cudaEvent_t a, b;
  double bytes;
  int kind;
};
static std::vector<EvPair> g_ev_pool;
static size_t g_ev_used = 0;
static int g_ev_open = -1;

void timing_pre(int kind, cudaStream_t s) {
  if (!(g_time_mask & (1u << kind))) return;
  if (g_ev_used == g_ev_pool.size()) {
    EvPair p;
    cudaEventCreate(&p.a);
    cudaEventCreate(&p.b);
    p.bytes = 0;
    p.kind = -1;
    g_ev_pool.push_back(p);
  }
  cudaEventRecord(g_ev_pool[g_ev_used].a, s);
  g_ev_open = kind;
}

void timing_post(int kind, cudaStream_t s, double alg_bytes) {
  if (!(g_time_mask & (1u << kind)) || g_ev_open != kind) return;
  cudaEventRecord(g_ev_pool[g_ev_used].b, s);
  g_ev_pool[g_ev_used].bytes = alg_bytes;
  g_ev_pool[g_ev_used].kind = kind;
  ++g_ev_used;
  g_ev_open = -1;
}

static const char* kKindNames[K_NUM_KINDS] = {
    "apply", "jacobi", "jor_rb", "residual", "restrict", "prolong", "mg_tail", "norm",
    "quadrature", "rhs", "residual_max", "fas", "correction_time", "interp_cubic", "copy",
    "lu", "mg_mid", "gauss_seidel", "direct", "apply_rhs"};

// ---------------------------------------------------------------------------
// SDC sweep (sdc.py:84-114)

static Coef coef_from(const double* a, int rows, int cols) {
  Coef c;
  std::memset(&c, 0, sizeof(c));
  c.rows = rows;
  c.cols = cols;
  std::memcpy(c.a, a, sizeof(double) * rows * cols);
  return c;
}

static int sdc_sweep(MgPlan* P, const pl_sweep_desc* d, double* Y, double* F, const double* y0,
                     const double* tau, double dt, double* ws, size_t ws_bytes, int* cycles,
                     int* sub_cycles, int* sub_status, int* failed, double* fres, int* fcyc,
                     cudaStream_t s) {
  const MgLevel& L = P->lv[0];
  const long long np = L.g.nstore;     // field stride / point-wise extent
  const int M = d->m;
  if (M < 1 || M + 1 > PL_MAX_NODES) {
    set_error("sweep needs 1 <= M <= %d", PL_MAX_NODES - 1);
    return PL_ERR_ARG;
  }
  if (ws_bytes < sizeof(double) * (size_t)np * (M + 1)) {
    set_error("sweep workspace too small");
    return PL_ERR_ARG;
  }
  double* S = ws;                       // M node-to-node integrals
  double* R = ws + (size_t)M * np;      // right-hand side
  // sigma of every sub-step: float(gamma_m) * dt  (sdc.py:101)
  std::vector<double> dtm(M);
  for (int m = 0; m < M; ++m) {
    dtm[m] = d->gammas[m] * dt;
    PL_TRY(mg_prepare(P, dtm[m], s));
  }
  // s = dt * tensordot(Q[1:] - Q[:-1], F)   (sdc.py:95)
  Coef qd = coef_from(d->qdelta, M, M + 1);
  PL_TRY(launch_chain(F, np, S, np, qd, dt, np, s));
  // y[0] = y0 ; f[0] = A y0   (sdc.py:96-97)
  if (Y != y0) {
    cudaError_t e = cudaMemcpyAsync(Y, y0, sizeof(double) * np, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "y0 copy");
    count_launch(K_COPY, 16.0 * L.g.npts);
  }
  // f[m] = A y[m] fused with the right-hand side of sub-step m (sdc.py:102-104,
  // 112): both read y[m]; rhs reads the OLD f[m+1], which the fusion leaves alone
  auto refresh_rhs = [&](int m) {
    return launch_apply_rhs(Y + (size_t)m * np, F + (size_t)m * np, F + (size_t)(m + 1) * np,
                            S + (size_t)m * np, tau ? tau + (size_t)m * np : nullptr,
                            tau ? tau + (size_t)(m + 1) * np : nullptr, dtm[m], R, np, L.g,
                            L.c, s);
  };
  PL_TRY(refresh_rhs(0));
  int total = 0;
  for (int m = 0; m < M; ++m) {
    double* ym1 = Y + (size_t)(m + 1) * np;
    if (d->policy == 0) {
      PL_TRY(mg_cycles(P, ym1, R, dtm[m], d->fixed_cycles, 0, s));
      total += d->fixed_cycles;
      if (sub_cycles) sub_cycles[m] = d->fixed_cycles;
      if (sub_status) sub_status[m] = PL_STATUS_FIXED;
    } else if (d->policy == 2) {      // Direct: 0 cycles (multigrid.py:263-264)
      PL_TRY(mg_direct(P, ym1, R, dtm[m], s));
      if (sub_cycles) sub_cycles[m] = 0;
      if (sub_status) sub_status[m] = PL_STATUS_DIRECT;
    } else {
      int c = 0, st = 0;
      double res = 0;
      int rc = mg_solve_tol(P, ym1, R, dtm[m], d->tol, d->stall, d->max_cycles, &c, &st, &res, s);
      if (rc == PL_ERR_MGCAP) {
        *failed = m + 1;
        *fres = res;
        *fcyc = c;
        *cycles = total;
        return rc;
      }
      if (rc) return rc;
      total += c;
      if (sub_cycles) sub_cycles[m] = c;
      if (sub_status) sub_status[m] = st;
    }
    if (m + 1 < M) PL_TRY(refresh_rhs(m + 1));
    else PL_TRY(launch_apply(ym1, F + (size_t)(m + 1) * np, L.g, L.c, s));   // sdc.py:112
  }
  *cycles = total;
  return 0;
}

// ---------------------------------------------------------------------------
// FAS (hierarchy.py:85-122)

static int restrict_field(const double* f, double* c, const Geo& gf, int kind, cudaStream_t s) {
  if (kind == PL_RESTRICT_FULL_WEIGHTING) return launch_fw(f, c, gf, s);
  if (kind == PL_RESTRICT_INJECT) return launch_inject(f, c, gf, s);
  cudaError_t e = cudaMemcpyAsync(c, f, sizeof(double) * gf.nstore, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "copy");
  count_launch(K_COPY, 16.0 * gf.npts);
  return 0;
}

}  // namespace pl

using namespace pl;

static bool check_grid(int dim, int n) {
  if (dim < 1 || dim > 3 || n < 2 || (n & (n - 1))) {
    set_error("bad grid dim=%d n=%d", dim, n);
    return false;
  }
  return true;
}

namespace {
template <int DIM>
__global__ void k_diag(double* out, Geo g, OpC c, double sigma, int shifted) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.npts) return;
  int x, y, z;
  decode_point(g, t, x, y, z);
  const long long p = g.at(x, y, z);
  if (shifted) {
    out[p] = shifted_diag<DIM>(g, c, sigma, x, y, z);
  } else {
    double t = 0.0;
    if (DIM == 3) t = t + ((c.order == 4 && (z == 0 || z == g.nz - 1)) ? c.d1_edge : c.d1_int);
    if (DIM >= 2) t = t + ((c.order == 4 && (y == 0 || y == g.ny - 1)) ? c.d1_edge : c.d1_int);
    t = t + ((c.order == 4 && (x == 0 || x == g.nx - 1)) ? c.d1_edge : c.d1_int);
    out[p] = c.nu * t;
  }
}
template <int DIM>
__global__ void k_shifted_apply(const double* __restrict__ u, double* __restrict__ out, Geo g,
                                OpC c, double sigma) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.npts) return;
  int x, y, z;
  decode_point(g, t, x, y, z);
  const long long p = g.at(x, y, z);
  out[p] = shifted_point<DIM>(u, g, c, sigma, x, y, z, p);
}
}  // namespace

extern "C" int g_graphs_enabled;

namespace pl {
extern int g_zmarch_enabled;
extern int g_zmarch_min_n;
extern int g_fuse_prolong;
extern int g_mid_enabled;
extern int g_mid_tail_n;
extern int g_rfw_enabled;
extern int g_zc_floor;
extern int g_zc_ctas;
extern int g_zc_fit;
extern int g_tol_device;
extern int g_fast_tail;
extern int g_mid_ctas;
extern int g_zrb_ring;
extern int g_zrev_mask;
}

extern "C" {

int pl_abi_version(void) { return PL_ABI_VERSION; }

static int set_option_impl(int key, int value);
// every option value accepted so far (INT_MIN: library default); part of the
// CUDA-graph key, so a sweep captured under other options never replays
static const int kMaxOptions = 64;
static std::vector<int> g_opt_values(kMaxOptions, INT_MIN);
static void drop_sweep_graphs(const void* plan);

int pl_set_option(int key, int value) {
  int rc = set_option_impl(key, value);
  if (rc == 0 && key >= 0 && key < kMaxOptions) {
    std::lock_guard<std::mutex> lk(g_stat_mu);
    g_opt_values[key] = value;
  }
  return rc;
}

static int set_option_impl(int key, int value) {
  if (key == PL_OPT_ZMARCH) {
    g_zmarch_enabled = value != 0;
    return 0;
  }
  if (key == PL_OPT_GRAPHS) {
    g_graphs_enabled = value != 0;
    return 0;
  }
  if (key == PL_OPT_ZC_CTAS) {
    if (value < 1) {
      set_error("CTA target must be positive");
      return PL_ERR_ARG;
    }
    g_zc_ctas = value;
    return 0;
  }
  if (key == PL_OPT_TOL_DEVICE) {
    g_tol_device = value != 0;
    return 0;
  }
  if (key == PL_OPT_ZC_FIT) {
    g_zc_fit = value != 0;
    return 0;
  }
  if (key == PL_OPT_FAST_TAIL) {
    g_fast_tail = value != 0;
    return 0;
  }
  if (key == PL_OPT_ZC_FLOOR) {
    if (value < 2 || (value & (value - 1))) {
      set_error("z chunk floor must be a power of two >= 2");
      return PL_ERR_ARG;
    }
    g_zc_floor = value;
    return 0;
  }
  if (key == PL_OPT_RFW) {
    g_rfw_enabled = value != 0;
    return 0;
  }
  if (key == PL_OPT_MID) {
    g_mid_enabled = value != 0;
    return 0;
  }
  if (key == PL_OPT_MID_CTAS) {
    if (value < 0) {
      set_error("mid CTA count must be >= 0");
      return PL_ERR_ARG;
    }
    g_mid_ctas = value;
    return 0;
  }
  if (key == PL_OPT_ZRB_RING) {
    if (value != 0 && value != 1 && value != 4) {
      set_error("zrb ring variant %d must be 0, 1 or 4", value);
      return PL_ERR_ARG;
    }
    g_zrb_ring = value;
    return 0;
  }
  if (key == PL_OPT_MID_TAIL_N) {
    g_mid_tail_n = value;
    return 0;
  }
  if (key == PL_OPT_FUSE_PROLONG) {
    g_fuse_prolong = value != 0;
    return 0;
  }
  if (key == PL_OPT_FUSE_FAS_FW) {
    g_fuse_fas_fw = value != 0;
    return 0;
  }
  if (key == PL_OPT_ZREV) {
    g_zrev_mask = value;
    return 0;
  }
  if (key == PL_OPT_FUSE_APPLY_RHS) {
    g_fuse_apply_rhs = value != 0;
    return 0;
  }
  if (key == PL_OPT_ZMARCH_MIN_N) {
    g_zmarch_min_n = value < 31 ? 31 : value;
    return 0;
  }
  set_error("unknown option %d", key);
  return PL_ERR_ARG;
}
const char* pl_last_error(void) { return g_err; }

int pl_heat_apply(const double* u, double* f, int dim, int n, double length, double nu,
                  int order, void* stream) {
  if (!check_grid(dim, n)) return PL_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  return launch_apply(u, f, make_geo(dim, n), make_opc(n, length, nu, order), s);
}


int pl_heat_diagonal(double* out, int dim, int n, double length, double nu, int order,
                     double sigma, int shifted, void* stream) {
  if (!check_grid(dim, n)) return PL_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  Geo g = make_geo(dim, n);
  OpC c = make_opc(n, length, nu, order);
  int blocks = ceil_div(g.npts, 256);
  PL_PRE(K_APPLY);
  if (dim == 1) k_diag<1><<<blocks, 256, 0, s>>>(out, g, c, sigma, shifted);
  else if (dim == 2) k_diag<2><<<blocks, 256, 0, s>>>(out, g, c, sigma, shifted);
  else k_diag<3><<<blocks, 256, 0, s>>>(out, g, c, sigma, shifted);
  PL_CHECK_LAUNCH(K_APPLY, 8.0 * g.npts);
  return 0;
}

int pl_shifted_apply(const double* u, double* out, int dim, int n, double length, double nu,
                     int order, double sigma, void* stream) {
  if (!check_grid(dim, n)) return PL_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  Geo g = make_geo(dim, n);
  OpC c = make_opc(n, length, nu, order);
  int blocks = ceil_div(g.npts, 256);
  PL_PRE(K_APPLY);
  if (dim == 1) k_shifted_apply<1><<<blocks, 256, 0, s>>>(u, out, g, c, sigma);
  else if (dim == 2) k_shifted_apply<2><<<blocks, 256, 0, s>>>(u, out, g, c, sigma);
  else k_shifted_apply<3><<<blocks, 256, 0, s>>>(u, out, g, c, sigma);
  PL_CHECK_LAUNCH(K_APPLY, 16.0 * g.npts);
  return 0;
}

int pl_full_weighting(const double* fine, double* coarse, int dim, int nf, void* stream) {
  if (!check_grid(dim, nf) || nf < 4) return PL_ERR_ARG;
  return launch_fw(fine, coarse, make_geo(dim, nf), (cudaStream_t)stream);
}

int pl_inject(const double* fine, double* coarse, int dim, int nf, void* stream) {
  if (!check_grid(dim, nf) || nf < 4) return PL_ERR_ARG;
  return launch_inject(fine, coarse, make_geo(dim, nf), (cudaStream_t)stream);
}

int pl_interp_linear(const double* coarse, double* fine, int dim, int nf, int accumulate,
                     void* stream) {
  if (!check_grid(dim, nf) || nf < 4) return PL_ERR_ARG;
  return launch_prolong(coarse, fine, make_geo(dim, nf), accumulate, (cudaStream_t)stream);
}

size_t pl_interp_cubic_scratch_bytes(int dim, int nf) {
  if (!check_grid(dim, nf) || nf < 4) return 0;
  return sizeof(double) * (size_t)cubic_scratch_doubles(make_geo(dim, nf));
}

int pl_interp_cubic(const double* coarse, double* fine, int dim, int nf, int accumulate,
                    double* scratch, void* stream) {
  if (!check_grid(dim, nf) || nf < 4) return PL_ERR_ARG;
  return launch_cubic(coarse, fine, make_geo(dim, nf), accumulate, scratch,
                      (cudaStream_t)stream);
}

size_t pl_mg_workspace_bytes(int dim, int n, int coarsest_n) {
  if (!check_grid(dim, n)) return 0;
  return mg_workspace_bytes(dim, n, coarsest_n);
}

int pl_mg_plan_create(pl_mg_plan** plan, int dim, int n, double length, double nu, int order,
                      int smoother, double omega, int pre_sweeps, int post_sweeps,
                      int coarsest_n, void* workspace, size_t workspace_bytes) {
  MgPlan* P = nullptr;
  int rc = mg_plan_create(&P, dim, n, length, nu, order, smoother, omega, pre_sweeps,
                          post_sweeps, coarsest_n, workspace, workspace_bytes);
  if (rc) return rc;
  *plan = (pl_mg_plan*)P;
  return 0;
}

int pl_mg_plan_destroy(pl_mg_plan* plan) {
  drop_sweep_graphs(plan);   // a recycled plan address must never replay a stale graph
  mg_plan_destroy((MgPlan*)plan);
  return 0;
}

int pl_mg_prepare(pl_mg_plan* plan, double sigma, void* stream) {
  return mg_prepare((MgPlan*)plan, sigma, (cudaStream_t)stream);
}

int pl_mg_set_coarsest_lu(pl_mg_plan* plan, double sigma, const double* lu, const int* piv,
                          void* stream) {
  return mg_set_coarsest_lu((MgPlan*)plan, sigma, lu, piv, (cudaStream_t)stream);
}

int pl_mg_coarsest_size(pl_mg_plan* plan) { return ((MgPlan*)plan)->m_lu; }

int pl_mg_set_direct(pl_mg_plan* plan, const double* w, const double* wt, const double* v,
                     const double* vt, const double* lam, void* stream) {
  return mg_set_direct((MgPlan*)plan, w, wt, v, vt, lam, (cudaStream_t)stream);
}

int pl_mg_direct(pl_mg_plan* plan, double* u, const double* b, double sigma, void* stream) {
  return mg_direct((MgPlan*)plan, u, b, sigma, (cudaStream_t)stream);
}

int pl_mg_smooth(pl_mg_plan* plan, double* u, const double* b, double sigma, int count,
                 void* stream) {
  if (count < 0) return PL_ERR_ARG;
  return mg_smooth((MgPlan*)plan, u, b, sigma, count, (cudaStream_t)stream);
}

int pl_mg_vcycles(pl_mg_plan* plan, double* u, const double* b, double sigma, int ncycles,
                  int zero_guess, void* stream) {
  if (ncycles < 1) {
    set_error("need at least one V-cycle");
    return PL_ERR_ARG;
  }
  return mg_cycles((MgPlan*)plan, u, b, sigma, ncycles, zero_guess, (cudaStream_t)stream);
}

int pl_mg_solve_tol(pl_mg_plan* plan, double* u, const double* b, double sigma, double tol,
                    double stall, int max_cycles, int* cycles, int* status, double* residual,
                    void* stream) {
  return mg_solve_tol((MgPlan*)plan, u, b, sigma, tol, stall, max_cycles, cycles, status,
                      residual, (cudaStream_t)stream);
}

long long pl_field_elems(int dim, int n) {
  if (!check_grid(dim, n)) return 0;
  return make_geo(dim, n).nstore;
}

size_t pl_sweep_workspace_bytes(int dim, int n, int m) {
  if (!check_grid(dim, n)) return 0;
  return sizeof(double) * (size_t)make_geo(dim, n).nstore * (m + 1);
}

// ---- CUDA-graph replay of FixedCycles sweeps -----------------------------
// A FixedCycles sweep is a fixed sequence of ~30 M launches for given buffers;
// the second call with the same (plan, buffers, dt, coefficients) captures it
// on a private stream and every later call replays it with one graph launch.
// Launch statistics recorded during capture are re-applied per replay.

struct SweepKey {
  const void *plan, *Y, *F, *y0, *tau, *ws;
  unsigned long long dt;
  std::vector<int> opts;
  std::vector<double> coef;
  bool operator<(const SweepKey& o) const {
    return std::tie(plan, Y, F, y0, tau, ws, dt, opts, coef) <
           std::tie(o.plan, o.Y, o.F, o.y0, o.tau, o.ws, o.dt, o.opts, o.coef);
  }
};
struct SweepGraph {
  int seen = 0;
  cudaGraphExec_t exec = nullptr;
  long long launches[K_NUM_KINDS];
  double bytes[K_NUM_KINDS];
};
// Bounded: a PFASST run uses one entry per (rank stream, level) buffer set;
// past kMaxSweepGraphs the whole cache is dropped and recaptured on demand.
static const size_t kMaxSweepGraphs = 512;
static std::map<SweepKey, SweepGraph> g_sweep_graphs;
static std::mutex g_graph_mu;
static cudaStream_t g_capture_stream = nullptr;
int g_graphs_enabled = 1;

// destroy the captured sweeps of one plan (plan != NULL) or all of them;
// callers must not hold g_graph_mu
static void drop_sweep_graphs(const void* plan) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (auto it = g_sweep_graphs.begin(); it != g_sweep_graphs.end();) {
    if (plan && it->first.plan != plan) {
      ++it;
      continue;
    }
    if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
    it = g_sweep_graphs.erase(it);
  }
}

static void add_graph_stats(const SweepGraph& G) {
  std::lock_guard<std::mutex> lk2(g_stat_mu);
  for (int i = 0; i < K_NUM_KINDS; ++i) {
    g_launches[i] += G.launches[i];
    g_bytes[i] += G.bytes[i];
  }
}

static void fixed_log(const pl_sweep_desc* d, int* sub_cycles, int* sub_status) {
  for (int m = 0; m < d->m; ++m) {
    if (sub_cycles) sub_cycles[m] = d->fixed_cycles;
    if (sub_status) sub_status[m] = PL_STATUS_FIXED;
  }
}

static int sweep_graphed(MgPlan* P, const pl_sweep_desc* d, double* Y, double* F,
                         const double* y0, const double* tau, double dt, double* ws,
                         size_t ws_bytes, int* cycles, int* sub_cycles, int* sub_status,
                         int* failed, double* fres, int* fcyc, cudaStream_t s) {
  SweepKey k{P, Y, F, y0, tau, ws, 0, {}, {}};
  {
    std::lock_guard<std::mutex> lk0(g_stat_mu);
    k.opts = g_opt_values;
  }
  std::memcpy(&k.dt, &dt, sizeof(dt));
  k.coef.assign(d->qdelta, d->qdelta + d->m * (d->m + 1));
  k.coef.insert(k.coef.end(), d->gammas, d->gammas + d->m);
  k.coef.push_back((double)d->fixed_cycles);
  std::unique_lock<std::mutex> lk(g_graph_mu);
  if (g_sweep_graphs.size() >= kMaxSweepGraphs && !g_sweep_graphs.count(k)) {
    lk.unlock();
    drop_sweep_graphs(nullptr);
    lk.lock();
  }
  SweepGraph& G = g_sweep_graphs[k];
  if (G.exec) {
    cudaError_t e = cudaGraphLaunch(G.exec, s);
    if (e != cudaSuccess) return cuda_status(e, "graph launch");
    add_graph_stats(G);
    *cycles = d->m * d->fixed_cycles;
    fixed_log(d, sub_cycles, sub_status);
    return 0;
  }
  if (++G.seen < 2)   // first use runs eagerly (lazy initialisation happens here)
    return sdc_sweep(P, d, Y, F, y0, tau, dt, ws, ws_bytes, cycles, sub_cycles, sub_status,
                     failed, fres, fcyc, s);
  cudaError_t e;
  if (!g_capture_stream) {
    e = cudaStreamCreateWithFlags(&g_capture_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_status(e, "capture stream");
  }
  long long l0[K_NUM_KINDS];
  double b0[K_NUM_KINDS];
  {
    std::lock_guard<std::mutex> lk2(g_stat_mu);
    std::memcpy(l0, g_launches, sizeof(l0));
    std::memcpy(b0, g_bytes, sizeof(b0));
  }
  cudaStream_t cs = g_capture_stream;
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_status(e, "begin capture");
  int rc = sdc_sweep(P, d, Y, F, y0, tau, dt, ws, ws_bytes, cycles, sub_cycles, sub_status,
                     failed, fres, fcyc, cs);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(cs, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return cuda_status(e, "end capture");
  e = cudaGraphInstantiate(&G.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    G.exec = nullptr;
    return cuda_status(e, "graph instantiate");
  }
  {
    std::lock_guard<std::mutex> lk2(g_stat_mu);
    for (int i = 0; i < K_NUM_KINDS; ++i) {
      G.launches[i] = g_launches[i] - l0[i];
      G.bytes[i] = g_bytes[i] - b0[i];
      g_launches[i] = l0[i];
      g_bytes[i] = b0[i];
    }
  }
  // the capture stream is empty: order the replay after prior work on s
  e = cudaGraphLaunch(G.exec, s);
  if (e != cudaSuccess) return cuda_status(e, "graph launch");
  add_graph_stats(G);
  return 0;
}

int pl_sdc_sweep(pl_mg_plan* plan, const pl_sweep_desc* desc, double* Y, double* F,
                 const double* y0, const double* tau, double dt, void* workspace,
                 size_t workspace_bytes, int* cycles, int* substep_cycles, int* substep_status,
                 int* failed_substep, double* fail_residual, int* fail_cycles, void* stream) {
  *failed_substep = 0;
  // per-launch event timing needs eager launches; ToTolerance syncs per solve
  if (g_graphs_enabled && desc->policy == 0 && g_time_mask == 0)
    return sweep_graphed((MgPlan*)plan, desc, Y, F, y0, tau, dt, (double*)workspace,
                         workspace_bytes, cycles, substep_cycles, substep_status, failed_substep,
                         fail_residual, fail_cycles, (cudaStream_t)stream);
  return sdc_sweep((MgPlan*)plan, desc, Y, F, y0, tau, dt, (double*)workspace, workspace_bytes,
                   cycles, substep_cycles, substep_status, failed_substep, fail_residual,
                   fail_cycles, (cudaStream_t)stream);
}

int pl_sdc_residual(const double* Y, const double* F, const double* y0, const double* tau,
                    const double* q, int m, double dt, int dim, int n, double* out_dev,
                    void* stream) {
  if (m < 1 || m + 1 > PL_MAX_NODES || !check_grid(dim, n)) return PL_ERR_ARG;
  Coef c = coef_from(q, m + 1, m + 1);
  const long long ns = make_geo(dim, n).nstore;
  return launch_resmax(Y, F, ns, y0, tau, c, dt, ns, out_dev, (cudaStream_t)stream);
}

int pl_restrict_state(const double* fineY, const int* idx, int nsel, double* coarseY,
                      double* coarseF, int dim, int nf, int nc, int restrict_kind,
                      double length, double nu_c, int order_c, void* stream) {
  if (!check_grid(dim, nf) || !check_grid(dim, nc)) return PL_ERR_ARG;
  if (nc == nf) restrict_kind = PL_RESTRICT_COPY;
  else if (nc * 2 != nf) {
    set_error("coarse n must equal fine n or half of it");
    return PL_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  Geo gf = make_geo(dim, nf), gc = make_geo(dim, nc);
  OpC cc = make_opc(nc, length, nu_c, order_c);
  // 3-D full weighting from 127^3 up: every selected node in one tiled launch
  const bool batched = restrict_kind == PL_RESTRICT_FULL_WEIGHTING && fw_select_ok(gf, nsel);
  if (batched) PL_TRY(launch_fw_select(fineY, gf.nstore, idx, nsel, coarseY, gc.nstore, gf, s));
  for (int j = 0; j < nsel; ++j) {
    double* cy = coarseY + (size_t)j * gc.nstore;
    if (!batched)
      PL_TRY(restrict_field(fineY + (size_t)idx[j] * gf.nstore, cy, gf, restrict_kind, s));
    PL_TRY(launch_apply(cy, coarseF + (size_t)j * gc.nstore, gc, cc, s));
  }
  return 0;
}

size_t pl_compute_fas_scratch_bytes(int dim, int nf, int nsel) {
  if (!check_grid(dim, nf)) return 0;
  return sizeof(double) * (size_t)make_geo(dim, nf).nstore * nsel;
}

int pl_compute_fas(const double* fineF, const double* fine_tau, int mf, const double* qf_rows,
                   const int* idx, int nsel, const double* coarseF, const double* qc, int mc,
                   double dt, double* tau_c, double* scratch, int dim, int nf, int nc,
                   int restrict_kind, void* stream) {
  if (!check_grid(dim, nf) || !check_grid(dim, nc)) return PL_ERR_ARG;
  if (mf + 1 > PL_MAX_NODES || mc + 1 > PL_MAX_NODES || nsel != mc + 1) return PL_ERR_ARG;
  if (nc == nf) restrict_kind = PL_RESTRICT_COPY;
  cudaStream_t s = (cudaStream_t)stream;
  Geo gf = make_geo(dim, nf), gc = make_geo(dim, nc);
  // fine integrals at the selected nodes: dt * (Q_f F_f)[idx] (+ tau_f[idx])
  Coef qf = coef_from(qf_rows, nsel, mf + 1);
  if (restrict_kind == PL_RESTRICT_FULL_WEIGHTING && chain_fw_ok(qf, gf)) {
    // integrals and full weighting in one pass: the fine integrals are never stored
    PL_TRY(launch_chain_fw(fineF, gf.nstore, qf, dt, fine_tau, gf.nstore, idx, tau_c, gc.nstore,
                           gf, s));
  } else {
    PL_TRY(launch_chain_ex(fineF, gf.nstore, scratch, gf.nstore, qf, dt, gf.nstore, fine_tau,
                           gf.nstore, idx, fine_tau ? 1 : 0, s));
    // restrict each into tau_c (temporarily)
    for (int j = 0; j < nsel; ++j)
      PL_TRY(restrict_field(scratch + (size_t)j * gf.nstore, tau_c + (size_t)j * gc.nstore, gf,
                            restrict_kind, s));
  }
  // then tau_c = R - dt (Q_c F_c)
  Coef q = coef_from(qc, mc + 1, mc + 1);
  PL_TRY(launch_chain_ex(coarseF, gc.nstore, tau_c, gc.nstore, q, dt, gc.nstore, tau_c,
                         gc.nstore, nullptr, 2, s));
  return 0;
}

size_t pl_coarse_correction_scratch_bytes(int dim, int nf, int nc, int mf, int interp_order) {
  if (!check_grid(dim, nf) || !check_grid(dim, nc)) return 0;
  size_t n = (size_t)make_geo(dim, nc).nstore * (mf + 1);
  if (nc != nf && interp_order == 4) n += cubic_scratch_doubles(make_geo(dim, nf));
  return sizeof(double) * n;
}

int pl_coarse_correction(double* fineY, double* fineF, int mf, const double* coarse_new,
                         const double* coarse_old, int mc, const double* pt, int dim, int nf,
                         int nc, int interp_order, double length, double nu_f, int order_f,
                         double* scratch, void* stream) {
  if (!check_grid(dim, nf) || !check_grid(dim, nc)) return PL_ERR_ARG;
  if (mf + 1 > PL_MAX_NODES || mc + 1 > PL_MAX_NODES) return PL_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  Geo gf = make_geo(dim, nf), gc = make_geo(dim, nc);
  OpC cf = make_opc(nf, length, nu_f, order_f);
  Coef p = coef_from(pt, mf + 1, mc + 1);
  double* dt_fields = scratch;   // (Mf+1) coarse fields
  PL_TRY(launch_delta_chain(coarse_new, coarse_old, gc.nstore, p, dt_fields, gc.nstore, gc.nstore,
                            s));
  double* cub = scratch + (size_t)gc.nstore * (mf + 1);
  for (int m = 0; m <= mf; ++m) {
    double* y = fineY + (size_t)m * gf.nstore;
    const double* d = dt_fields + (size_t)m * gc.nstore;
    if (nc == nf) {
      PL_TRY(launch_axpby(y, d, y, 0, gf.nstore, s));
    } else if (interp_order == 2) {
      PL_TRY(launch_prolong(d, y, gf, 1, s));
    } else {
      PL_TRY(launch_cubic(d, y, gf, 1, cub, s));
    }
    PL_TRY(launch_apply(y, fineF + (size_t)m * gf.nstore, gf, cf, s));
  }
  return 0;
}

int pl_stats_reset(void) {
  std::lock_guard<std::mutex> lk(g_stat_mu);
  for (int k = 0; k < K_NUM_KINDS; ++k) {
    g_launches[k] = 0;
    g_bytes[k] = 0;
  }
  return 0;
}

int pl_stats_get(long long* launches, double* alg_bytes, int nkinds) {
  std::lock_guard<std::mutex> lk(g_stat_mu);
  for (int k = 0; k < nkinds && k < K_NUM_KINDS; ++k) {
    launches[k] = g_launches[k];
    alg_bytes[k] = g_bytes[k];
  }
  return 0;
}

int pl_timing_enable(unsigned mask) {
  g_time_mask = mask;
  g_ev_used = 0;
  g_ev_open = -1;
  return 0;
}

int pl_timing_collect(int kind, long long* launches, double* total_ms, double* alg_bytes) {
  double t = 0, b = 0;
  long long n = 0;
  for (size_t i = 0; i < g_ev_used; ++i) {
    if (g_ev_pool[i].kind != kind) continue;
    cudaError_t e = cudaEventSynchronize(g_ev_pool[i].b);
    if (e != cudaSuccess) return cuda_status(e, "event sync");
    float ms = 0;
    cudaEventElapsedTime(&ms, g_ev_pool[i].a, g_ev_pool[i].b);
    t += ms;
    b += g_ev_pool[i].bytes;
    ++n;
  }
  *launches = n;
  *total_ms = t;
  *alg_bytes = b;
  return 0;
}

int pl_timing_dump(int kind, long long nmax, double* bytes, float* ms, long long* n) {
  long long c = 0;
  for (size_t i = 0; i < g_ev_used && c < nmax; ++i) {
    if (g_ev_pool[i].kind != kind) continue;
    cudaError_t e = cudaEventSynchronize(g_ev_pool[i].b);
    if (e != cudaSuccess) return cuda_status(e, "event sync");
    cudaEventElapsedTime(&ms[c], g_ev_pool[i].a, g_ev_pool[i].b);
    bytes[c] = g_ev_pool[i].bytes;
    ++c;
  }
  *n = c;
  return 0;
}

const char* pl_kind_name(int kind) {
  return (kind >= 0 && kind < K_NUM_KINDS) ? kKindNames[kind] : "?";
}

}  // extern "C"
