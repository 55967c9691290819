// Geometric multigrid plan for (I - sigma nu Lap_h) u = b  (multigrid.py).
#pragma once
#include <map>
#include <vector>

#include "common.cuh"

namespace pl {

enum Smoother { SM_JACOBI = 0, SM_GS = 1, SM_RB = 2 };
enum SolveStatus { ST_FIXED = 0, ST_CONVERGED = 1, ST_STALLED = 2, ST_DIRECT = 3 };

OpC make_opc(int n, double length, double nu, int order);

struct MgLevel {
  Geo g;
  OpC c;
  int n;
  bool coarsest;     // n <= coarsest_n: dense LU (multigrid.py:240-243)
  double* u = nullptr;
  double* b = nullptr;
  double* t = nullptr;
};

struct LuEntry {
  double* dev = nullptr;   // m*m LU (row-major) followed by m pivots (as doubles)
  double* host = nullptr;  // pinned staging copy
};

struct MgPlan {
  int dim, n, order, smoother, pre, post, coarsest_n;
  double length, nu, omega;
  std::vector<MgLevel> lv;
  int tail_start;          // first level run by the single-CTA tail kernel
  size_t tail_smem;
  int m_lu;                // unknowns on the coarsest grid
  std::map<unsigned long long, LuEntry> lu;
  // ToTolerance norms
  double* partials = nullptr;
  int npartials = 0;
  double* norm_dev = nullptr;    // 2 doubles
  double* norm_host = nullptr;   // pinned, 2 doubles
  char* ws = nullptr;
  size_t ws_bytes = 0;
  // Direct policy (direct.cu): W, W^T, V, V^T, lam on the device, two scratch
  // fields
  double* dir_mats = nullptr;
  double* dir_work = nullptr;
  int dir_ready = 0;
};

size_t mg_workspace_bytes(int dim, int n, int coarsest_n);
int mg_plan_create(MgPlan** out, int dim, int n, double length, double nu, int order,
                   int smoother, double omega, int pre, int post, int coarsest_n, void* ws,
                   size_t ws_bytes);
void mg_plan_destroy(MgPlan* p);
// make sure the coarsest LU for sigma exists (host factorisation + async
// upload); call outside CUDA-graph capture
int mg_prepare(MgPlan* p, double sigma, cudaStream_t s);
// install caller-provided LAPACK getrf factors (row-major LU, 0-based pivots)
int mg_set_coarsest_lu(MgPlan* p, double sigma, const double* lu, const int* piv,
                       cudaStream_t s);
// `count` smoothing sweeps in place on u (multigrid.py:211-234)
int mg_smooth(MgPlan* p, double* u, const double* b, double sigma, int count, cudaStream_t s);
// `ncycles` V-cycles in place on u (multigrid.py:237-251, 265-269);
// zero_guess: u is taken as 0 on entry (and need not be initialised)
int mg_cycles(MgPlan* p, double* u, const double* b, double sigma, int ncycles,
              int zero_guess, cudaStream_t s);
// ToTolerance loop (multigrid.py:270-288), synchronous on s.  Returns 0, or 1
// when the cycle cap is hit (residual/cycles describe the failure).
int mg_solve_tol(MgPlan* p, double* u, const double* b, double sigma, double tol, double stall,
                 int max_cycles, int* cycles, int* status, double* residual, cudaStream_t s);

// Direct policy by fast diagonalisation (direct.cu): install the eigen-
// decomposition T = V diag(lam) V^-1 of the level-0 1-D stencil matrix
// (row-major N x N W = V^-1, W^T, V, V^T and lam, host arrays), then
// u = (I - sigma nu Lap)^-1 b
int mg_set_direct(MgPlan* P, const double* w, const double* wt, const double* v,
                  const double* vt, const double* lam, cudaStream_t s);
int mg_direct(MgPlan* P, double* u, const double* b, double sigma, cudaStream_t s);
void mg_direct_destroy(MgPlan* P);

}  // namespace pl
