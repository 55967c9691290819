/*
 * pintlab_b200.h -- C ABI of the B200 (sm_100a) PFASST x multigrid hot path.
 *
 * This is the drop-in boundary for the reference package `pintlab`
 * (/root/reference/pkg/src/pintlab).  The reference is pure Python/numpy and
 * exposes no FFI of its own; each entry point below replaces one reference
 * function on the hot path (cited file:line), and the Python package
 * `paper_1407_6486_b200` binds them with ctypes behind the reference's own
 * class/function names.
 *
 * Conventions
 *  - All arrays are fp64, C order, interior points only, x fastest
 *    (heat.py:1-6): a grid with n cells per axis holds (n-1)^dim values.
 *    Device layout: for dim >= 2 each x-row of n-1 values is stored with a
 *    pitch of n doubles (one zero pad per row, 16-byte aligned rows for TMA);
 *    1-D fields are one unpadded row.  pl_field_elems(dim, n) is the storage
 *    size of one field; nodal arrays (M+1 fields) are contiguous with that
 *    stride.  Pads must hold zeros.
 *  - Device buffers are allocated and owned by the caller; the library owns
 *    only plans (level descriptors, coarsest-grid LU factors, norm scratch).
 *  - Every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) unless documented as synchronous.
 *  - Return status: PL_OK, PL_ERR_MGCAP (ToTolerance cycle cap, maps to
 *    MultigridError / SubStepError), PL_ERR_CUDA, or a negative argument /
 *    support error (ValueError / NotImplementedError).  pl_last_error()
 *    returns the message of the last failure on this process.
 */
#ifndef PINTLAB_B200_H
#define PINTLAB_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PL_ABI_VERSION 2

#define PL_OK 0
#define PL_ERR_MGCAP 1
#define PL_ERR_CUDA 2
#define PL_ERR_ARG (-1)
#define PL_ERR_UNSUPPORTED (-2)
#define PL_ERR_STATE (-3)

/* smoother kinds (multigrid.py:26) */
#define PL_SMOOTHER_JACOBI 0
#define PL_SMOOTHER_GAUSS_SEIDEL 1 /* lexicographic, hyperplane wavefront (gs.cu) */
#define PL_SMOOTHER_JOR_RB 2

/* solve status (multigrid.py:258) */
#define PL_STATUS_FIXED 0
#define PL_STATUS_CONVERGED 1
#define PL_STATUS_STALLED 2
#define PL_STATUS_DIRECT 3

/* spatial restriction kinds (hierarchy.py:34, 66-71) */
#define PL_RESTRICT_FULL_WEIGHTING 0
#define PL_RESTRICT_INJECT 1
#define PL_RESTRICT_COPY 2 /* coarse level with the same n */

typedef struct pl_mg_plan pl_mg_plan;

int pl_abi_version(void);
const char* pl_last_error(void);

/* runtime options (A/B testing of kernel variants; results are bit-identical).
   Keys 3, 5, 12, 15, 16, 18 and 21 belonged to removed variants and are
   rejected. */
#define PL_OPT_ZMARCH 0       /* 1 (default): TMA z-marching + fused sweeps, 3-D order 2 */
#define PL_OPT_ZMARCH_MIN_N 1 /* smallest n-1 using them (default 127, >= 31) */
#define PL_OPT_GRAPHS 2       /* 1 (default): FixedCycles sweeps replay as CUDA graphs */
#define PL_OPT_FUSE_PROLONG 4 /* 1: prolongation fused into the first Jacobi post-sweep pair (TMA levels);
                                 default 0 (separate per-cell prolongation is faster) */
#define PL_OPT_MID 6          /* 1 (default): V-cycle levels below the TMA threshold and the tail
                                 run as one cooperative launch (3-D order-2 jor-rb) */
#define PL_OPT_MID_TAIL_N 7   /* largest n-1 the cooperative kernel leaves to its one-CTA tail
                                 (default 15) */
#define PL_OPT_RFW 8          /* 1 (default): residual + full weighting fused (TMA levels) */
#define PL_OPT_ZC_FLOOR 9     /* smallest z-chunk of the TMA kernels (power of two, default 16) */
#define PL_OPT_FAST_TAIL 10   /* 1 (default): compile-time-sized 15^3/7^3 -> 3^3 jor-rb tail */
#define PL_OPT_ZC_CTAS 11     /* CTA count the TMA kernels' z chunking aims for (default 1184) */
#define PL_OPT_MID_CTAS 13    /* CTAs of the cooperative small-level kernels (0, default: one per
                                 SM); pfasst_run's rank-stream schedule sets 32 for its duration
                                 so the other ranks' streams keep the remaining SMs */
#define PL_OPT_ZRB_RING 14    /* fused jor-rb sweep rings: 0 (default) 6 u + 3 b planes,
                                 4 CTAs/SM, z chunks >= 32 from 255^3 up, else 8 u + 4 b planes,
                                 3 CTAs/SM; 1: always 6 + 3; 4: always 8 + 4; bit-identical */
#define PL_OPT_FUSE_APPLY_RHS 17 /* 1 (default): the sweep's f refresh of node m and the next
                                    sub-step's right-hand side share one pass over y[m] (TMA
                                    levels); 0: separate apply and rhs launches; bit-identical */
#define PL_OPT_ZREV 19        /* bit mask of TMA kernels that visit their z chunks top-down, so
                                 they start on the planes the previous kernel left in L2:
                                 1 apply (+ rhs), 2 residual + full weighting (default 3) */
#define PL_OPT_FUSE_FAS_FW 20 /* 1 (default): restrict_state full-weights all selected nodes in one
                                 tiled launch, and the FAS fine node integrals are full-weighted in
                                 the same pass (3-D, >= 127^3), never stored; 0: separate
                                 chain and full-weighting launches; bit-identical */
#define PL_OPT_ZC_FIT 22       /* 1 (default): z chunks of the jor-rb sweep and the cubic kernel
                                  chosen by a wave-quantisation model of the device's resident
                                  CTA slots; 0: power-of-two chunks aiming at PL_OPT_ZC_CTAS */
#define PL_OPT_TOL_DEVICE 24   /* 1 (default): ToTolerance solves whose whole hierarchy fits the
                                  one-CTA tail kernel (1-D, small grids) run their norm / cycle
                                  loop on the device, one launch and one readback per solve;
                                  0: host loop with a readback per V-cycle */
int pl_set_option(int key, int value);

/* storage elements of one field (incl. row pads) */
long long pl_field_elems(int dim, int n);

/* ---- heat operator (heat.py) ------------------------------------------- */
/* f = nu * Lap_h u, order 2 or 4 (HeatOperator.apply, heat.py:111-142) */
int pl_heat_apply(const double* u, double* f, int dim, int n, double length, double nu,
                  int order, void* stream);
/* out = 1 - sigma * diag(nu Lap_h) (ShiftedOperator._diag, multigrid.py:186;
   sigma = 0 and shifted = 0 give HeatOperator.diagonal, heat.py:144-158) */
int pl_heat_diagonal(double* out, int dim, int n, double length, double nu, int order,
                     double sigma, int shifted, void* stream);
/* out = (I - sigma A) u  (ShiftedOperator.apply, multigrid.py:192-193) */
int pl_shifted_apply(const double* u, double* out, int dim, int n, double length, double nu,
                     int order, double sigma, void* stream);

/* ---- grid transfers (transfers.py) -------------------------------------- */
/* nf = fine cells per axis; coarse has nf/2 cells */
int pl_full_weighting(const double* fine, double* coarse, int dim, int nf, void* stream);
int pl_inject(const double* fine, double* coarse, int dim, int nf, void* stream);
/* fine = (accumulate ? fine : 0) + P coarse, P linear (transfers.py:37-50) */
int pl_interp_linear(const double* coarse, double* fine, int dim, int nf, int accumulate,
                     void* stream);
/* cubic (transfers.py:53-89); scratch of pl_interp_cubic_scratch_bytes */
size_t pl_interp_cubic_scratch_bytes(int dim, int nf);
int pl_interp_cubic(const double* coarse, double* fine, int dim, int nf, int accumulate,
                    double* scratch, void* stream);

/* ---- geometric multigrid (multigrid.py) ---------------------------------- */
size_t pl_mg_workspace_bytes(int dim, int n, int coarsest_n);
/* MgConfig + the fine HeatOperator -> plan (multigrid.py:24-38, 178-201) */
/* smoother: 0 jacobi, 1 gauss-seidel (lexicographic, hyperplane wavefront,
   bit-identical to scipy solve_banded), 2 jor-rb */
int pl_mg_plan_create(pl_mg_plan** plan, int dim, int n, double length, double nu, int order,
                      int smoother, double omega, int pre_sweeps, int post_sweeps,
                      int coarsest_n, void* workspace, size_t workspace_bytes);
int pl_mg_plan_destroy(pl_mg_plan* plan);
/* factor the coarsest-grid system for sigma ahead of time (capture-safe) */
int pl_mg_prepare(pl_mg_plan* plan, double sigma, void* stream);
/* install the LAPACK getrf factors of the coarsest-grid system for sigma
   (row-major packed L\U, 0-based pivots, m = pl_mg_coarsest_size unknowns);
   the Python layer passes scipy.linalg.lu_factor's result -- the call the
   reference makes (multigrid.py:161-164) -- so the factors are the
   reference's own; without it the plan factors on the host itself */
int pl_mg_set_coarsest_lu(pl_mg_plan* plan, double sigma, const double* lu, const int* piv,
                          void* stream);
int pl_mg_coarsest_size(pl_mg_plan* plan);
/* smooth(op, u, b, cfg, count), in place on u (multigrid.py:211-234) */
int pl_mg_smooth(pl_mg_plan* plan, double* u, const double* b, double sigma, int count,
                 void* stream);
/* ncycles x v_cycle, in place on u (multigrid.py:237-251, FixedCycles 265-269);
   zero_guess != 0: u is treated as zero on entry */
int pl_mg_vcycles(pl_mg_plan* plan, double* u, const double* b, double sigma, int ncycles,
                  int zero_guess, void* stream);
/* ToTolerance solve (multigrid.py:270-288).  SYNCHRONOUS on stream.
   PL_ERR_MGCAP when max_cycles is exhausted (residual, cycles describe it). */
int pl_mg_solve_tol(pl_mg_plan* plan, double* u, const double* b, double sigma, double tol,
                    double stall, int max_cycles, int* cycles, int* status, double* residual,
                    void* stream);

/* Direct policy (multigrid.py:63-65, 203-208, 263-264: SuperLU of the shifted
   matrix) by fast diagonalisation: install T = V diag(lam) V^-1 of the plan's
   1-D stencil matrix (host arrays, row-major (n-1) x (n-1): W = V^-1, W^T, V,
   V^T, then lam), computed by the caller with numpy eigh/eig; then
   u = (I - sigma nu Lap_h)^-1 b with dense fp64 products along each axis
   (a tiled GEMM kernel of this library).
   Agrees with SuperLU to rounding (tolerance, not bitwise). */
int pl_mg_set_direct(pl_mg_plan* plan, const double* w, const double* wt, const double* v,
                     const double* vt, const double* lam, void* stream);
int pl_mg_direct(pl_mg_plan* plan, double* u, const double* b, double sigma, void* stream);

/* ---- SDC sweeper (sdc.py) ------------------------------------------------ */
#define PL_MAX_NODES 17 /* M + 1 <= 17 */

typedef struct pl_sweep_desc {
  int m;                                  /* sub-steps M */
  double qdelta[PL_MAX_NODES * PL_MAX_NODES]; /* rows m: Q[m+1,:] - Q[m,:], M x (M+1) */
  double gammas[PL_MAX_NODES];            /* float(gamma_m), sub-step fractions */
  int policy;                             /* 0 FixedCycles, 1 ToTolerance, 2 Direct */
  int fixed_cycles;
  double tol, stall;
  int max_cycles;
} pl_sweep_desc;

/* scratch for one sweep: M node-to-node integrals + one right-hand side */
size_t pl_sweep_workspace_bytes(int dim, int n, int m);
/* sdc_sweep(states, y0, dt, op, mg_cfg, policy, tau) (sdc.py:84-114): Y, F are
   (M+1) x npts, in place; tau is (M+1) x npts or NULL.  Returns the V-cycles
   in *cycles and, when substep_cycles / substep_status are non-NULL (host
   arrays of M ints), the SolveResult.cycles and .status (PL_STATUS_*) of every
   sub-step's solve (multigrid.py:261-288 as called at sdc.py:105-113).
   FixedCycles is asynchronous; ToTolerance synchronises per solve.  On
   PL_ERR_MGCAP, *failed_substep (1-based), *fail_residual and *fail_cycles
   describe the failed solve (SubStepError) and the sub-step arrays hold the
   solves before it. */
int pl_sdc_sweep(pl_mg_plan* plan, const pl_sweep_desc* desc, double* Y, double* F,
                 const double* y0, const double* tau, double dt, void* workspace,
                 size_t workspace_bytes, int* cycles, int* substep_cycles, int* substep_status,
                 int* failed_substep, double* fail_residual, int* fail_cycles, void* stream);
/* residual(states, y0, dt, tau) (sdc.py:117-124): max-norm into out_dev
   (device double, asynchronous).  q is (M+1)x(M+1) row-major (host). */
int pl_sdc_residual(const double* Y, const double* F, const double* y0, const double* tau,
                    const double* q, int m, double dt, int dim, int n, double* out_dev,
                    void* stream);

/* ---- FAS machinery (hierarchy.py) ---------------------------------------- */
/* restrict_state (hierarchy.py:85-93): coarse Y[j] = R(fine Y[idx[j]]) for
   j < nsel, then coarse F = A_c coarse Y.  `restrict` is PL_RESTRICT_*. */
int pl_restrict_state(const double* fineY, const int* idx, int nsel, double* coarseY,
                      double* coarseF, int dim, int nf, int nc, int restrict_kind,
                      double length, double nu_c, int order_c, void* stream);
/* compute_fas (hierarchy.py:96-109): tau_c[j] = R((dt Q_f F_f + tau_f)[idx[j]])
   - dt (Q_c F_c)[j].  qf_rows: nsel x (Mf+1) selected rows of Q_f; qc:
   (Mc+1) x (Mc+1).  scratch: nsel fine fields. */
int pl_compute_fas(const double* fineF, const double* fine_tau, int mf, const double* qf_rows,
                   const int* idx, int nsel, const double* coarseF, const double* qc, int mc,
                   double dt, double* tau_c, double* scratch, int dim, int nf, int nc,
                   int restrict_kind, void* stream);
size_t pl_compute_fas_scratch_bytes(int dim, int nf, int nsel);
/* coarse_correction (hierarchy.py:112-122): fine Y[m] += P_space(sum_j
   P_t[m,j] (new_j - old_j)), then fine F = A_f fine Y.  pt: (Mf+1)x(Mc+1).
   interp_order 2 (linear) or 4 (cubic); nc == nf means no spatial
   interpolation.  scratch: pl_coarse_correction_scratch_bytes. */
int pl_coarse_correction(double* fineY, double* fineF, int mf, const double* coarse_new,
                         const double* coarse_old, int mc, const double* pt, int dim, int nf,
                         int nc, int interp_order, double length, double nu_f, int order_f,
                         double* scratch, void* stream);
size_t pl_coarse_correction_scratch_bytes(int dim, int nf, int nc, int mf, int interp_order);

/* ---- runtime statistics (for bench.py / tests) -------------------------- */
/* counts and algorithmic bytes (SURVEY.md 8(d) model) of launched kernels */
int pl_stats_reset(void);
int pl_stats_get(long long* launches, double* alg_bytes, int nkinds);
/* CUDA-event timing of every launch of the kernel kinds in `mask` (bit k =
   kind k; 0 = off); pl_timing_collect returns, for one kind, the launches
   timed, their total milliseconds and their algorithmic bytes */
int pl_timing_enable(unsigned mask);
int pl_timing_collect(int kind, long long* launches, double* total_ms, double* alg_bytes);
/* the individual timed launches of one kind: algorithmic bytes and ms */
int pl_timing_dump(int kind, long long nmax, double* bytes, float* ms, long long* n);
const char* pl_kind_name(int kind);

#ifdef __cplusplus
}
#endif

#endif /* PINTLAB_B200_H */
