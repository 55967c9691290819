// Host-side launchers of the grid-wide kernels (stencil.cu, transfer.cu,
// sdc.cu).  All launch on the given stream and are asynchronous; they return
// 0 or a CUDA status (see common.cuh).
#pragma once
#include "common.cuh"

namespace pl {

// ---- stencil.cu ------------------------------------------------------------
// f = nu Lap(u)                                         heat.py:111-142
int launch_apply(const double* u, double* f, const Geo& g, const OpC& c, cudaStream_t s);
// r = b - (I - sigma A) u                               multigrid.py:245
int launch_residual(const double* u, const double* b, double* r, const Geo& g,
                    const OpC& c, double sigma, cudaStream_t s);
// out = u + (omega (b - A_sigma u)) / diag ; zero_in: u == 0     multigrid.py:217-218
int launch_jacobi(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                  double sigma, double omega, int zero_in, cudaStream_t s);
// one colour of jor-rb (multigrid.py:225-233); in place when in == out
int launch_rb(const double* in, const double* b, double* out, const Geo& g, const OpC& c,
              double sigma, double omega, int red, cudaStream_t s);
// partial sums of squares of (b - A_sigma u) (u may be null: plain b),
// deterministic two-stage reduction into *out (device double)
int launch_sumsq(const double* u, const double* b, const Geo& g, const OpC& c, double sigma,
                 double* partials, int npartials, double* out, cudaStream_t s);
int sumsq_partials(const Geo& g);

// ---- gs.cu -----------------------------------------------------------------
// `count` lexicographic Gauss-Seidel sweeps in place on u (multigrid.py:219-224);
// t is scratch of the field's size
int launch_gs(double* u, const double* b, double* t, const Geo& g, const OpC& c, double sigma,
              int count, cudaStream_t s);

// ---- zmarch.cu: cp.async-pipelined 3-D order-2 versions (zmarch_ok) -------
bool zmarch_ok(const Geo& g, const OpC& c);
bool zmarch_enabled();
bool zmarch_size_ok(int N);
bool zmarch_fuse_prolong();   // PL_OPT_FUSE_PROLONG
int zlaunch_apply(const double* u, double* f, const Geo& g, const OpC& c, cudaStream_t s);
int zlaunch_apply_rhs(const double* u, double* f, const double* fnext, const double* sm,
                      const double* tau0, const double* tau1, double dtm, double* rhs,
                      const Geo& g, const OpC& c, cudaStream_t s);
// f = A u, then rhs = (u - dtm fnext) + sm (+ (tau1 - tau0)): fused on TMA grids
// (PL_OPT_FUSE_APPLY_RHS), two launches otherwise
int launch_apply_rhs(const double* u, double* f, const double* fnext, const double* sm,
                     const double* tau0, const double* tau1, double dtm, double* rhs,
                     long long np, const Geo& g, const OpC& c, cudaStream_t s);
extern int g_fuse_apply_rhs;
int zlaunch_residual(const double* u, const double* b, double* r, const Geo& g, const OpC& c,
                     double sigma, cudaStream_t s);
int zlaunch_jacobi(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                   double sigma, double omega, int zero_in, cudaStream_t s);
// two fused Jacobi sweeps u -> out (out != u); e non-null: u + P_lin e first
int zlaunch_jacobi2(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                    double sigma, double omega, int zero_in, const double* e, cudaStream_t s);
// one fused red+black jor-rb sweep u -> out (out != u)
int zlaunch_rb(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
               double sigma, double omega, cudaStream_t s);

// coarse = FW(b - (I - sigma A) u) in one pass (residual never stored)
bool zmarch_rfw();   // PL_OPT_RFW
int zlaunch_rfw(const double* u, const double* b, double* coarse, const Geo& g, const OpC& c,
                double sigma, cudaStream_t s);


// fine (+)= P_cubic coarse, 3-D, TMA-staged coarse planes (taps of cubic_taps)
int zlaunch_cubic(const double* coarse, double* fine, const Geo& gf, const int* cnt,
                  const int* idx, const double* w, int accumulate, cudaStream_t s);

// ---- transfer.cu -----------------------------------------------------------
// coarse = FW(fine) (transfers.py:27-34); fine geometry gf
int launch_fw(const double* fine, double* coarse, const Geo& gf, cudaStream_t s);
// coarse = fine[1::2, ...] (transfers.py:19-24)
int launch_inject(const double* fine, double* coarse, const Geo& gf, cudaStream_t s);
// fine = (accumulate ? fine : 0) + P_lin coarse (transfers.py:37-50)
int launch_prolong(const double* coarse, double* fine, const Geo& gf, int accumulate,
                   cudaStream_t s);

// cubic taps for one axis refinement nf: per fine array index up to 4
// (coarse index, weight) pairs in increasing coarse index (transfers.py:53-79)
struct CubicTaps {
  int nf;
  int* cnt;     // device [nf-1]
  int* idx;     // device [(nf-1)*4]
  double* w;    // device [(nf-1)*4]
};
const CubicTaps* cubic_taps(int nf);   // cached per nf; null + error on failure
// fine (+)= P_cubic coarse, axis by axis with scratch of
// cubic_scratch_doubles(gf) doubles
long long cubic_scratch_doubles(const Geo& gf);
int launch_cubic(const double* coarse, double* fine, const Geo& gf, int accumulate,
                 double* scratch, cudaStream_t s);

// ---- sdc.cu ---------------------------------------------------------------
struct Coef {          // small dense coefficient matrix, row-major, <= 17 x 17
  int rows, cols;
  double a[17 * 17];
};
// out[m] = scale * chain_k a[m][k] in[k]  for m in [0, rows); in fields of
// `npts` with stride `stride`; zero coefficients skipped; optional
// elementwise add of add[m] (when `add` non-null, computes chain + add[m]).
int launch_chain(const double* in, long long in_stride, double* out, long long out_stride,
                 const Coef& a, double scale, long long npts, cudaStream_t s);
// general form: mode 1 adds add[add_rows[m]] after scaling, mode 2 computes
// add[add_rows[m]] - scale*chain (add_rows null: identity map)
int launch_chain_ex(const double* in, long long in_stride, double* out, long long out_stride,
                    const Coef& a, double scale, long long npts, const double* add,
                    long long add_stride, const int* add_rows, int mode, cudaStream_t s);
// rhs = ((y - dtm f) + s) [+ (tau1 - tau0)]              sdc.py:102-104
int launch_rhs(const double* y, const double* f, const double* sm, const double* tau0,
               const double* tau1, double dtm, double* rhs, long long npts, cudaStream_t s);
// max_m max_i |(y0 + dt chain(q[m], F)) - y[m] (+ tau[m])|    sdc.py:117-124
int launch_resmax(const double* Y, const double* F, long long stride, const double* y0,
                  const double* tau, const Coef& q, double dt, long long npts,
                  double* out_dev, cudaStream_t s);
// d = new - old  (coarse node deltas), then out[m] = chain(P_t[m], d)
// FAS: coarse rows = FW(scale * chain(F) (+ add rows)) in one pass (3-D, >= 127^3,
// 2..5 rows, <= 9 columns; chain_fw_ok); bit-identical to launch_chain_ex + launch_fw
bool chain_fw_ok(const Coef& a, const Geo& gf);
int launch_chain_fw(const double* F, long long stride, const Coef& a, double scale,
                    const double* add, long long add_stride, const int* add_rows,
                    double* coarse, long long cstride, const Geo& gf, cudaStream_t s);
extern int g_fuse_fas_fw;
bool fw_select_ok(const Geo& gf, int nsel);
int launch_fw_select(const double* fine, long long stride, const int* idx, int nsel,
                     double* coarse, long long cstride, const Geo& gf, cudaStream_t s);
int launch_delta_chain(const double* ynew, const double* yold, long long stride,
                       const Coef& pt, double* out, long long out_stride, long long npts,
                       cudaStream_t s);
// out = a + b (elementwise) / out = a - b
int launch_axpby(const double* a, const double* b, double* out, int sub, long long npts,
                 cudaStream_t s);

}  // namespace pl
