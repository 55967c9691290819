// Node-axis kernels of the SDC sweeper and the FAS machinery: the streaming
// quadrature (sdc.py:95), right-hand-side build (sdc.py:102-104), collocation
// residual max-norm (sdc.py:117-124), the FAS integrals (hierarchy.py:102-108)
// and the time interpolation of coarse corrections (hierarchy.py:116-118).
//
// Each thread owns one grid point and walks the node axis, so every nodal
// field is streamed exactly once per launch (coalesced 256 B per warp per
// field).  The host compacts the small coefficient matrix to the columns
// that carry a non-zero (column 0 of Q is structurally zero, so F[0] is never
// read) and the kernels are instantiated per column count K, so every
// coefficient index is a compile-time constant.  Contractions over nodes are
// sequential FMA chains in column order -- how the reference's BLAS
// evaluates np.tensordot for these shapes (verified bit-for-bit by the
// oracle tests).  Zero entries inside a used column are FMA'd like BLAS does
// (they can only change the sign of an exact zero).
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace pl {

namespace {

constexpr int MAXN = 17;

struct NodeCoef {
  int rows;            // R <= MAXN
  int col[MAXN];       // source field index of compacted column k
  int addrow[MAXN];    // field index of `add` for output row m
  double a[MAXN * MAXN];   // R x K, row-major over compacted columns
};

// mode 0: out = scale*chain ; 1: out = scale*chain + add ; 2: out = add - scale*chain
template <int K>
__global__ void __launch_bounds__(256) k_chain(const double* __restrict__ in, long long in_stride,
                                               double* out, long long out_stride,
                                               NodeCoef c, double scale, long long npts,
                                               const double* add,   // may alias out
                                               long long add_stride, int mode) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = in[c.col[k] * in_stride + i];
#pragma unroll
  for (int m = 0; m < MAXN; ++m) {
    if (m < c.rows) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) acc = __fma_rn(c.a[m * K + k], v[k], acc);
      double r = scale * acc;
      if (mode == 1) r = r + add[c.addrow[m] * add_stride + i];
      else if (mode == 2) r = add[c.addrow[m] * add_stride + i] - r;
      out[m * out_stride + i] = r;
    }
  }
}

// sdc.py:117-124, max-reduced as IEEE bit patterns (non-negative doubles
// order like unsigned integers; NaN propagates like np.max).
template <int K>
__global__ void __launch_bounds__(256) k_resmax(const double* __restrict__ Y,
                                                const double* __restrict__ F, long long stride,
                                                const double* __restrict__ y0,
                                                const double* __restrict__ tau, NodeCoef q,
                                                double dt, long long npts,
                                                unsigned long long* out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long best = 0ull;
  if (i < npts) {
    double f[K];
#pragma unroll
    for (int k = 0; k < K; ++k) f[k] = F[q.col[k] * stride + i];
    const double base = y0[i];
#pragma unroll
    for (int m = 0; m < MAXN; ++m) {
      if (m < q.rows) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) acc = __fma_rn(q.a[m * K + k], f[k], acc);
        double r = (base + dt * acc) - Y[m * stride + i];
        if (tau) r = r + tau[m * stride + i];
        unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(r));
        best = bits > best ? bits : best;
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    unsigned long long o = __shfl_down_sync(0xffffffffu, best, off);
    best = o > best ? o : best;
  }
  __shared__ unsigned long long sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = sh[w] > best ? sh[w] : best;
    if (best) atomicMax(out, best);
  }
}

// hierarchy.py:116-118: d_j = new_j - old_j ; out[m] = chain_j P_t[m][j] d_j
template <int K>
__global__ void __launch_bounds__(256) k_delta_chain(const double* __restrict__ ynew,
                                                     const double* __restrict__ yold,
                                                     long long stride, NodeCoef pt,
                                                     double* __restrict__ out,
                                                     long long out_stride, long long npts) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  double d[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    long long o = pt.col[k] * stride + i;
    d[k] = ynew[o] - yold[o];
  }
#pragma unroll
  for (int m = 0; m < MAXN; ++m) {
    if (m < pt.rows) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) acc = __fma_rn(pt.a[m * K + k], d[k], acc);
      out[m * out_stride + i] = acc;
    }
  }
}

// sdc.py:102-104
__global__ void __launch_bounds__(256) k_rhs(const double* __restrict__ y,
                                             const double* __restrict__ f,
                                             const double* __restrict__ sm,
                                             const double* __restrict__ tau0,
                                             const double* __restrict__ tau1, double dtm,
                                             double* __restrict__ rhs, long long npts) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  double r = (y[i] - dtm * f[i]) + sm[i];
  if (tau0) r = r + (tau1[i] - tau0[i]);
  rhs[i] = r;
}

__global__ void __launch_bounds__(256) k_axpby(const double* __restrict__ a,
                                               const double* __restrict__ b,
                                               double* __restrict__ out, int sub,
                                               long long npts) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  out[i] = sub ? a[i] - b[i] : a[i] + b[i];
}

// compact a dense R x C matrix to its used columns; false if too large
bool compact(const Coef& a, NodeCoef& c, int& K) {
  if (a.rows > MAXN || a.cols > MAXN) {
    set_error("coefficient matrix %dx%d exceeds %d", a.rows, a.cols, MAXN);
    return false;
  }
  std::memset(&c, 0, sizeof(c));
  c.rows = a.rows;
  K = 0;
  for (int k = 0; k < a.cols; ++k) {
    bool used = false;
    for (int m = 0; m < a.rows; ++m) used |= a.a[m * a.cols + k] != 0.0;
    if (used) c.col[K++] = k;
  }
  for (int m = 0; m < a.rows; ++m)
    for (int k = 0; k < K; ++k) c.a[m * K + k] = a.a[m * a.cols + c.col[k]];
  for (int m = 0; m < MAXN; ++m) c.addrow[m] = m;
  if (K == 0) {            // all-zero matrix: one zero column keeps the chain exact
    c.col[0] = 0;
    K = 1;
  }
  return true;
}

#define PL_K_DISPATCH(K, CALL)                                                    \
  switch (K) {                                                                    \
    case 1: CALL(1); break; case 2: CALL(2); break; case 3: CALL(3); break;      \
    case 4: CALL(4); break; case 5: CALL(5); break; case 6: CALL(6); break;      \
    case 7: CALL(7); break; case 8: CALL(8); break; case 9: CALL(9); break;      \
    case 10: CALL(10); break; case 11: CALL(11); break; case 12: CALL(12); break; \
    case 13: CALL(13); break; case 14: CALL(14); break; case 15: CALL(15); break; \
    case 16: CALL(16); break; default: CALL(17); break;                           \
  }

}  // namespace

int launch_chain_ex(const double* in, long long in_stride, double* out, long long out_stride,
                    const Coef& a, double scale, long long npts, const double* add,
                    long long add_stride, const int* add_rows, int mode, cudaStream_t s) {
  NodeCoef c;
  int K;
  if (!compact(a, c, K)) return -1;
  if (add_rows)
    for (int m = 0; m < a.rows; ++m) c.addrow[m] = add_rows[m];
  const int blocks = ceil_div(npts, 256);
  PL_PRE(K_QUAD);
#define CALL(KK)                                                                          \
  k_chain<KK><<<blocks, 256, 0, s>>>(in, in_stride, out, out_stride, c, scale, npts, add, \
                                     add_stride, mode)
  PL_K_DISPATCH(K, CALL);
#undef CALL
  PL_CHECK_LAUNCH(K_QUAD, 8.0 * npts * (K + a.rows + (mode ? a.rows : 0)));
  return 0;
}

int launch_chain(const double* in, long long in_stride, double* out, long long out_stride,
                 const Coef& a, double scale, long long npts, cudaStream_t s) {
  return launch_chain_ex(in, in_stride, out, out_stride, a, scale, npts, nullptr, 0, nullptr, 0,
                         s);
}

int launch_rhs(const double* y, const double* f, const double* sm, const double* tau0,
               const double* tau1, double dtm, double* rhs, long long npts, cudaStream_t s) {
  PL_PRE(K_RHS);
  k_rhs<<<ceil_div(npts, 256), 256, 0, s>>>(y, f, sm, tau0, tau1, dtm, rhs, npts);
  PL_CHECK_LAUNCH(K_RHS, (tau0 ? 48.0 : 32.0) * npts);
  return 0;
}

int launch_resmax(const double* Y, const double* F, long long stride, const double* y0,
                  const double* tau, const Coef& q, double dt, long long npts,
                  double* out_dev, cudaStream_t s) {
  NodeCoef c;
  int K;
  if (!compact(q, c, K)) return -1;
  cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(double), s);
  if (e != cudaSuccess) return cuda_status(e, "memset");
  const int blocks = ceil_div(npts, 256);
  unsigned long long* o = (unsigned long long*)out_dev;
  PL_PRE(K_RESMAX);
#define CALL(KK) k_resmax<KK><<<blocks, 256, 0, s>>>(Y, F, stride, y0, tau, c, dt, npts, o)
  PL_K_DISPATCH(K, CALL);
#undef CALL
  PL_CHECK_LAUNCH(K_RESMAX, 8.0 * npts * (K + q.rows + 1 + (tau ? q.rows : 0)));
  return 0;
}

int launch_delta_chain(const double* ynew, const double* yold, long long stride,
                       const Coef& pt, double* out, long long out_stride, long long npts,
                       cudaStream_t s) {
  NodeCoef c;
  int K;
  if (!compact(pt, c, K)) return -1;
  const int blocks = ceil_div(npts, 256);
  PL_PRE(K_CORR);
#define CALL(KK) \
  k_delta_chain<KK><<<blocks, 256, 0, s>>>(ynew, yold, stride, c, out, out_stride, npts)
  PL_K_DISPATCH(K, CALL);
#undef CALL
  PL_CHECK_LAUNCH(K_CORR, 8.0 * npts * (2 * K + pt.rows));
  return 0;
}

int launch_axpby(const double* a, const double* b, double* out, int sub, long long npts,
                 cudaStream_t s) {
  PL_PRE(K_COPY);
  k_axpby<<<ceil_div(npts, 256), 256, 0, s>>>(a, b, out, sub, npts);
  PL_CHECK_LAUNCH(K_COPY, 24.0 * npts);
  return 0;
}

}  // namespace pl
