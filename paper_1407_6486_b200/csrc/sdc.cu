// Node-axis kernels of the SDC sweeper and the FAS machinery: the streaming
// quadrature (sdc.py:95), right-hand-side build (sdc.py:102-104), collocation
// residual max-norm (sdc.py:117-124), the FAS integrals (hierarchy.py:102-108)
// and the time interpolation of coarse corrections (hierarchy.py:116-118).
//
// Each thread owns one grid point and walks the node axis, so every nodal
// field is streamed exactly once per launch (coalesced 256 B per warp per
// field) and the small M x M coefficient matrix sits in kernel parameter
// (constant) space.  The contractions over nodes are sequential FMA chains
// in column order, which is how the reference's BLAS evaluates
// np.tensordot for these shapes (verified bit-for-bit by the oracle tests).
#include "common.cuh"
#include "kernels.cuh"

namespace pl {

namespace {

constexpr int MAXN = 17;

struct AddMap {
  int row[MAXN];  // field index of `add` for output row m
};

// mode 0: out = scale*chain ; 1: out = scale*chain + add ; 2: out = add - scale*chain
__global__ void __launch_bounds__(256) k_chain(const double* __restrict__ in, long long in_stride,
                                               double* out, long long out_stride,
                                               Coef c, double scale, long long npts,
                                               const double* add,   // may alias out
                                               long long add_stride, AddMap am, int mode) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  double v[MAXN];
#pragma unroll
  for (int k = 0; k < MAXN; ++k) {
    if (k < c.cols) {
      bool used = false;
      for (int m = 0; m < c.rows; ++m) used |= c.a[m * c.cols + k] != 0.0;
      v[k] = used ? in[k * in_stride + i] : 0.0;
    }
  }
  for (int m = 0; m < c.rows; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < MAXN; ++k) {
      if (k < c.cols) {
        double w = c.a[m * c.cols + k];
        if (w != 0.0) acc = __fma_rn(w, v[k], acc);
      }
    }
    double r = scale * acc;
    if (mode == 1) r = r + add[am.row[m] * add_stride + i];
    else if (mode == 2) r = add[am.row[m] * add_stride + i] - r;
    out[m * out_stride + i] = r;
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

// sdc.py:117-124, max-reduced as IEEE bit patterns (non-negative doubles
// order like unsigned integers; NaN propagates like np.max).
__global__ void __launch_bounds__(256) k_resmax(const double* __restrict__ Y,
                                                const double* __restrict__ F, long long stride,
                                                const double* __restrict__ y0,
                                                const double* __restrict__ tau, Coef q,
                                                double dt, long long npts,
                                                unsigned long long* out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long best = 0ull;
  if (i < npts) {
    double f[MAXN];
#pragma unroll
    for (int k = 0; k < MAXN; ++k)
      if (k < q.cols) f[k] = F[k * stride + i];
    double base = y0[i];
    for (int m = 0; m < q.rows; ++m) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < MAXN; ++k) {
        if (k < q.cols) {
          double w = q.a[m * q.cols + k];
          if (w != 0.0) acc = __fma_rn(w, f[k], acc);
        }
      }
      double r = (base + dt * acc) - Y[m * stride + i];
      if (tau) r = r + tau[m * stride + i];
      unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(r));
      best = bits > best ? bits : best;
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
__global__ void __launch_bounds__(256) k_delta_chain(const double* __restrict__ ynew,
                                                     const double* __restrict__ yold,
                                                     long long stride, Coef pt,
                                                     double* __restrict__ out,
                                                     long long out_stride, long long npts) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  double d[MAXN];
#pragma unroll
  for (int j = 0; j < MAXN; ++j)
    if (j < pt.cols) d[j] = ynew[j * stride + i] - yold[j * stride + i];
  for (int m = 0; m < pt.rows; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < MAXN; ++j) {
      if (j < pt.cols) {
        double w = pt.a[m * pt.cols + j];
        if (w != 0.0) acc = __fma_rn(w, d[j], acc);
      }
    }
    out[m * out_stride + i] = acc;
  }
}

__global__ void __launch_bounds__(256) k_axpby(const double* __restrict__ a,
                                               const double* __restrict__ b,
                                               double* __restrict__ out, int sub,
                                               long long npts) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  out[i] = sub ? a[i] - b[i] : a[i] + b[i];
}

}  // namespace

static int used_cols(const Coef& a) {
  int n = 0;
  for (int k = 0; k < a.cols; ++k) {
    bool u = false;
    for (int m = 0; m < a.rows; ++m) u |= a.a[m * a.cols + k] != 0.0;
    n += u;
  }
  return n;
}

int launch_chain_ex(const double* in, long long in_stride, double* out, long long out_stride,
                    const Coef& a, double scale, long long npts, const double* add,
                    long long add_stride, const int* add_rows, int mode, cudaStream_t s) {
  if (a.rows > MAXN || a.cols > MAXN) {
    set_error("coefficient matrix %dx%d exceeds %d", a.rows, a.cols, MAXN);
    return -1;
  }
  AddMap am;
  for (int m = 0; m < MAXN; ++m) am.row[m] = (add_rows && m < a.rows) ? add_rows[m] : m;
  PL_PRE(K_QUAD);
  k_chain<<<ceil_div(npts, 256), 256, 0, s>>>(in, in_stride, out, out_stride, a, scale, npts,
                                              add, add_stride, am, mode);
  PL_CHECK_LAUNCH(K_QUAD, 8.0 * npts * (used_cols(a) + a.rows + (mode ? a.rows : 0)));
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
  if (q.rows > MAXN || q.cols > MAXN) {
    set_error("quadrature matrix too large");
    return -1;
  }
  cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(double), s);
  if (e != cudaSuccess) return cuda_status(e, "memset");
  PL_PRE(K_RESMAX);
  k_resmax<<<ceil_div(npts, 256), 256, 0, s>>>(Y, F, stride, y0, tau, q, dt, npts,
                                               (unsigned long long*)out_dev);
  PL_CHECK_LAUNCH(K_RESMAX, 8.0 * npts * (used_cols(q) + q.rows + 1 + (tau ? q.rows : 0)));
  return 0;
}

int launch_delta_chain(const double* ynew, const double* yold, long long stride,
                       const Coef& pt, double* out, long long out_stride, long long npts,
                       cudaStream_t s) {
  if (pt.rows > MAXN || pt.cols > MAXN) {
    set_error("interpolation matrix too large");
    return -1;
  }
  PL_PRE(K_CORR);
  k_delta_chain<<<ceil_div(npts, 256), 256, 0, s>>>(ynew, yold, stride, pt, out, out_stride,
                                                    npts);
  PL_CHECK_LAUNCH(K_CORR, 8.0 * npts * (2 * pt.cols + pt.rows));
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
