// Direct solve of (I - sigma nu Lap_h) u = b (multigrid.py:63-65, 203-208,
// 263-264) by fast diagonalisation.
//
// The reference factors the sparse shifted matrix with SuperLU.  The matrix
// is a Kronecker sum of one 1-D stencil matrix T (the same on every axis):
// with T = V diag(lam) V^-1,
//   u = (V x V x V) diag(1 / (1 - sigma nu (lam_i + lam_j + lam_k))) (W x W x W) b,
// W = V^-1, i.e. one dense N x N product per direction and way (k_dgemm_rm,
// a tiled fp64 GEMM written here) and one point-wise scale.
// V, W and lam come from the host (numpy eigh / eig + inv, like the
// reference's own host factorisations); the solve is on the GPU.  Results
// agree with SuperLU to rounding (not bitwise): tolerance-tested.
#include <cstring>

#include "common.cuh"
#include "mg.h"

namespace pl {

namespace {

template <int DIM>
__global__ void k_direct_scale(double* w, Geo g, const double* __restrict__ lam, double nu,
                               double sigma) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.npts) return;
  int x, y, z;
  decode_point(g, t, x, y, z);
  double s = lam[x];
  if (DIM >= 2) s = lam[y] + s;
  if (DIM == 3) s = lam[z] + s;
  const long long p = g.at(x, y, z);
  w[p] = w[p] / (1.0 - sigma * (nu * s));
}

// row-major C (m x n) = A (m x k) * B (k x n), batched with element strides.
// 64 x 64 output tile per CTA, 256 threads with 4 x 4 outputs each, k in
// steps of 16 through shared memory; every output is one FMA chain over k in
// increasing order (deterministic).  Out-of-range rows / columns / k load
// zeros and store nothing.
constexpr int GBM = 64, GBN = 64, GBK = 16;

__global__ void __launch_bounds__(256) k_dgemm_rm(int m, int n, int k, const double* __restrict__ A,
                                                  long long lda, long long sa,
                                                  const double* __restrict__ B, long long ldb,
                                                  long long sb, double* __restrict__ C,
                                                  long long ldc, long long sc) {
  __shared__ double As[GBK][GBM + 2];   // As[kk][i] = A[i0 + i][k0 + kk]
  __shared__ double Bs[GBK][GBN + 2];   // Bs[kk][j] = B[k0 + kk][j0 + j]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = blockIdx.y * GBM, j0 = blockIdx.x * GBN;
  A += (long long)blockIdx.z * sa;
  B += (long long)blockIdx.z * sb;
  C += (long long)blockIdx.z * sc;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < k; k0 += GBK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {            // A tile: 64 rows x 16 k
      const int e = tid + q * 256, i = e >> 4, kk = e & 15;
      const int gi = i0 + i, gk = k0 + kk;
      As[kk][i] = gi < m && gk < k ? A[(long long)gi * lda + gk] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {            // B tile: 16 k x 64 columns
      const int e = tid + q * 256, kk = e >> 6, j = e & 63;
      const int gk = k0 + kk, gj = j0 + j;
      Bs[kk][j] = gk < k && gj < n ? B[(long long)gk * ldb + gj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[kk][tx + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = __fma_rn(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int gi = i0 + ty * 4 + r;
    if (gi >= m) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int gj = j0 + tx + 16 * c;
      if (gj < n) C[(long long)gi * ldc + gj] = acc[r][c];
    }
  }
}

int gemm_rm(cudaStream_t s, int m, int n, int k, const double* A, long long lda, long long sa,
            const double* B, long long ldb, long long sb, double* C, long long ldc, long long sc,
            int batch) {
  dim3 grid(ceil_div(n, GBN), ceil_div(m, GBM), batch);
  k_dgemm_rm<<<grid, 256, 0, s>>>(m, n, k, A, lda, sa, B, ldb, sb, C, ldc, sc);
  return cuda_status(cudaGetLastError(), "direct transform");
}

// out = M applied along axis `ax` (0 = slowest) of in; M row-major N x N,
// MT its transpose (row-major).  Pads of `out` are written only by the
// slowest-axis product, from the zero pads of `in`.
int apply_axis(cudaStream_t h, const Geo& g, int ax, const double* M, const double* MT,
               const double* in, double* out) {
  const int N = g.N;
  const int fast = g.dim - 1;
  if (ax == fast) {   // rows of the field: out_row = M in_row  ->  OUT = IN * M^T
    const int rows = (int)(g.npts / N);
    return gemm_rm(h, rows, N, N, in, g.dim == 1 ? N : g.sy, 0, MT, N, 0, out,
                   g.dim == 1 ? N : g.sy, 0, 1);
  }
  if (ax == 0) {      // slowest axis: OUT (N x plane) = M * IN (N x plane)
    const long long plane = g.dim == 3 ? g.sz : g.sy;
    return gemm_rm(h, N, (int)plane, N, M, N, 0, in, plane, 0, out, plane, 0, 1);
  }
  // 3-D middle axis: per z plane OUT_z (N x nx) = M * IN_z
  return gemm_rm(h, N, N, N, M, N, 0, in, g.sy, g.sz, out, g.sy, g.sz, g.nz);
}

}  // namespace

int mg_set_direct(MgPlan* P, const double* w, const double* wt, const double* v,
                  const double* vt, const double* lam, cudaStream_t s) {
  const MgLevel& L = P->lv[0];
  const size_t N = (size_t)L.g.N;
  if (!P->dir_mats) {
    cudaError_t e = cudaMalloc(&P->dir_mats, sizeof(double) * (4 * N * N + N));
    if (e != cudaSuccess) return cuda_status(e, "cudaMalloc direct factors");
    e = cudaMalloc(&P->dir_work, sizeof(double) * 2 * (size_t)L.g.nstore);
    if (e != cudaSuccess) return cuda_status(e, "cudaMalloc direct scratch");
    // pads of the scratch fields must read as zeros (apply_axis)
    e = cudaMemsetAsync(P->dir_work, 0, sizeof(double) * 2 * (size_t)L.g.nstore, s);
    if (e != cudaSuccess) return cuda_status(e, "memset direct scratch");
  }
  const double* src[5] = {w, wt, v, vt, lam};
  const size_t cnt[5] = {N * N, N * N, N * N, N * N, N};
  size_t off = 0;
  for (int i = 0; i < 5; ++i) {
    cudaError_t e = cudaMemcpyAsync(P->dir_mats + off, src[i], sizeof(double) * cnt[i],
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "upload direct factors");
    off += cnt[i];
  }
  // the host arrays may be released on return
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "sync");
  P->dir_ready = 1;
  return 0;
}

int mg_direct(MgPlan* P, double* u, const double* b, double sigma, cudaStream_t s) {
  if (!P->dir_ready) {
    set_error("direct solve: factors not installed (pl_mg_set_direct)");
    return -3;
  }
  const MgLevel& L = P->lv[0];
  const Geo& g = L.g;
  const size_t N = (size_t)g.N;
  const double* W = P->dir_mats;
  const double* WT = W + N * N;
  const double* V = WT + N * N;
  const double* VT = V + N * N;
  const double* lam = VT + N * N;
  double* t0 = P->dir_work;
  double* t1 = P->dir_work + g.nstore;
  cudaStream_t h = s;
  PL_PRE(K_DIRECT);
  // forward transform W along every axis (fastest first), scale, V back
  const double* in = b;
  double* bufs[2] = {t0, t1};
  int nb = 0;
  for (int ax = g.dim - 1; ax >= 0; --ax) {
    PL_TRY(apply_axis(h, g, ax, W, WT, in, bufs[nb]));
    in = bufs[nb];
    nb ^= 1;
  }
  double* w = const_cast<double*>(in);
  const int blocks = ceil_div(g.npts, 256);
  if (g.dim == 1) k_direct_scale<1><<<blocks, 256, 0, s>>>(w, g, lam, L.c.nu, sigma);
  else if (g.dim == 2) k_direct_scale<2><<<blocks, 256, 0, s>>>(w, g, lam, L.c.nu, sigma);
  else k_direct_scale<3><<<blocks, 256, 0, s>>>(w, g, lam, L.c.nu, sigma);
  for (int ax = g.dim - 1; ax >= 0; --ax) {
    double* dst = ax == 0 ? u : bufs[nb];
    PL_TRY(apply_axis(h, g, ax, V, VT, in, dst));
    in = dst;
    nb ^= 1;
  }
  // algorithmic bytes: 2 * dim dense passes (read + write a field) + the scale
  PL_CHECK_LAUNCH(K_DIRECT, (32.0 * g.dim + 16.0) * g.npts);
  return 0;
}

void mg_direct_destroy(MgPlan* P) {
  cudaFree(P->dir_mats);
  cudaFree(P->dir_work);
  P->dir_mats = P->dir_work = nullptr;
}

}  // namespace pl
