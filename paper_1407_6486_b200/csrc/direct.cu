// Direct solve of (I - sigma nu Lap_h) u = b (multigrid.py:63-65, 203-208,
// 263-264) by fast diagonalisation.
//
// The reference factors the sparse shifted matrix with SuperLU.  The matrix
// is a Kronecker sum of one 1-D stencil matrix T (the same on every axis):
// with T = V diag(lam) V^-1,
//   u = (V x V x V) diag(1 / (1 - sigma nu (lam_i + lam_j + lam_k))) (W x W x W) b,
// W = V^-1, i.e. three batched dense GEMMs with an N x N matrix per
// direction (cuBLAS dgemm -- plain library GEMMs) and one point-wise scale.
// V, W and lam come from the host (numpy eigh / eig + inv, like the
// reference's own host factorisations); the solve is on the GPU.  Results
// agree with SuperLU to rounding (not bitwise): tolerance-tested.
#include <cublas_v2.h>

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

// row-major C (m x n) = A (m x k) * B (k x n), batched with element strides
int gemm_rm(cublasHandle_t h, int m, int n, int k, const double* A, long long lda, long long sa,
            const double* B, long long ldb, long long sb, double* C, long long ldc, long long sc,
            int batch) {
  const double one = 1.0, zero = 0.0;
  cublasStatus_t st = cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, n, m, k, &one, B,
                                                (int)ldb, sb, A, (int)lda, sa, &zero, C,
                                                (int)ldc, sc, batch);
  if (st != CUBLAS_STATUS_SUCCESS) {
    set_error("cublasDgemmStridedBatched failed (%d)", (int)st);
    return 2;
  }
  return 0;
}

// out = M applied along axis `ax` (0 = slowest) of in; M row-major N x N,
// MT its transpose (row-major).  Pads of `out` are written only by the
// slowest-axis product, from the zero pads of `in`.
int apply_axis(cublasHandle_t h, const Geo& g, int ax, const double* M, const double* MT,
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
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) {
      set_error("cublasCreate failed");
      return 2;
    }
    P->cublas = h;
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
  cublasHandle_t h = (cublasHandle_t)P->cublas;
  cublasSetStream(h, s);
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
  if (P->cublas) cublasDestroy((cublasHandle_t)P->cublas);
  cudaFree(P->dir_mats);
  cudaFree(P->dir_work);
  P->cublas = nullptr;
  P->dir_mats = P->dir_work = nullptr;
}

}  // namespace pl
