// Grid-wide stencil kernels: heat operator, residual, Jacobi and red-black
// smoother sweeps, residual 2-norm.  All fp64, HBM-bound.
//
// Thread mapping: a CTA covers a 32 x BY tile of the (x, y) plane and marches
// through a chunk of z planes, so consecutive iterations of one thread touch
// the plane above the previous one (its z-neighbours are still in L1) and the
// in-plane neighbours are shared with adjacent lanes / warps through L1.  A
// warp reads 32 consecutive x values: 256 B, fully coalesced.
#include "common.cuh"
#include "kernels.cuh"

namespace pl {

namespace {

constexpr int TX = 32;
constexpr int TY = 4;

struct Launch {
  dim3 grid, block;
  int zc;
};

// z planes per thread: large grids march through a chunk (z-neighbours stay
// in L1); small grids take one plane per thread so the grid still fills the
// 148 SMs -- a long per-thread chain over few CTAs is latency-bound
inline Launch plan_launch(const Geo& g) {
  Launch L;
  if (g.dim == 1) {
    L.block = dim3(256, 1, 1);
    L.grid = dim3(ceil_div(g.nx, 256), 1, 1);
    L.zc = 1;
  } else {
    L.block = dim3(TX, TY, 1);
    long long cols = (long long)ceil_div(g.nx, TX) * ceil_div(g.ny, TY);
    int zc = 16;
    while (zc > 1 && cols * ceil_div(g.nz, zc) < 148 * 16) zc /= 2;
    L.zc = zc;
    L.grid = dim3(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc));
  }
  return L;
}

// iterate the points of this thread: (x, y, z, idx)
#define PL_FOR_POINTS(g)                                                       \
  const int x = blockIdx.x * blockDim.x + threadIdx.x;                         \
  const int y = blockIdx.y * blockDim.y + threadIdx.y;                         \
  if (x >= g.nx || y >= g.ny) return;                                          \
  const int z0 = blockIdx.z * zc;                                              \
  const int z1 = min(z0 + zc, g.nz);                                           \
  for (int z = z0; z < z1; ++z)

template <int DIM>
__global__ void __launch_bounds__(256) k_apply(const double* __restrict__ u,
                                               double* __restrict__ f, Geo g, OpC c, int zc) {
  PL_FOR_POINTS(g) {
    long long idx = (long long)z * g.sz + (long long)y * g.sy + x;
    f[idx] = lap_point<DIM>(u, g, c, x, y, z, idx);
  }
}

template <int DIM>
__global__ void __launch_bounds__(256) k_residual(const double* __restrict__ u,
                                                  const double* __restrict__ b,
                                                  double* __restrict__ r, Geo g, OpC c,
                                                  double sigma, int zc) {
  PL_FOR_POINTS(g) {
    long long idx = (long long)z * g.sz + (long long)y * g.sy + x;
    r[idx] = b[idx] - shifted_point<DIM>(u, g, c, sigma, x, y, z, idx);
  }
}

// multigrid.py:218: u + ((omega * (b - A u)) / diag)
template <int DIM>
__global__ void __launch_bounds__(256) k_jacobi(const double* __restrict__ u,
                                                const double* __restrict__ b,
                                                double* __restrict__ out, Geo g, OpC c,
                                                double sigma, double omega, int zero_in, int zc) {
  ConstDiag cd;
  cd.init<DIM>(g, c, sigma);
  PL_FOR_POINTS(g) {
    long long idx = (long long)z * g.sz + (long long)y * g.sy + x;
    if (zero_in) {
      out[idx] = 0.0 + cd.div<DIM>(omega * b[idx], g, c, sigma, x, y, z);
    } else {
      double au = shifted_point<DIM>(u, g, c, sigma, x, y, z, idx);
      out[idx] = u[idx] + cd.div<DIM>(omega * (b[idx] - au), g, c, sigma, x, y, z);
    }
  }
}

// multigrid.py:230-233: u[c] += omega * r[c] / diag[c] for one colour.
template <int DIM>
__global__ void __launch_bounds__(256) k_rb(const double* in, const double* __restrict__ b,
                                            double* out, Geo g, OpC c, double sigma,
                                            double omega, int red, int inplace, int zc) {
  ConstDiag cd;
  cd.init<DIM>(g, c, sigma);
  PL_FOR_POINTS(g) {
    long long idx = (long long)z * g.sz + (long long)y * g.sy + x;
    bool mine = is_red<DIM>(x, y, z) == (red != 0);
    if (mine) {
      double r = b[idx] - shifted_point<DIM>(in, g, c, sigma, x, y, z, idx);
      out[idx] = in[idx] + cd.div<DIM>(omega * r, g, c, sigma, x, y, z);
    } else if (!inplace) {
      out[idx] = in[idx];
    }
  }
}

constexpr int NORM_THREADS = 256;
constexpr int NORM_BLOCKS = 1184;   // 8 x 148 SMs

template <int DIM>
__global__ void __launch_bounds__(NORM_THREADS) k_sumsq(const double* __restrict__ u,
                                                        const double* __restrict__ b,
                                                        Geo g, OpC c, double sigma,
                                                        double* __restrict__ partials) {
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < g.npts;
       t += stride) {
    int x, y, z;
    decode_point(g, t, x, y, z);
    const long long idx = g.at(x, y, z);
    double v;
    if (u) {
      v = b[idx] - shifted_point<DIM>(u, g, c, sigma, x, y, z, idx);
    } else {
      v = b[idx];
    }
    acc = acc + v * v;
  }
  // deterministic tree: warp shuffle, then fixed-order block combine
  for (int off = 16; off > 0; off >>= 1) acc = acc + __shfl_down_sync(0xffffffffu, acc, off);
  __shared__ double wsum[NORM_THREADS / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < NORM_THREADS / 32; ++w) s = s + wsum[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void k_sum_final(const double* __restrict__ partials, int n, double* out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = acc + partials[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

}  // namespace

#define PL_DISPATCH_DIM(g, KERNEL, L, s, ...)                                   \
  do {                                                                         \
    if ((g).dim == 1) KERNEL<1><<<L.grid, L.block, 0, s>>>(__VA_ARGS__);        \
    else if ((g).dim == 2) KERNEL<2><<<L.grid, L.block, 0, s>>>(__VA_ARGS__);   \
    else KERNEL<3><<<L.grid, L.block, 0, s>>>(__VA_ARGS__);                     \
  } while (0)

int launch_apply(const double* u, double* f, const Geo& g, const OpC& c, cudaStream_t s) {
  if (zmarch_ok(g, c)) return zlaunch_apply(u, f, g, c, s);
  Launch L = plan_launch(g);
  PL_PRE(K_APPLY);
  PL_DISPATCH_DIM(g, k_apply, L, s, u, f, g, c, L.zc);
  PL_CHECK_LAUNCH(K_APPLY, 16.0 * g.npts);
  return 0;
}

int g_fuse_apply_rhs = 1;   // PL_OPT_FUSE_APPLY_RHS

int launch_apply_rhs(const double* u, double* f, const double* fnext, const double* sm,
                     const double* tau0, const double* tau1, double dtm, double* rhs,
                     long long np, const Geo& g, const OpC& c, cudaStream_t s) {
  if (g_fuse_apply_rhs && zmarch_ok(g, c))
    return zlaunch_apply_rhs(u, f, fnext, sm, tau0, tau1, dtm, rhs, g, c, s);
  PL_TRY(launch_apply(u, f, g, c, s));
  return launch_rhs(u, fnext, sm, tau0, tau1, dtm, rhs, np, s);
}

int launch_residual(const double* u, const double* b, double* r, const Geo& g, const OpC& c,
                    double sigma, cudaStream_t s) {
  if (zmarch_ok(g, c)) return zlaunch_residual(u, b, r, g, c, sigma, s);
  Launch L = plan_launch(g);
  PL_PRE(K_RESID);
  PL_DISPATCH_DIM(g, k_residual, L, s, u, b, r, g, c, sigma, L.zc);
  PL_CHECK_LAUNCH(K_RESID, 24.0 * g.npts);
  return 0;
}

int launch_jacobi(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                  double sigma, double omega, int zero_in, cudaStream_t s) {
  if (zmarch_ok(g, c)) return zlaunch_jacobi(u, b, out, g, c, sigma, omega, zero_in, s);
  Launch L = plan_launch(g);
  PL_PRE(K_JACOBI);
  PL_DISPATCH_DIM(g, k_jacobi, L, s, u, b, out, g, c, sigma, omega, zero_in, L.zc);
  PL_CHECK_LAUNCH(K_JACOBI, (zero_in ? 16.0 : 24.0) * g.npts);
  return 0;
}

int launch_rb(const double* in, const double* b, double* out, const Geo& g, const OpC& c,
              double sigma, double omega, int red, cudaStream_t s) {
  Launch L = plan_launch(g);
  int inplace = in == out;
  PL_PRE(K_RB);
  PL_DISPATCH_DIM(g, k_rb, L, s, in, b, out, g, c, sigma, omega, red, inplace, L.zc);
  // one colour: half of a full red+black sweep's 24 B/DOF
  PL_CHECK_LAUNCH(K_RB, 12.0 * g.npts);
  return 0;
}

int sumsq_partials(const Geo& g) {
  long long want = (g.npts + NORM_THREADS * 4 - 1) / (NORM_THREADS * 4);
  return (int)(want < NORM_BLOCKS ? (want < 1 ? 1 : want) : NORM_BLOCKS);
}

int launch_sumsq(const double* u, const double* b, const Geo& g, const OpC& c, double sigma,
                 double* partials, int npartials, double* out, cudaStream_t s) {
  dim3 grid(npartials), block(NORM_THREADS);
  PL_PRE(K_NORM);
  PL_DISPATCH_DIM(g, k_sumsq, (Launch{grid, block, 1}), s, u, b, g, c, sigma, partials);
  PL_CHECK_LAUNCH(K_NORM, (u ? 16.0 : 8.0) * g.npts);
  PL_PRE(K_NORM);
  k_sum_final<<<1, 256, 0, s>>>(partials, npartials, out);
  PL_CHECK_LAUNCH(K_NORM, 8.0 * npartials);
  return 0;
}

}  // namespace pl
