// Geometric multigrid V-cycle (multigrid.py:211-288) on B200.
//
// Levels whose whole remaining hierarchy fits in one SM's shared memory run
// as ONE single-CTA "tail" kernel (smoothers, residual, full weighting,
// dense LU on the coarsest grid, prolongation, post-smoothing) -- these
// levels are latency-bound, and folding them into one launch removes ~7
// launches per level.  Larger levels use the grid-wide HBM-streaming kernels
// of stencil.cu / transfer.cu.  Both paths evaluate the same device
// arithmetic (common.cuh / transfer_dev.cuh), so where a level runs does not
// change a single bit of the result.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "kernels.cuh"
#include "mg.h"
#include "transfer_dev.cuh"
#include "gs.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace pl {

// ---------------------------------------------------------------------------
// operator constants (heat.py:114, 148-152) computed with the same libm pow
// the reference's Python floats use

OpC make_opc(int n, double length, double nu, int order) {
  static double (*volatile powp)(double, double) = std::pow;
  OpC c;
  volatile double dx = length / (double)n;
  c.dx2 = powp(dx, 2.0);
  int e;
  double mant = std::frexp(c.dx2, &e);
  // a power of two no larger than one: scaling by 1 / dx^2 is then exact and
  // cannot underflow, which the FMA folds of the stencil kernels rely on
  c.pow2 = (mant == 0.5) && c.dx2 <= 1.0;
  c.inv_dx2 = 1.0 / c.dx2;
  c.d12 = 12.0 * c.dx2;
  c.nu = nu;
  c.order = order;
  c.d1_edge = -2.0 / c.dx2;
  c.d1_int = order == 2 ? -2.0 / c.dx2 : -30.0 / (12.0 * c.dx2);
  return c;
}

// ---------------------------------------------------------------------------
// single-CTA tail

int g_fast_tail = 1;   // PL_OPT_FAST_TAIL

namespace {

constexpr int TAIL_THREADS = 1024;
constexpr int MAX_LEVELS = 16;
constexpr size_t TAIL_SMEM_BUDGET = 200 * 1024;

struct TailLevel {
  Geo g;
  OpC c;
  int off_u, off_b, off_t;   // offsets (doubles) into shared memory
  int coarsest;
};

struct TailArgs {
  Geo g0;             // global (storage) geometry of the first tail level
  int nlev;
  TailLevel lv[MAX_LEVELS];
  int smoother, pre, post;
  double omega, sigma;
  const double* lu;   // m*m factors + m pivots (global)
  int m;
  int lu_off;         // >= 0: factors staged in shared memory at this offset
  int fast;           // 15 or 7: compile-time-sized 3-D order-2 jor-rb path (ft_*)
  unsigned long long* trace;   // PL_MID_TRACE: [0] count, then %globaltimer per tail phase
};

// ToTolerance loop run inside the tail kernel (multigrid.py:270-288) when the
// whole hierarchy fits one CTA: norms are block reductions, the loop control
// is on the device, and the outcome goes to out[0] = residual, out[1] =
// 4 * cycles + (status + 1) with status -1 for the cycle cap.  u is written
// back only when the solve succeeds (the reference solves on a copy).
struct TolArgs {
  int on;
  double tol, stall;
  int max_cycles;
  double* out;
};

// diagnostics only (PL_MID_TRACE): thread 0 stamps the end of a tail phase
__device__ __forceinline__ void ft_stamp(const TailArgs& a) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long k = a.trace[0]++;
    if (k < 62) a.trace[1 + k] = t;
  }
}

#define PL_FOR_SM_POINTS(g)                                                  \
  for (int p = threadIdx.x; p < (int)(g).npts; p += blockDim.x)

__device__ __forceinline__ void decode(const Geo& g, int p, int& x, int& y, int& z) {
  decode_point(g, p, x, y, z);
}

// `count` sweeps on shared-memory level L; result ends in u.
template <int DIM>
__device__ void tail_smooth(const TailArgs& a, const TailLevel& L, double* sm, int count,
                            bool zero) {
  double* u = sm + L.off_u;
  double* b = sm + L.off_b;
  double* t = sm + L.off_t;
  if (count == 0) {
    if (zero) {
      PL_FOR_SM_POINTS(L.g) u[p] = 0.0;
      __syncthreads();
    }
    return;
  }
  ConstDiag cd;
  cd.init<DIM>(L.g, L.c, a.sigma);
  if (a.smoother == SM_JACOBI) {
    // ping-pong u <-> t; one copy back only for an odd sweep count
    for (int k = 0; k < count; ++k) {
      const bool z0 = zero && k == 0;
      const double* src = (k & 1) ? t : u;
      double* dst = (k & 1) ? u : t;
      PL_FOR_SM_POINTS(L.g) {
        int x, y, z;
        decode(L.g, p, x, y, z);
        if (z0) {
          dst[p] = 0.0 + cd.div<DIM>(a.omega * b[p], L.g, L.c, a.sigma, x, y, z);
        } else {
          double au = shifted_point<DIM>(src, L.g, L.c, a.sigma, x, y, z, p);
          dst[p] = src[p] + cd.div<DIM>(a.omega * (b[p] - au), L.g, L.c, a.sigma, x, y, z);
        }
      }
      __syncthreads();
    }
    if (count & 1) {
      PL_FOR_SM_POINTS(L.g) u[p] = t[p];
      __syncthreads();
    }
    return;
  }
  if (a.smoother == SM_GS) {
    // lexicographic Gauss-Seidel (gs.cuh): residual into t, then the
    // hyperplanes x + y + z = s in order (1-D: one thread), y over r in t
    if (zero) {
      PL_FOR_SM_POINTS(L.g) u[p] = 0.0;
      __syncthreads();
    }
    const int smax = (L.g.nx - 1) + (DIM >= 2 ? L.g.ny - 1 : 0) + (DIM == 3 ? L.g.nz - 1 : 0);
    for (int k = 0; k < count; ++k) {
      PL_FOR_SM_POINTS(L.g) {
        int x, y, z;
        decode(L.g, p, x, y, z);
        t[p] = b[p] - shifted_point<DIM>(u, L.g, L.c, a.sigma, x, y, z, p);
      }
      __syncthreads();
      if (DIM == 1) {
        if (threadIdx.x == 0)
          for (int x = 0; x < L.g.nx; ++x) {
            const double yi = gs_lower_point<DIM>(t, t[x], L.g, L.c, a.sigma, x, 0, 0, x);
            t[x] = yi;
            u[x] = u[x] + yi / shifted_diag<DIM>(L.g, L.c, a.sigma, x, 0, 0);
          }
        __syncthreads();
        continue;
      }
      for (int s = 0; s <= smax; ++s) {
        PL_FOR_SM_POINTS(L.g) {
          int x, y, z;
          decode(L.g, p, x, y, z);
          if (x + y + z != s) continue;
          const double yi = gs_lower_point<DIM>(t, t[p], L.g, L.c, a.sigma, x, y, z, p);
          t[p] = yi;
          u[p] = u[p] + yi / shifted_diag<DIM>(L.g, L.c, a.sigma, x, y, z);
        }
        __syncthreads();
      }
    }
    return;
  }
  // jor-rb: red then black per sweep; out of place (t) so that order-4
  // same-colour neighbours read pre-update values like the reference.
  if (zero) {
    PL_FOR_SM_POINTS(L.g) u[p] = 0.0;
    __syncthreads();
  }
  for (int k = 0; k < count; ++k) {
    for (int colour = 1; colour >= 0; --colour) {
      if (L.c.order == 2) {
        // same-colour points never neighbour: update in place, visiting only
        // this colour (x = 2h + s on each (y, z) row)
        const int N = L.g.nx, H = (N + 1) / 2;
        const int rows = (DIM >= 2 ? L.g.ny : 1) * (DIM == 3 ? L.g.nz : 1);
        for (int t = threadIdx.x; t < H * rows; t += blockDim.x) {
          const int row = t / H, h = t - row * H;
          const int y = DIM >= 2 ? row % L.g.ny : 0;
          const int z = DIM == 3 ? row / L.g.ny : 0;
          // is_red: x + y + z + DIM even
          const int x = 2 * h + (((y + z + DIM) & 1) ^ colour ^ 1);
          if (x >= N) continue;
          const int p = (z * L.g.ny + y) * N + x;
          double r = b[p] - shifted_point<DIM>(u, L.g, L.c, a.sigma, x, y, z, p);
          u[p] = u[p] + cd.div<DIM>(a.omega * r, L.g, L.c, a.sigma, x, y, z);
        }
        __syncthreads();
        continue;
      }
      PL_FOR_SM_POINTS(L.g) {
        int x, y, z;
        decode(L.g, p, x, y, z);
        if (is_red<DIM>(x, y, z) == (colour == 1)) {
          double d = shifted_diag<DIM>(L.g, L.c, a.sigma, x, y, z);
          double r = b[p] - shifted_point<DIM>(u, L.g, L.c, a.sigma, x, y, z, p);
          t[p] = u[p] + ((a.omega * r) / d);
        } else {
          t[p] = u[p];
        }
      }
      __syncthreads();
      PL_FOR_SM_POINTS(L.g) u[p] = t[p];
      __syncthreads();
    }
  }
}

// dense LU solve on the coarsest grid: b (smem) -> u (smem), one warp.
// LAPACK getrs order: row interchanges, unit-lower forward, upper backward.
__device__ void tail_lu(const TailArgs& a, const double* lu, const double* b, double* u) {
  const int m = a.m;
  const double* A = lu;
  const double* piv = a.lu + (size_t)m * m;
  if (threadIdx.x < 32) {
    for (int i = threadIdx.x; i < m; i += 32) u[i] = b[i];
    __syncwarp();
    if (threadIdx.x == 0) {
      for (int i = 0; i < m; ++i) {
        int pi = (int)piv[i];
        if (pi != i) {
          double tmp = u[i];
          u[i] = u[pi];
          u[pi] = tmp;
        }
      }
    }
    __syncwarp();
    // column-oriented substitutions with FMA axpy updates and a true
    // division by the pivot -- the operation order of LAPACK getrs over
    // BLAS trsv/axpy (bit-identical to scipy.linalg.lu_solve, see
    // tests/test_gpu_parity.py::test_coarsest_direct)
    for (int j = 0; j < m; ++j) {            // L y = Pb (unit lower)
      double yj = u[j];
      __syncwarp();
      for (int i = j + 1 + threadIdx.x; i < m; i += 32) u[i] = __fma_rn(-yj, A[i * m + j], u[i]);
      __syncwarp();
    }
    const double* rcp = A + (size_t)m * m + m;   // RN(1 / U_jj), host-computed
    for (int j = m - 1; j >= 0; --j) {       // U x = y
      if (threadIdx.x == 0) u[j] = div_diag(u[j], A[j * m + j], rcp[j]);
      __syncwarp();
      double xj = u[j];
      for (int i = threadIdx.x; i < j; i += 32) u[i] = __fma_rn(-xj, A[i * m + j], u[i]);
      __syncwarp();
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// fast tail: 3-D order-2 jor-rb tails 15^3 -> 7^3 -> 3^3 (LU, 27 unknowns) or
// 7^3 -> 3^3 with compile-time level sizes (index arithmetic folds away),
// colour-only sweeps and the LU solve as a register/shuffle chain in one
// warp.  Per point it calls the generic tail's device functions
// (shifted_point, shifted_diag, fw_point, lin_point) in the same order, so
// the result is bit-identical to tail_run's generic path.

template <int N>
__device__ __forceinline__ Geo ct_geo() {
  Geo g;
  g.dim = 3;
  g.N = N;
  g.nx = N;
  g.ny = N;
  g.nz = N;
  g.sy = N;
  g.sz = N * N;
  g.npts = N * N * N;
  g.nstore = N * N * N;
  return g;
}

// (I - sigma A) u at point p of a dense N^3 shared-memory level, order 2 with
// a power-of-two dx^2: lap_point / shifted_point's operations in their order
// (axes z, y, x accumulated from 0.0, x / dx2 == x * inv_dx2 exactly, zero
// ghosts), with the order and pow2 branches folded away at compile time
template <int N>
__device__ __forceinline__ double ft_shifted(const double* u, double inv, double nu,
                                            double sigma, int x, int y, int z, int p) {
  const double c0 = u[p];
  const double zm = z > 0 ? u[p - N * N] : 0.0, zp = z < N - 1 ? u[p + N * N] : 0.0;
  const double ym = y > 0 ? u[p - N] : 0.0, yp = y < N - 1 ? u[p + N] : 0.0;
  const double xm = x > 0 ? u[p - 1] : 0.0, xp = x < N - 1 ? u[p + 1] : 0.0;
  double acc = 0.0;
  acc = acc + ((zm - 2.0 * c0) + zp) * inv;
  acc = acc + ((ym - 2.0 * c0) + yp) * inv;
  acc = acc + ((xm - 2.0 * c0) + xp) * inv;
  return c0 - sigma * (nu * acc);
}

template <int N>
__device__ __forceinline__ void ft_colour(double* u, const double* b, const OpC& c, double sigma,
                                          double omega, int red, bool zero) {
  const Geo g = ct_geo<N>();
  // order 2: the diagonal is the same at every point (shifted_diag's operations)
  const double d = shifted_diag<3>(g, c, sigma, 1, 1, 1);
  const double dr = rcp_diag(d);  // the quotients below are div_const's (exact RN)
  if (zero) {   // u == 0 on entry: red points 0 + (omega b) / d, black points 0
    for (int p = threadIdx.x; p < N * N * N; p += blockDim.x) {
      const int x = p % N, y = (p / N) % N, z = p / (N * N);
      u[p] = is_red<3>(x, y, z) ? 0.0 + div_diag(omega * b[p], d, dr) : 0.0;
    }
    return;
  }
  const double inv = c.inv_dx2, nu = c.nu;
  constexpr int H = (N + 1) / 2;
  for (int t = threadIdx.x; t < H * N * N; t += blockDim.x) {
    const int h = t % H, row = t / H;
    const int y = row % N, z = row / N;
    const int x = 2 * h + (((y + z + 3) & 1) ^ red ^ 1);
    if (x >= N) continue;
    const int p = (z * N + y) * N + x;
    const double r = b[p] - ft_shifted<N>(u, inv, nu, sigma, x, y, z, p);
    u[p] = u[p] + div_diag(omega * r, d, dr);
  }
}

// LAPACK getrs order (tail_lu) for m = 27: lane i of warp 0 holds u[i]
__device__ __forceinline__ void ft_lu27(const double* A, const double* b, double* u) {
  constexpr int m = 27;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const double* piv = A + m * m;
    // the sequential row interchanges, traced back to the source row
    int q = lane;
    for (int i = m - 1; i >= 0; --i) {
      const int pi = (int)piv[i];
      if (q == i) q = pi;
      else if (q == pi) q = i;
    }
    double v = lane < m ? b[q] : 0.0;
    for (int j = 0; j < m; ++j) {              // L y = P b (unit lower)
      const double yj = __shfl_sync(0xffffffffu, v, j);
      if (lane > j && lane < m) v = __fma_rn(-yj, A[lane * m + j], v);
    }
    const double* rcp = A + m * m + m;        // RN(1 / U_jj), host-computed
    for (int j = m - 1; j >= 0; --j) {          // U x = y
      if (lane == j) v = div_diag(v, A[j * m + j], rcp[j]);
      const double xj = __shfl_sync(0xffffffffu, v, j);
      if (lane < j) v = __fma_rn(-xj, A[lane * m + j], v);
    }
    if (lane < m) u[lane] = v;
  }
  __syncthreads();
}

// ft_colour's zero-guess red pass at one point (u == 0 on entry)
__device__ __forceinline__ double ft_red0(double bv, double omega, double d, double dr, int x,
                                          int y, int z) {
  return is_red<3>(x, y, z) ? 0.0 + div_diag(omega * bv, d, dr) : 0.0;
}

// fused: the zero-guess red pass (zero && pre > 0) was already applied by the
// producer of b (the parent's full weighting or the tail's load loop)
template <int N, int L>
__device__ void ft_level(const TailArgs& a, double* sm, bool zero, bool fused = false) {
  const TailLevel& T = a.lv[L];
  double* u = sm + T.off_u;
  double* b = sm + T.off_b;
  if constexpr (N == 3) {
    ft_lu27(sm + a.lu_off, b, u);
    ft_stamp(a);
  } else {
    constexpr int NC = (N - 1) / 2;
    double* t = sm + T.off_t;
    const Geo g = ct_geo<N>();
    const Geo gc = ct_geo<NC>();
    if (zero && a.pre == 0) {
      for (int p = threadIdx.x; p < N * N * N; p += blockDim.x) u[p] = 0.0;
      __syncthreads();
      ft_stamp(a);
    }
    for (int k = 0; k < a.pre; ++k) {
      if (!(fused && zero && k == 0)) {
        ft_colour<N>(u, b, T.c, a.sigma, a.omega, 1, zero && k == 0);
        __syncthreads();
        ft_stamp(a);
      }
      ft_colour<N>(u, b, T.c, a.sigma, a.omega, 0, false);
      __syncthreads();
      ft_stamp(a);
    }
    for (int p = threadIdx.x; p < N * N * N; p += blockDim.x) {
      const int x = p % N, y = (p / N) % N, z = p / (N * N);
      t[p] = b[p] - ft_shifted<N>(u, T.c.inv_dx2, T.c.nu, a.sigma, x, y, z, p);
    }
    __syncthreads();
      ft_stamp(a);
    const TailLevel& C = a.lv[L + 1];
    double* bc = sm + C.off_b;
    // the coarse level starts from zero: its first red pass is fused here
    // (NC == 3 is the LU, which has no sweeps)
    constexpr bool FUSE = NC > 3;
    const bool fz = FUSE && a.pre > 0;
    double* uc = sm + C.off_u;
    const double dc = shifted_diag<3>(gc, C.c, a.sigma, 1, 1, 1), dcr = rcp_diag(dc);
    for (int p = threadIdx.x; p < NC * NC * NC; p += blockDim.x) {
      const int x = p % NC, y = (p / NC) % NC, z = p / (NC * NC);
      const double v = fw_point<3>(t, g, x, y, z);
      bc[p] = v;
      if (fz) uc[p] = ft_red0(v, a.omega, dc, dcr, x, y, z);
    }
    __syncthreads();
      ft_stamp(a);
    ft_level<NC, L + 1>(a, sm, true, fz);
    const double* ec = sm + C.off_u;
    for (int p = threadIdx.x; p < N * N * N; p += blockDim.x) {
      const int x = p % N, y = (p / N) % N, z = p / (N * N);
      u[p] = u[p] + lin_point<3>(ec, gc, x, y, z);
    }
    __syncthreads();
      ft_stamp(a);
    for (int k = 0; k < a.post; ++k) {
      ft_colour<N>(u, b, T.c, a.sigma, a.omega, 1, false);
      __syncthreads();
      ft_stamp(a);
      ft_colour<N>(u, b, T.c, a.sigma, a.omega, 0, false);
      __syncthreads();
      ft_stamp(a);
    }
  }
}

// one V-cycle of the tail levels on the shared-memory state (level 0 u, b)
template <int DIM>
__device__ void tail_vcycle(const TailArgs& a, double* sm, bool zero0) {
  int l = 0;
  // ---- down: pre-smooth, residual, full weighting
  for (; !a.lv[l].coarsest; ++l) {
    const TailLevel& L = a.lv[l];
    const TailLevel& C = a.lv[l + 1];
    tail_smooth<DIM>(a, L, sm, a.pre, l == 0 ? zero0 : true);
    double* u = sm + L.off_u;
    double* b = sm + L.off_b;
    double* t = sm + L.off_t;
    PL_FOR_SM_POINTS(L.g) {
      int x, y, z;
      decode(L.g, p, x, y, z);
      t[p] = b[p] - shifted_point<DIM>(u, L.g, L.c, a.sigma, x, y, z, p);
    }
    __syncthreads();
    double* bc = sm + C.off_b;
    PL_FOR_SM_POINTS(C.g) {
      int x, y, z;
      decode(C.g, p, x, y, z);
      bc[p] = fw_point<DIM>(t, L.g, x, y, z);
    }
    __syncthreads();
  }
  // ---- coarsest: dense LU (ignores the initial guess, multigrid.py:240-243)
  tail_lu(a, a.lu_off >= 0 ? sm + a.lu_off : a.lu, sm + a.lv[l].off_b, sm + a.lv[l].off_u);
  // ---- up: prolongate, correct, post-smooth
  for (--l; l >= 0; --l) {
    const TailLevel& L = a.lv[l];
    const TailLevel& C = a.lv[l + 1];
    double* u = sm + L.off_u;
    const double* ec = sm + C.off_u;
    PL_FOR_SM_POINTS(L.g) {
      int x, y, z;
      decode(L.g, p, x, y, z);
      u[p] = u[p] + lin_point<DIM>(ec, C.g, x, y, z);
    }
    __syncthreads();
    tail_smooth<DIM>(a, L, sm, a.post, false);
  }
}

// sum of squares over level 0 of b (u == nullptr) or of b - A_sigma u, in a
// fixed order (per-thread strided sums, warp shuffles, then warp 0)
template <int DIM>
__device__ double tail_sumsq(const TailArgs& a, const double* sm, bool resid) {
  __shared__ double part[TAIL_THREADS / 32];
  const TailLevel& L = a.lv[0];
  const double* u = sm + L.off_u;
  const double* b = sm + L.off_b;
  double acc = 0.0;
  PL_FOR_SM_POINTS(L.g) {
    double v = b[p];
    if (resid) {
      int x, y, z;
      decode(L.g, p, x, y, z);
      v = v - shifted_point<DIM>(u, L.g, L.c, a.sigma, x, y, z, p);
    }
    acc = acc + v * v;
  }
  for (int o = 16; o > 0; o >>= 1) acc = acc + __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) part[0] = v;
  }
  __syncthreads();
  tot = part[0];
  __syncthreads();
  return tot;
}

// the whole V-cycle of the tail levels by one CTA in shared memory
template <int DIM>
__device__ void tail_run(const TailArgs& a, const double* __restrict__ b_in, double* u_io,
                         int zero_guess, int ncycles, double* sm, const TolArgs& tol) {
  const TailLevel& L0 = a.lv[0];
  if (DIM == 3 && a.fast) {
    ft_stamp(a);
    for (int i = threadIdx.x; i < a.m * a.m + 2 * a.m; i += blockDim.x) sm[a.lu_off + i] = a.lu[i];
    // zero guess: the first red pass of level 0 is fused into the load
    const bool fz = zero_guess && a.pre > 0;
    const double d0 = shifted_diag<3>(L0.g, L0.c, a.sigma, 1, 1, 1), d0r = rcp_diag(d0);
    PL_FOR_SM_POINTS(L0.g) {
      int x, y, z;
      decode(L0.g, p, x, y, z);
      const long long gi = a.g0.at(x, y, z);
      const double bv = b_in[gi];
      sm[L0.off_b + p] = bv;
      if (!zero_guess) sm[L0.off_u + p] = u_io[gi];
      else if (fz) sm[L0.off_u + p] = ft_red0(bv, a.omega, d0, d0r, x, y, z);
    }
    __syncthreads();
    ft_stamp(a);
    for (int cyc = 0; cyc < ncycles; ++cyc) {
      if (a.fast == 15) ft_level<15, 0>(a, sm, zero_guess && cyc == 0, fz && cyc == 0);
      else ft_level<7, 0>(a, sm, zero_guess && cyc == 0, fz && cyc == 0);
    }
    PL_FOR_SM_POINTS(L0.g) {
      int x, y, z;
      decode(L0.g, p, x, y, z);
      u_io[a.g0.at(x, y, z)] = sm[L0.off_u + p];
    }
    ft_stamp(a);
    return;
  }
  if (a.lu_off >= 0)
    for (int i = threadIdx.x; i < a.m * a.m + 2 * a.m; i += blockDim.x) sm[a.lu_off + i] = a.lu[i];
  PL_FOR_SM_POINTS(L0.g) {
    int x, y, z;
    decode(L0.g, p, x, y, z);
    const long long gi = a.g0.at(x, y, z);
    sm[L0.off_b + p] = b_in[gi];
    if (!zero_guess) sm[L0.off_u + p] = u_io[gi];
  }
  __syncthreads();
  if (tol.on) {
    // ToTolerance (multigrid.py:270-288), entirely on the device
    const double bn = sqrt(tail_sumsq<DIM>(a, sm, false));
    int c = 0, st = 1;
    double res = 0.0;
    if (bn == 0.0) {
      PL_FOR_SM_POINTS(L0.g) sm[L0.off_u + p] = 0.0;
      __syncthreads();
    } else {
      res = sqrt(tail_sumsq<DIM>(a, sm, true));
      while (res > tol.tol * bn) {
        if (c >= tol.max_cycles) {
          st = -1;
          break;
        }
        tail_vcycle<DIM>(a, sm, false);
        ++c;
        const double nres = sqrt(tail_sumsq<DIM>(a, sm, true));
        if (nres > tol.tol * bn && nres >= tol.stall * res) {
          st = 2;
          res = nres;
          break;
        }
        res = nres;
      }
    }
    if (threadIdx.x == 0) {
      tol.out[0] = res;
      tol.out[1] = 4.0 * c + (st + 1);
      tol.out[2] = bn;
    }
    if (st == -1) return;          // the failed solve leaves u untouched
  } else {
    for (int cyc = 0; cyc < ncycles; ++cyc) tail_vcycle<DIM>(a, sm, zero_guess && cyc == 0);
  }
  PL_FOR_SM_POINTS(L0.g) {
    int x, y, z;
    decode(L0.g, p, x, y, z);
    u_io[a.g0.at(x, y, z)] = sm[L0.off_u + p];
  }
}

template <int DIM>
__global__ void __launch_bounds__(TAIL_THREADS) k_tail(TailArgs a,
                                                       const double* __restrict__ b_in,
                                                       double* u_io, int zero_guess,
                                                       int ncycles, TolArgs tol) {
  extern __shared__ double sm[];
  tail_run<DIM>(a, b_in, u_io, zero_guess, ncycles, sm, tol);
}

// ---------------------------------------------------------------------------
// cooperative "mid" V-cycle: the grid-wide levels below the TMA threshold plus
// the tail in ONE persistent launch.  Each former kernel becomes a phase of a
// grid-stride loop separated by grid-wide barriers: per level and sweep one
// red and one black phase (colour points only, in place), then residual and
// full weighting on the way down; prolongation and the post-sweeps on the way
// up; CTA 0 runs the tail levels (shared memory, dense LU) in between.  The
// per-point arithmetic is that of k_rb / k_residual / fw_point / lin_point,
// so results are bit-identical to the separate launches.

constexpr int MID_THREADS = 1024;
constexpr int MID_MAX = 8;

struct MidLevel {
  double* u;
  double* b;
  double* t;
  Geo g;
  OpC c;
  int pow2;   // order 2 with a power-of-two dx^2: mid_shifted / constant diagonal
};

// shifted_point's operations for order 2 and a power-of-two dx^2 (x / dx2 ==
// x * inv_dx2 exactly): axes z, y, x accumulated from 0.0, zero ghosts
__device__ __forceinline__ double mid_shifted(const double* __restrict__ u, const Geo& g,
                                             const OpC& c, double sigma, int x, int y, int z,
                                             long long idx) {
  const double c0 = u[idx];
  const double zm = z > 0 ? u[idx - g.sz] : 0.0, zp = z < g.nz - 1 ? u[idx + g.sz] : 0.0;
  const double ym = y > 0 ? u[idx - g.sy] : 0.0, yp = y < g.ny - 1 ? u[idx + g.sy] : 0.0;
  const double xm = x > 0 ? u[idx - 1] : 0.0, xp = x < g.nx - 1 ? u[idx + 1] : 0.0;
  double acc = 0.0;
  acc = acc + ((zm - 2.0 * c0) + zp) * c.inv_dx2;
  acc = acc + ((ym - 2.0 * c0) + yp) * c.inv_dx2;
  acc = acc + ((xm - 2.0 * c0) + xp) * c.inv_dx2;
  return c0 - sigma * (c.nu * acc);
}

struct MidArgs {
  unsigned long long* trace;   // PL_MID_TRACE diagnostics: %globaltimer per phase (or null)
  int nmid;                 // grid-wide levels 0 .. nmid-1; level nmid starts the tail
  MidLevel lv[MID_MAX + 1];
  int pre, post;
  double omega, sigma;
  int zero;                 // level 0 starts from a zero guess
};

// one colour of jor-rb, in place (k_rb arithmetic); zero: u == 0 on entry,
// so red points get 0 + (omega b) / d and black points are set to 0
template <int DIM>
__device__ __forceinline__ void mid_colour(const MidLevel& L, const MidArgs& m, int red,
                                           bool zero, long long gt, long long gs) {
  const Geo& g = L.g;
  ConstDiag cd;
  cd.init<DIM>(g, L.c, m.sigma);
  if (zero) {
    for (long long t = gt; t < g.npts; t += gs) {
      int x, y, z;
      decode_point(g, t, x, y, z);
      const long long idx = g.at(x, y, z);
      if (is_red<DIM>(x, y, z)) {
        L.u[idx] = 0.0 + cd.div<DIM>(m.omega * L.b[idx], g, L.c, m.sigma, x, y, z);
      } else {
        L.u[idx] = 0.0;
      }
    }
    return;
  }
  const int N = g.nx, H = (N + 1) / 2;
  const long long cnt = (long long)H * g.ny * g.nz;
  for (long long t = gt; t < cnt; t += gs) {
    const unsigned tt = (unsigned)t;
    const unsigned row = tt / (unsigned)H;
    const int h = (int)(tt - row * (unsigned)H);
    const int z = (int)(row / (unsigned)g.ny);
    const int y = (int)(row - (unsigned)z * (unsigned)g.ny);
    const int x = 2 * h + (((y + z + DIM) & 1) ^ red ^ 1);
    if (x >= N) continue;
    const long long idx = g.at(x, y, z);
    const double r = L.b[idx] - (DIM == 3 && L.pow2
                                     ? mid_shifted(L.u, g, L.c, m.sigma, x, y, z, idx)
                                     : shifted_point<DIM>(L.u, g, L.c, m.sigma, x, y, z, idx));
    L.u[idx] = L.u[idx] + cd.div<DIM>(m.omega * r, g, L.c, m.sigma, x, y, z);
  }
}

template <int DIM>
__global__ void __launch_bounds__(MID_THREADS) k_mid(MidArgs m, TailArgs ta) {
  cg::grid_group grid = cg::this_grid();
  int ph = 0;
#define MID_SYNC()                                                              \
  do {                                                                          \
    grid.sync();                                                                \
    if (m.trace && blockIdx.x == 0 && threadIdx.x == 0) {                       \
      unsigned long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
      if (ph < 63) m.trace[1 + ph++] = t_;                                      \
    }                                                                           \
  } while (0)
  if (m.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    m.trace[0] = t_;
  }
  extern __shared__ double sm[];
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (int l = 0; l < m.nmid; ++l) {
    const MidLevel& L = m.lv[l];
    const MidLevel& C = m.lv[l + 1];
    const bool zero = l == 0 ? m.zero != 0 : true;
    if (zero && m.pre == 0) {
      for (long long t = gt; t < L.g.nstore; t += gs) L.u[t] = 0.0;
      MID_SYNC();
    }
    for (int k = 0; k < m.pre; ++k) {
      mid_colour<DIM>(L, m, 1, zero && k == 0, gt, gs);
      MID_SYNC();
      mid_colour<DIM>(L, m, 0, false, gt, gs);
      MID_SYNC();
    }
    for (long long t = gt; t < L.g.npts; t += gs) {       // residual (k_residual)
      int x, y, z;
      decode_point(L.g, t, x, y, z);
      const long long idx = L.g.at(x, y, z);
      L.t[idx] = L.b[idx] - (DIM == 3 && L.pow2
                                 ? mid_shifted(L.u, L.g, L.c, m.sigma, x, y, z, idx)
                                 : shifted_point<DIM>(L.u, L.g, L.c, m.sigma, x, y, z, idx));
    }
    MID_SYNC();
    for (long long t = gt; t < C.g.npts; t += gs) {       // full weighting (k_fw)
      int x, y, z;
      decode_point(C.g, t, x, y, z);
      C.b[C.g.at(x, y, z)] = fw_point<DIM>(L.t, L.g, x, y, z);
    }
    MID_SYNC();
  }
  if (blockIdx.x == 0) tail_run<DIM>(ta, m.lv[m.nmid].b, m.lv[m.nmid].u, 1, 1, sm, TolArgs{});
  MID_SYNC();
  for (int l = m.nmid - 1; l >= 0; --l) {
    const MidLevel& L = m.lv[l];
    const MidLevel& C = m.lv[l + 1];
    for (long long t = gt; t < L.g.npts; t += gs) {       // u += P_lin e (k_prolong)
      int x, y, z;
      decode_point(L.g, t, x, y, z);
      const long long idx = L.g.at(x, y, z);
      L.u[idx] = L.u[idx] + lin_point<DIM>(C.u, C.g, x, y, z);
    }
    MID_SYNC();
    for (int k = 0; k < m.post; ++k) {
      mid_colour<DIM>(L, m, 1, false, gt, gs);
      MID_SYNC();
      mid_colour<DIM>(L, m, 0, false, gt, gs);
      if (l > 0 || k + 1 < m.post) MID_SYNC();
    }
  }
}
#undef MID_SYNC

}  // namespace

static int tail_args(MgPlan* P, int l0, double sigma, TailArgs& a, size_t* smem_out) {
  std::memset(&a, 0, sizeof(a));
  a.smoother = P->smoother;
  a.pre = P->pre;
  a.post = P->post;
  a.omega = P->omega;
  a.sigma = sigma;
  a.m = P->m_lu;
  auto it = P->lu.find(*(unsigned long long*)&sigma);
  if (it == P->lu.end()) {
    set_error("coarsest LU for sigma=%.17g not prepared", sigma);
    return -3;
  }
  a.lu = it->second.dev;
  int off = 0;
  a.nlev = (int)P->lv.size() - l0;
  a.g0 = P->lv[l0].g;
  for (int i = 0; i < a.nlev; ++i) {
    const MgLevel& L = P->lv[l0 + i];
    TailLevel& T = a.lv[i];
    T.g = make_geo_compact(P->dim, L.n);     // shared memory is dense
    T.c = L.c;
    T.coarsest = L.coarsest;
    int np = (int)L.g.npts;
    T.off_u = off; off += np;
    T.off_b = off; off += np;
    T.off_t = off; off += np;
  }
  a.lu_off = -1;
  const int lu_n = a.m * a.m + 2 * a.m;
  if (sizeof(double) * (off + lu_n) <= TAIL_SMEM_BUDGET + 8192) {
    a.lu_off = off;
    off += lu_n;
  }
  // compile-time-sized path: 3-D order-2 jor-rb, levels 15 -> 7 -> 3 or 7 -> 3
  a.fast = 0;
  {
    const int N0 = P->lv[l0].g.N;
    bool chain = P->dim == 3 && P->order == 2 && P->smoother == SM_RB && a.lu_off >= 0 &&
                 a.m == 27 && g_fast_tail && (N0 == 15 || N0 == 7);
    // ft_shifted multiplies by 1 / dx^2: exact only for power-of-two dx^2
    for (int i = 0, n = N0; chain && i < a.nlev; ++i, n = (n - 1) / 2)
      chain = P->lv[l0 + i].g.N == n && (P->lv[l0 + i].coarsest == (n == 3)) &&
              P->lv[l0 + i].c.pow2;
    if (chain) a.fast = N0;
  }
  *smem_out = sizeof(double) * off;
  return 0;
}

static int launch_tail(MgPlan* P, int l0, double* u, const double* b, double sigma,
                       int zero_guess, int ncycles, cudaStream_t s,
                       const TolArgs& tol = TolArgs{}) {
  TailArgs a;
  size_t smem = 0;
  PL_TRY(tail_args(P, l0, sigma, a, &smem));
  if (tol.on) a.fast = 0;    // the device ToTolerance loop runs the generic levels
  void (*kern)(TailArgs, const double*, double*, int, int, TolArgs) =
      P->dim == 1 ? k_tail<1> : (P->dim == 2 ? k_tail<2> : k_tail<3>);
  static bool attr_set[4] = {false, false, false, false};
  if (!attr_set[P->dim]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TAIL_SMEM_BUDGET + 8192);
    attr_set[P->dim] = true;
  }
  PL_PRE(K_TAIL);
  kern<<<1, TAIL_THREADS, smem, s>>>(a, b, u, zero_guess, ncycles, tol);
  double bytes = 8.0 * P->lv[l0].g.npts * (zero_guess ? 2 : 3);
  PL_CHECK_LAUNCH(K_TAIL, bytes);
  return 0;
}

int g_mid_enabled = 1;      // PL_OPT_MID
int g_mid_tail_n = 15;      // PL_OPT_MID_TAIL_N: largest N the mid kernel leaves to its tail
int g_mid_ctas = 0;         // PL_OPT_MID_CTAS: CTAs of the cooperative mid kernels (0: one per SM)

// first tail level of the mid kernel (>= the plan's tail_start)
static int mid_tail_level(const MgPlan* P) {
  for (int l = 0; l < (int)P->lv.size(); ++l)
    if (l >= P->tail_start && P->lv[l].g.N <= g_mid_tail_n) return l;
  return P->tail_start;
}

static bool mid_applies(const MgPlan* P, int l) {
  return g_mid_enabled && P->dim == 3 && P->order == 2 && P->smoother == SM_RB &&
         l < mid_tail_level(P) && mid_tail_level(P) - l <= MID_MAX;
}

static int launch_mid(MgPlan* P, int l0, double* u, const double* b, double sigma, int zero,
                      cudaStream_t s) {
  const int lt = mid_tail_level(P);
  MidArgs m;
  std::memset(&m, 0, sizeof(m));
  m.nmid = lt - l0;
  m.pre = P->pre;
  m.post = P->post;
  m.omega = P->omega;
  m.sigma = sigma;
  m.zero = zero;
  double bytes = 0.0;
  for (int i = 0; i <= m.nmid; ++i) {
    const MgLevel& L = P->lv[l0 + i];
    MidLevel& M = m.lv[i];
    M.u = i == 0 ? u : L.u;
    M.b = i == 0 ? const_cast<double*>(b) : L.b;
    M.t = L.t;
    M.g = L.g;
    M.c = L.c;
    M.pow2 = L.c.order == 2 && L.c.pow2;
    if (i < m.nmid) {   // the unfused kernels' algorithmic bytes
      const double np = (double)L.g.npts, nc = (double)P->lv[l0 + i + 1].g.npts;
      bytes += np * (24.0 * (P->pre + P->post) + 24.0 + 8.0 + 16.0) + nc * 16.0;
    }
  }
  TailArgs ta;
  size_t smem = 0;
  PL_TRY(tail_args(P, lt, sigma, ta, &smem));
  // one CTA per SM, cached per device once the occupancy check has passed
  static int grid_of[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& grid = grid_of[dev & 63];
  if (grid == 0) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_mid<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TAIL_SMEM_BUDGET + 8192);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mid<3>, MID_THREADS,
                                                  TAIL_SMEM_BUDGET + 8192);
    if (per < 1) {
      set_error("mid kernel does not fit one CTA per SM");
      return 2;
    }
    grid = sms;
  }
  const int nblk = g_mid_ctas > 0 && g_mid_ctas < grid ? g_mid_ctas : grid;
  static unsigned long long* trace = nullptr;
  static const bool tracing = std::getenv("PL_MID_TRACE") != nullptr;
  if (tracing && !trace) cudaMalloc(&trace, 128 * sizeof(unsigned long long));
  m.trace = tracing ? trace : nullptr;
  ta.trace = tracing ? trace + 64 : nullptr;
  if (tracing) cudaMemsetAsync(trace, 0, 128 * sizeof(unsigned long long), s);
  void* args[] = {&m, &ta};
  PL_PRE(K_MID);
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_mid<3>, nblk, MID_THREADS, args, smem, s);
  if (e != cudaSuccess) return cuda_status(e, "cooperative mid launch");
  bytes += 8.0 * P->lv[lt].g.npts * 3;
  if (tracing) {   // diagnostics only: per-phase durations of this launch
    unsigned long long h[64];
    cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "mid n=%d levels=%d:", P->lv[l0].g.N, m.nmid);
    for (int i = 1; i < 64 && h[i]; ++i) std::fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    std::fprintf(stderr, " us\n  tail phases:");
    unsigned long long ht[64];
    cudaMemcpyAsync(ht, trace + 64, sizeof(ht), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    for (int i = 2; i < 63 && i <= (int)ht[0]; ++i)
      std::fprintf(stderr, " %.2f", (ht[i] - ht[i - 1]) * 1e-3);
    std::fprintf(stderr, " us\n");
  }
  PL_CHECK_LAUNCH(K_MID, bytes);
  return 0;
}

// ---------------------------------------------------------------------------
// plan

static std::vector<int> level_ns(int n, int coarsest_n) {
  std::vector<int> ns;
  int m = n;
  while (true) {
    ns.push_back(m);
    if (m <= coarsest_n || m < 4) break;
    m /= 2;
  }
  return ns;
}

size_t mg_workspace_bytes(int dim, int n, int coarsest_n) {
  std::vector<int> ns = level_ns(n, coarsest_n);
  size_t total = 0;
  for (size_t l = 0; l < ns.size(); ++l) {
    Geo g = make_geo(dim, ns[l]);
    size_t per = (l == 0 ? 1 : 3) * (size_t)g.nstore;   // fine: t only; coarse: u, b, t
    total += ((per * 8 + 255) / 256) * 256;
  }
  return total;
}

int mg_plan_create(MgPlan** out, int dim, int n, double length, double nu, int order,
                   int smoother, double omega, int pre, int post, int coarsest_n, void* ws,
                   size_t ws_bytes) {
  if (dim < 1 || dim > 3 || n < 2 || (n & (n - 1))) {
    set_error("bad grid dim=%d n=%d", dim, n);
    return -1;
  }
  if (order != 2 && order != 4) {
    set_error("stencil order must be 2 or 4");
    return -1;
  }
  if (smoother != SM_JACOBI && smoother != SM_RB && smoother != SM_GS) {
    set_error("smoother %d is not implemented on the GPU path", smoother);
    return -2;
  }
  if (pre < 0 || post < 0 || coarsest_n < 2) {
    set_error("bad MG configuration");
    return -1;
  }
  size_t need = mg_workspace_bytes(dim, n, coarsest_n);
  if (ws_bytes < need) {
    set_error("MG workspace too small: %zu < %zu", ws_bytes, need);
    return -1;
  }
  MgPlan* P = new MgPlan();
  P->dim = dim; P->n = n; P->order = order; P->smoother = smoother;
  P->pre = pre; P->post = post; P->coarsest_n = coarsest_n;
  P->length = length; P->nu = nu; P->omega = omega;
  P->ws = (char*)ws; P->ws_bytes = ws_bytes;
  std::vector<int> ns = level_ns(n, coarsest_n);
  char* cur = (char*)ws;
  for (size_t l = 0; l < ns.size(); ++l) {
    MgLevel L;
    L.n = ns[l];
    L.g = make_geo(dim, ns[l]);
    L.c = make_opc(ns[l], length, nu, order);
    L.coarsest = ns[l] <= coarsest_n || ns[l] < 4;
    size_t per = (l == 0 ? 1 : 3) * (size_t)L.g.nstore;
    double* base = (double*)cur;
    if (l == 0) {
      L.t = base;
    } else {
      L.u = base;
      L.b = base + L.g.nstore;
      L.t = base + 2 * L.g.nstore;
    }
    cur += ((per * 8 + 255) / 256) * 256;
    P->lv.push_back(L);
  }
  P->m_lu = (int)P->lv.back().g.npts;
  // tail: deepest suffix of levels whose u, b, t fit the shared-memory budget
  size_t acc = 0;
  int start = (int)P->lv.size();
  for (int l = (int)P->lv.size() - 1; l >= 0; --l) {
    size_t lvl = 3 * sizeof(double) * (size_t)P->lv[l].g.npts;
    if (acc + lvl > TAIL_SMEM_BUDGET) break;
    acc += lvl;
    start = l;
  }
  if (start == (int)P->lv.size()) {
    delete P;
    set_error("coarsest grid does not fit the tail kernel");
    return -1;
  }
  P->tail_start = start;
  P->tail_smem = acc;
  // norms
  P->npartials = sumsq_partials(P->lv[0].g);
  cudaError_t e = cudaMalloc(&P->partials, sizeof(double) * (P->npartials + 4));
  if (e != cudaSuccess) {
    delete P;
    return cuda_status(e, "cudaMalloc partials");
  }
  P->norm_dev = P->partials + P->npartials;
  e = cudaMallocHost(&P->norm_host, 4 * sizeof(double));
  if (e != cudaSuccess) {
    cudaFree(P->partials);
    delete P;
    return cuda_status(e, "cudaMallocHost");
  }
  *out = P;
  return 0;
}

void mg_plan_destroy(MgPlan* P) {
  if (!P) return;
  for (auto& kv : P->lu) {
    cudaFree(kv.second.dev);
    cudaFreeHost(kv.second.host);
  }
  cudaFree(P->partials);
  cudaFreeHost(P->norm_host);
  mg_direct_destroy(P);
  delete P;
}

// Dense I - sigma A on the coarsest grid with the reference's entry values
// (multigrid.py:86-135: 1-D stencils / dx2, Kronecker sum in axis order,
// times nu, identity minus sigma times it), then partial-pivoting LU.
static void coarsest_lu_host(const MgPlan* P, double sigma, double* out) {
  const MgLevel& L = P->lv.back();
  const int N = L.g.N, d = P->dim, m = (int)L.g.npts;
  const double dx2 = L.c.dx2;
  std::vector<double> d1((size_t)N * N, 0.0);
  for (int i = 0; i < N; ++i) {
    if (P->order == 2) {
      d1[i * N + i] = -2.0 / dx2;
      if (i > 0) d1[i * N + i - 1] = 1.0 / dx2;
      if (i < N - 1) d1[i * N + i + 1] = 1.0 / dx2;
    } else if (i == 0 || i == N - 1) {
      d1[i * N + i] = -2.0 / dx2;
      if (i > 0) d1[i * N + i - 1] = 1.0 / dx2;
      if (i < N - 1) d1[i * N + i + 1] = 1.0 / dx2;
    } else {
      const int offs[5] = {-2, -1, 0, 1, 2};
      const double ws[5] = {-1.0, 16.0, -30.0, 16.0, -1.0};
      for (int q = 0; q < 5; ++q) {
        int j = i + offs[q];
        if (j >= 0 && j < N) d1[i * N + j] = ws[q] / (12.0 * dx2);
      }
    }
  }
  std::vector<double> A((size_t)m * m, 0.0);
  auto coord = [&](int p, int axis) {   // axis 0 slowest
    int c[3] = {0, 0, 0};
    int r = p;
    for (int ax = d - 1; ax >= 0; --ax) { c[ax] = r % N; r /= N; }
    return c[axis];
  };
  for (int p = 0; p < m; ++p)
    for (int q = 0; q < m; ++q) {
      double total = 0.0;
      bool any = false;
      for (int ax = 0; ax < d; ++ax) {
        bool same = true;
        for (int o = 0; o < d; ++o)
          if (o != ax && coord(p, o) != coord(q, o)) same = false;
        if (!same) continue;
        double v = d1[coord(p, ax) * N + coord(q, ax)];
        if (v == 0.0) continue;
        total = any ? total + v : v;
        any = true;
      }
      double a = P->nu * total;
      A[(size_t)p * m + q] = (p == q ? 1.0 : 0.0) - sigma * a;
    }
  std::vector<double> piv(m);
  for (int k = 0; k < m; ++k) {
    int pr = k;
    double best = std::fabs(A[(size_t)k * m + k]);
    for (int i = k + 1; i < m; ++i) {
      double v = std::fabs(A[(size_t)i * m + k]);
      if (v > best) { best = v; pr = i; }
    }
    piv[k] = pr;
    if (pr != k)
      for (int j = 0; j < m; ++j) std::swap(A[(size_t)k * m + j], A[(size_t)pr * m + j]);
    double inv = 1.0 / A[(size_t)k * m + k];
    for (int i = k + 1; i < m; ++i) A[(size_t)i * m + k] = A[(size_t)i * m + k] * inv;
    for (int i = k + 1; i < m; ++i) {
      double lik = A[(size_t)i * m + k];
      if (lik == 0.0) continue;
      for (int j = k + 1; j < m; ++j)
        A[(size_t)i * m + j] = A[(size_t)i * m + j] - lik * A[(size_t)k * m + j];
    }
  }
  std::memcpy(out, A.data(), sizeof(double) * (size_t)m * m);
  std::memcpy(out + (size_t)m * m, piv.data(), sizeof(double) * m);
}

// RN(1 / U_jj) after the m x m factors and the m pivots (0: IEEE division):
// the device solves divide by the diagonal with div_diag, whose quotient is
// the IEEE one
static void lu_reciprocals(int m, double* e) {
  for (int j = 0; j < m; ++j) {
    const double d = e[(size_t)j * m + j];
    e[(size_t)m * m + m + j] = diag_div_ok(d) ? 1.0 / d : 0.0;
  }
}

static int lu_entry(MgPlan* P, double sigma, LuEntry** out) {
  unsigned long long key = *(unsigned long long*)&sigma;
  auto it = P->lu.find(key);
  if (it != P->lu.end()) {
    *out = &it->second;
    return 0;
  }
  size_t count = (size_t)P->m_lu * P->m_lu + 2 * (size_t)P->m_lu;
  LuEntry E;
  cudaError_t e = cudaMallocHost(&E.host, count * sizeof(double));
  if (e != cudaSuccess) return cuda_status(e, "cudaMallocHost lu");
  e = cudaMalloc(&E.dev, count * sizeof(double));
  if (e != cudaSuccess) {
    cudaFreeHost(E.host);
    return cuda_status(e, "cudaMalloc lu");
  }
  P->lu[key] = E;
  *out = &P->lu[key];
  return 1;   // new, not filled
}

int mg_prepare(MgPlan* P, double sigma, cudaStream_t s) {
  LuEntry* E = nullptr;
  int rc = lu_entry(P, sigma, &E);
  if (rc <= 0) return rc;
  size_t count = (size_t)P->m_lu * P->m_lu + 2 * (size_t)P->m_lu;
  coarsest_lu_host(P, sigma, E->host);
  lu_reciprocals(P->m_lu, E->host);
  cudaError_t e = cudaMemcpyAsync(E->dev, E->host, count * sizeof(double),
                                  cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "upload lu");
  return 0;
}

int mg_set_coarsest_lu(MgPlan* P, double sigma, const double* lu, const int* piv,
                       cudaStream_t s) {
  LuEntry* E = nullptr;
  int rc = lu_entry(P, sigma, &E);
  if (rc < 0) return rc;
  const size_t mm = (size_t)P->m_lu * P->m_lu;
  // the previous upload of this entry must have landed before the staging
  // buffer is rewritten
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "sync");
  std::memcpy(E->host, lu, sizeof(double) * mm);
  for (int i = 0; i < P->m_lu; ++i) E->host[mm + i] = (double)piv[i];
  lu_reciprocals(P->m_lu, E->host);
  e = cudaMemcpyAsync(E->dev, E->host, (mm + 2 * P->m_lu) * sizeof(double),
                      cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "upload lu");
  return 0;
}

// ---------------------------------------------------------------------------
// grid-wide levels

// sweeps on a grid-wide level; *cur holds the iterate (u or t) and is updated
static int level_smooth(MgPlan* P, MgLevel& L, double** cur, double* alt_u, const double* b,
                        double sigma, int count, bool zero, cudaStream_t s) {
  double* u = *cur;
  double* other = (u == alt_u) ? L.t : alt_u;
  if (count == 0) {
    if (zero) {
      cudaError_t e = cudaMemsetAsync(u, 0, sizeof(double) * L.g.nstore, s);
      if (e != cudaSuccess) return cuda_status(e, "memset");
    }
    return 0;
  }
  const bool fused = zmarch_ok(L.g, L.c);
  if (P->smoother == SM_GS) {   // in place; t is the solve's scratch
    if (zero) {
      cudaError_t e = cudaMemsetAsync(u, 0, sizeof(double) * L.g.nstore, s);
      if (e != cudaSuccess) return cuda_status(e, "memset");
    }
    double* scratch = (u == L.t) ? alt_u : L.t;
    PL_TRY(launch_gs(u, b, scratch, L.g, L.c, sigma, count, s));
    *cur = u;
    return 0;
  }
  if (P->smoother == SM_JACOBI) {
    int k = 0;
    if (fused) {             // pairs of sweeps in one pass (temporal blocking)
      for (; k + 1 < count; k += 2) {
        PL_TRY(zlaunch_jacobi2(u, b, other, L.g, L.c, sigma, P->omega, zero && k == 0, nullptr,
                               s));
        std::swap(u, other);
      }
    }
    for (; k < count; ++k) {
      PL_TRY(launch_jacobi(u, b, other, L.g, L.c, sigma, P->omega, zero && k == 0, s));
      std::swap(u, other);
    }
    *cur = u;
    return 0;
  }
  if (zero) {
    cudaError_t e = cudaMemsetAsync(u, 0, sizeof(double) * L.g.nstore, s);
    if (e != cudaSuccess) return cuda_status(e, "memset");
  }
  for (int k = 0; k < count; ++k) {
    if (fused) {            // red and black in one pass, out of place
      PL_TRY(zlaunch_rb(u, b, other, L.g, L.c, sigma, P->omega, s));
      std::swap(u, other);
    } else if (P->order == 2) {    // same-colour points never neighbour: in place
      PL_TRY(launch_rb(u, b, u, L.g, L.c, sigma, P->omega, 1, s));
      PL_TRY(launch_rb(u, b, u, L.g, L.c, sigma, P->omega, 0, s));
    } else {                // order 4: +-2 neighbours share the colour
      PL_TRY(launch_rb(u, b, other, L.g, L.c, sigma, P->omega, 1, s));
      PL_TRY(launch_rb(other, b, u, L.g, L.c, sigma, P->omega, 0, s));
    }
  }
  *cur = u;
  return 0;
}

static int vcycle(MgPlan* P, int l, double* u, const double* b, double sigma, bool zero,
                  cudaStream_t s) {
  if (l >= P->tail_start) return launch_tail(P, l, u, b, sigma, zero, 1, s);
  if (!zmarch_ok(P->lv[l].g, P->lv[l].c) && mid_applies(P, l))
    return launch_mid(P, l, u, b, sigma, zero, s);
  MgLevel& L = P->lv[l];
  MgLevel& C = P->lv[l + 1];
  double* cur = u;
  const bool zm = zmarch_ok(L.g, L.c);
  PL_TRY(level_smooth(P, L, &cur, u, b, sigma, P->pre, zero, s));
  if (zm && zmarch_rfw()) {
    PL_TRY(zlaunch_rfw(cur, b, C.b, L.g, L.c, sigma, s));
  } else {
    double* r = (cur == u) ? L.t : u;
    PL_TRY(launch_residual(cur, b, r, L.g, L.c, sigma, s));
    PL_TRY(launch_fw(r, C.b, L.g, s));
  }
  PL_TRY(vcycle(P, l + 1, C.u, C.b, sigma, true, s));
  // u += P e_c, then post-smoothing (multigrid.py:250-251); with
  // PL_OPT_FUSE_PROLONG the Jacobi pair on the TMA levels does both
  int post = P->post;
  if (zmarch_ok(L.g, L.c) && zmarch_fuse_prolong() && P->smoother == SM_JACOBI &&
             post >= 2) {
    double* other = (cur == u) ? L.t : u;
    PL_TRY(zlaunch_jacobi2(cur, b, other, L.g, L.c, sigma, P->omega, 0, C.u, s));
    cur = other;
    post -= 2;
  } else {
    PL_TRY(launch_prolong(C.u, cur, L.g, 1, s));
  }
  PL_TRY(level_smooth(P, L, &cur, u, b, sigma, post, false, s));
  if (cur != u) {
    cudaError_t e = cudaMemcpyAsync(u, cur, sizeof(double) * L.g.nstore,
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "copy");
    count_launch(K_COPY, 16.0 * L.g.npts);
  }
  return 0;
}

int mg_cycles(MgPlan* P, double* u, const double* b, double sigma, int ncycles, int zero_guess,
              cudaStream_t s) {
  PL_TRY(mg_prepare(P, sigma, s));
  if (P->tail_start == 0) return launch_tail(P, 0, u, b, sigma, zero_guess, ncycles, s);
  for (int c = 0; c < ncycles; ++c)
    PL_TRY(vcycle(P, 0, u, b, sigma, zero_guess && c == 0, s));
  return 0;
}

int mg_smooth(MgPlan* P, double* u, const double* b, double sigma, int count, cudaStream_t s) {
  MgLevel& L = P->lv[0];
  double* cur = u;
  PL_TRY(level_smooth(P, L, &cur, u, b, sigma, count, false, s));
  if (cur != u) {
    cudaError_t e = cudaMemcpyAsync(u, cur, sizeof(double) * L.g.nstore,
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "copy");
  }
  return 0;
}

static int norm2(MgPlan* P, const double* u, const double* b, double sigma, double* out,
                 cudaStream_t s) {
  MgLevel& L = P->lv[0];
  PL_TRY(launch_sumsq(u, b, L.g, L.c, sigma, P->partials, P->npartials, P->norm_dev, s));
  cudaError_t e = cudaMemcpyAsync(P->norm_host, P->norm_dev, sizeof(double),
                                  cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_status(e, "norm readback");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "sync");
  *out = std::sqrt(P->norm_host[0]);
  return 0;
}

int g_tol_device = 1;   // PL_OPT_TOL_DEVICE

int mg_solve_tol(MgPlan* P, double* u, const double* b, double sigma, double tol, double stall,
                 int max_cycles, int* cycles, int* status, double* residual, cudaStream_t s) {
  PL_TRY(mg_prepare(P, sigma, s));
  MgLevel& L = P->lv[0];
  if (g_tol_device && P->tail_start == 0) {
    // the whole solve in one single-CTA launch, one readback
    TolArgs ta{1, tol, stall, max_cycles, P->norm_dev};
    PL_TRY(launch_tail(P, 0, u, b, sigma, 0, 0, s, ta));
    cudaError_t e = cudaMemcpyAsync(P->norm_host, P->norm_dev, 3 * sizeof(double),
                                    cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_status(e, "tolerance readback");
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "sync");
    const long long code = (long long)P->norm_host[1];
    const int st = (int)(code & 3) - 1;
    *cycles = (int)(code >> 2);
    *residual = P->norm_host[0];
    if (st < 0) {
      *status = -1;
      set_error("no convergence after %d V-cycles (relative residual %.3e)", *cycles,
                *residual / P->norm_host[2]);
      return 1;
    }
    *status = st == 2 ? ST_STALLED : ST_CONVERGED;
    return 0;
  }
  double bnorm;
  PL_TRY(norm2(P, nullptr, b, sigma, &bnorm, s));
  *cycles = 0;
  if (bnorm == 0.0) {
    cudaError_t e = cudaMemsetAsync(u, 0, sizeof(double) * L.g.nstore, s);
    if (e != cudaSuccess) return cuda_status(e, "memset");
    *status = ST_CONVERGED;
    *residual = 0.0;
    return 0;
  }
  double res;
  PL_TRY(norm2(P, u, b, sigma, &res, s));
  int c = 0;
  while (res > tol * bnorm) {
    if (c >= max_cycles) {
      *cycles = c;
      *residual = res;
      *status = -1;
      set_error("no convergence after %d V-cycles (relative residual %.3e)", c, res / bnorm);
      return 1;
    }
    PL_TRY(mg_cycles(P, u, b, sigma, 1, 0, s));
    ++c;
    double nres;
    PL_TRY(norm2(P, u, b, sigma, &nres, s));
    if (nres > tol * bnorm && nres >= stall * res) {
      *cycles = c;
      *status = ST_STALLED;
      *residual = nres;
      return 0;
    }
    res = nres;
  }
  *cycles = c;
  *status = ST_CONVERGED;
  *residual = res;
  return 0;
}

}  // namespace pl
