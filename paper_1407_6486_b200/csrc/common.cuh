// Common definitions for the sm_100a PFASST x multigrid kernels.
//
// Numerics contract ("parity mode"): every element-wise
// expression evaluates exactly the reference's numpy expression tree, one
// IEEE rounding per operation, with FMA contraction disabled at compile time
// (-fmad=false).  The only FMAs are explicit __fma_rn chains that restate the
// reference's BLAS dgemm contractions (np.tensordot over the node axis), which
// the oracle tests showed to be a sequential fused multiply-add chain in
// column order.  Under that contract the stencil, smoother, transfer and
// quadrature kernels are bit-identical to numpy on the same inputs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace pl {

// ---------------------------------------------------------------------------
// error state / launch accounting

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);   // 0 or 2 (+ message)
void count_launch(int kind, double alg_bytes);       // runtime stats (capi.cu)
void timing_pre(int kind, cudaStream_t s);           // optional CUDA-event timing
void timing_post(int kind, cudaStream_t s, double alg_bytes);

// Bracket every kernel launch: PL_PRE(kind) before, PL_CHECK_LAUNCH after
// (both use the launcher's stream variable `s`).
#define PL_PRE(kind) ::pl::timing_pre(kind, s)
#define PL_CHECK_LAUNCH(kind, bytes)                                  \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::pl::cuda_status(_e, #kind);       \
    ::pl::count_launch(kind, bytes);                                  \
    ::pl::timing_post(kind, s, bytes);                                \
  } while (0)

#define PL_TRY(expr)                 \
  do {                               \
    int _s = (expr);                 \
    if (_s != 0) return _s;          \
  } while (0)

// kernel families for the launch counter / per-kernel event timing
enum KernelKind {
  K_APPLY = 0, K_JACOBI, K_RB, K_RESID, K_RESTRICT, K_PROLONG, K_TAIL,
  K_NORM, K_QUAD, K_RHS, K_RESMAX, K_FAS, K_CORR, K_INTERP, K_COPY, K_LU, K_MID, K_GS,
  K_DIRECT, K_APPLY_RHS, K_NUM_KINDS
};

// ---------------------------------------------------------------------------
// geometry: interior-only Dirichlet grid, C order, x fastest (heat.py:1-6).
//
// Device layout: for dim >= 2 every row of N = n-1 interior values is stored
// with a pitch of n doubles (one zero pad per row), so rows start 16-byte
// aligned and TMA tensor maps (strides must be multiples of 16 B) can address
// the field; the pad is outside the tensor map's extent and is never read as
// data.  1-D fields are a single unpadded row.  Pads hold zeros: buffers are
// zero-initialised and every point-wise kernel maps zeros to zeros.

struct Geo {
  int dim;        // 1, 2, 3
  int N;          // interior points per axis = n - 1
  int nx, ny, nz; // nz = ny = 1 for lower dims
  long long sy, sz;   // storage strides in elements
  long long npts;     // logical points (n-1)^dim
  long long nstore;   // storage elements per field (incl. pads)
  __host__ __device__ long long at(int x, int y, int z) const { return z * sz + y * sy + x; }
};

inline Geo make_geo_pitch(int dim, int n, int pitch) {
  Geo g;
  g.dim = dim;
  g.N = n - 1;
  g.nx = g.N;
  g.ny = dim >= 2 ? g.N : 1;
  g.nz = dim >= 3 ? g.N : 1;
  g.sy = pitch;
  g.sz = (long long)pitch * g.ny;
  g.npts = (long long)g.nx * g.ny * g.nz;
  g.nstore = g.sz * g.nz;
  return g;
}

// the device (storage) layout of a grid with n cells per axis
inline Geo make_geo(int dim, int n) { return make_geo_pitch(dim, n, dim >= 2 ? n : n - 1); }
// dense layout (shared-memory tiles, scratch)
inline Geo make_geo_compact(int dim, int n) { return make_geo_pitch(dim, n, n - 1); }

// logical linear index -> (x, y, z); 32-bit division (every grid here has
// fewer than 2^32 points; 64-bit division is a ~70-instruction subroutine)
__host__ __device__ inline void decode_point(const Geo& g, long long t, int& x, int& y, int& z) {
  const unsigned tt = (unsigned)t, nx = (unsigned)g.nx, ny = (unsigned)g.ny;
  const unsigned r = tt / nx;
  x = (int)(tt - r * nx);
  z = (int)(r / ny);
  y = (int)(r - (unsigned)z * ny);
}

// Operator constants, all computed on the host with the reference's own
// Python-float expressions (heat.py:114,148-152; multigrid.py:186).
struct OpC {
  double dx2;       // (length / n) ** 2
  double inv_dx2;   // 1 / dx2, used only when dx2 is a power of two (exact)
  double d12;       // 12.0 * dx2
  double nu;
  double d1_edge;   // -2.0 / dx2
  double d1_int;    // order 2: -2.0 / dx2 ; order 4: -30.0 / (12.0 * dx2)
  int order;
  int pow2;         // x / dx2 == x * inv_dx2 exactly
};

__device__ __forceinline__ double div_dx2(double x, const OpC& c) {
  return c.pow2 ? x * c.inv_dx2 : x / c.dx2;
}

// One axis term of heat.py:119-140 at position i of an axis of length N,
// given the neighbours along that axis (zero outside the domain).
__device__ __forceinline__ double axis_term(double m2, double m1, double c0,
                                            double p1, double p2, int i, int N,
                                            const OpC& c) {
  if (c.order == 2 || i == 0 || i == N - 1)
    return div_dx2((m1 - 2.0 * c0) + p1, c);
  return ((((-m2 + 16.0 * m1) - 30.0 * c0) + 16.0 * p1) - p2) / c.d12;
}

// nu * Lap(u) at point (x,y,z) reading u from memory `u` (global or shared)
// with strides of geometry g.  Axes accumulate slowest first from 0.0.
template <int DIM>
__device__ __forceinline__ double lap_point(const double* __restrict__ u,
                                            const Geo& g, const OpC& c,
                                            int x, int y, int z, long long idx) {
  const double c0 = u[idx];
  double acc = 0.0;
  if (DIM == 3) {
    double m1 = z > 0 ? u[idx - g.sz] : 0.0;
    double p1 = z < g.nz - 1 ? u[idx + g.sz] : 0.0;
    double m2 = 0.0, p2 = 0.0;
    if (c.order == 4) {
      m2 = z > 1 ? u[idx - 2 * g.sz] : 0.0;
      p2 = z < g.nz - 2 ? u[idx + 2 * g.sz] : 0.0;
    }
    acc = acc + axis_term(m2, m1, c0, p1, p2, z, g.nz, c);
  }
  if (DIM >= 2) {
    double m1 = y > 0 ? u[idx - g.sy] : 0.0;
    double p1 = y < g.ny - 1 ? u[idx + g.sy] : 0.0;
    double m2 = 0.0, p2 = 0.0;
    if (c.order == 4) {
      m2 = y > 1 ? u[idx - 2 * g.sy] : 0.0;
      p2 = y < g.ny - 2 ? u[idx + 2 * g.sy] : 0.0;
    }
    acc = acc + axis_term(m2, m1, c0, p1, p2, y, g.ny, c);
  }
  {
    double m1 = x > 0 ? u[idx - 1] : 0.0;
    double p1 = x < g.nx - 1 ? u[idx + 1] : 0.0;
    double m2 = 0.0, p2 = 0.0;
    if (c.order == 4) {
      m2 = x > 1 ? u[idx - 2] : 0.0;
      p2 = x < g.nx - 2 ? u[idx + 2] : 0.0;
    }
    acc = acc + axis_term(m2, m1, c0, p1, p2, x, g.nx, c);
  }
  return c.nu * acc;
}

// 1 - sigma * diag(nu Lap) at (x,y,z): heat.py:144-158, multigrid.py:186.
template <int DIM>
__device__ __forceinline__ double shifted_diag(const Geo& g, const OpC& c,
                                               double sigma, int x, int y, int z) {
  double t = 0.0;
  if (DIM == 3) t = t + ((c.order == 4 && (z == 0 || z == g.nz - 1)) ? c.d1_edge : c.d1_int);
  if (DIM >= 2) t = t + ((c.order == 4 && (y == 0 || y == g.ny - 1)) ? c.d1_edge : c.d1_int);
  t = t + ((c.order == 4 && (x == 0 || x == g.nx - 1)) ? c.d1_edge : c.d1_int);
  return 1.0 - sigma * (c.nu * t);
}

// (I - sigma A) u at a point: multigrid.py:192-193.
template <int DIM>
__device__ __forceinline__ double shifted_point(const double* __restrict__ u,
                                                const Geo& g, const OpC& c,
                                                double sigma, int x, int y, int z,
                                                long long idx) {
  return u[idx] - sigma * lap_point<DIM>(u, g, c, x, y, z, idx);
}

// Red points: even 1-based coordinate sum (multigrid.py:167-175).
template <int DIM>
__device__ __forceinline__ bool is_red(int x, int y, int z) {
  int s = x + 1;
  if (DIM >= 2) s += y + 1;
  if (DIM == 3) s += z + 1;
  return (s & 1) == 0;
}

__host__ __device__ inline int ceil_div(long long a, long long b) {
  return (int)((a + b - 1) / b);
}

// correctly rounded a / b given y = RN(1/b): q0 = RN(a y) is within 1.5 ulp,
// one Markstein correction makes it faithful, the second exact (Markstein's
// theorem: y within half an ulp of 1/b, q faithful, remainder exact by FMA).
// Zeros (sign), subnormals, huge values and non-finite a take the IEEE
// division.  (The coarsest LU's reciprocals come from the host; every other
// y is RN(1/b) computed once per thread for a constant diagonal.)
static __device__ __noinline__ double div_slow(double a, double b) { return a / b; }
static __device__ __forceinline__ double div_const(double a, double b, double y) {
  double q = a * y;
  double r = __fma_rn(-b, q, a);
  q = __fma_rn(r, y, q);
  r = __fma_rn(-b, q, a);
  q = __fma_rn(r, y, q);
  const double aa = fabs(a);
  if (__builtin_expect(!(aa >= 0x1p-960 && aa <= 0x1p960), 0)) q = div_slow(a, b);
  return q;
}

// div_const's preconditions for a divisor d used across a whole level: RN(1/d)
// normal and every quotient of an in-range a normal.  Otherwise the IEEE
// division is used (rd = 0 marks it).
__host__ __device__ inline bool diag_div_ok(double d) {
  const double ad = fabs(d);
  return ad >= 0x1p-64 && ad <= 0x1p64;
}
__device__ __forceinline__ double rcp_diag(double d) { return diag_div_ok(d) ? 1.0 / d : 0.0; }
__device__ __forceinline__ double div_diag(double a, double d, double rd) {
  return rd != 0.0 ? div_const(a, d, rd) : a / d;
}

// a / d for the shifted diagonal d of an order-2 level, which is one value for
// the whole level: dc and its reciprocal rc = RN(1/dc) are computed once per
// thread (ConstDiag) and the quotient is div_const's correctly rounded one --
// the same bits as the IEEE division.  Order 4 (boundary rows differ) divides.
struct ConstDiag {
  bool on;
  double d, r;
  template <int DIM>
  __device__ __forceinline__ void init(const Geo& g, const OpC& c, double sigma) {
    d = c.order == 2 ? shifted_diag<DIM>(g, c, sigma, 0, 0, 0) : 1.0;
    on = c.order == 2 && diag_div_ok(d);
    r = 1.0 / d;
  }
  template <int DIM>
  __device__ __forceinline__ double div(double a, const Geo& g, const OpC& c, double sigma,
                                        int x, int y, int z) const {
    return on ? div_const(a, d, r) : a / shifted_diag<DIM>(g, c, sigma, x, y, z);
  }
};

}  // namespace pl
