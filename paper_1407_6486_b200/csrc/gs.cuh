// Lexicographic Gauss-Seidel (multigrid.py:219-224): u += (D + L)^-1 (b - A_sigma u).
//
// The reference solves the lower-triangular system with
// scipy.linalg.solve_banded on the lower band of the shifted matrix, i.e.
// LAPACK gbtrf/gbtrs.  Without pivoting (the diagonal dominates every
// column) that is, bit for bit (checked in oracle/gs_order.py):
//   l_ij = A_ij * RN(1 / D_j)                       (gbtrf DSCAL by ONE/pivot)
//   y_i  = r_i;  y_i = fma(-y_j, l_ij, y_i) for the lower neighbours j of i in
//          increasing linear index, i.e. axis 0 first, offset -2 before -1
//                                                   (gbtrs DGER, FMA)
//   du_i = y_i / D_i                                 (gbtrs DTBSV, true division)
// with the matrix entries of multigrid.py:86-135:
//   A_ij = -(sigma * (nu * w)), w = 1/dx^2 (order 2 and the boundary-adjacent
//   rows of order 4), -1/(12 dx^2) and 16/(12 dx^2) (order-4 offsets -2, -1).
// The dependency structure is the hyperplane x + y + z = s: every point of a
// hyperplane depends only on the two previous ones, so the GPU sweeps the
// hyperplanes in order and updates each in parallel.
#pragma once
#include "common.cuh"

namespace pl {

// y_i after the lower neighbours along one axis (position ia of extent na,
// linear stride st); jd(k) gives D_j of the neighbour at offset -k
template <typename DiagFn>
__device__ __forceinline__ double gs_axis(const double* __restrict__ yv, double yi, long long idx,
                                          long long st, int ia, int na, const OpC& c,
                                          double sigma, DiagFn jd) {
  if (c.order == 2 || ia == 0 || ia == na - 1) {
    if (ia >= 1) {
      const double a = -(sigma * (c.nu * c.inv_dx2));
      yi = __fma_rn(-yv[idx - st], a * (1.0 / jd(1)), yi);
    }
    return yi;
  }
  if (ia >= 2) {
    const double a = -(sigma * (c.nu * (-1.0 / c.d12)));
    yi = __fma_rn(-yv[idx - 2 * st], a * (1.0 / jd(2)), yi);
  }
  const double a = -(sigma * (c.nu * (16.0 / c.d12)));
  return __fma_rn(-yv[idx - st], a * (1.0 / jd(1)), yi);
}

// y_i of (D + L) y = r at (x, y, z); yv holds the final y of every lower
// neighbour (strides of g), ri = r_i
template <int DIM>
__device__ __forceinline__ double gs_lower_point(const double* __restrict__ yv, double ri,
                                                 const Geo& g, const OpC& c, double sigma,
                                                 int x, int y, int z, long long idx) {
  double yi = ri;
  if (DIM == 3)
    yi = gs_axis(yv, yi, idx, g.sz, z, g.nz, c, sigma,
                 [&](int k) { return shifted_diag<DIM>(g, c, sigma, x, y, z - k); });
  if (DIM >= 2)
    yi = gs_axis(yv, yi, idx, g.sy, y, g.ny, c, sigma,
                 [&](int k) { return shifted_diag<DIM>(g, c, sigma, x, y - k, z); });
  yi = gs_axis(yv, yi, idx, 1, x, g.nx, c, sigma,
               [&](int k) { return shifted_diag<DIM>(g, c, sigma, x - k, y, z); });
  return yi;
}

}  // namespace pl
