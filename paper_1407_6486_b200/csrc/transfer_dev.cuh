// Device-side transfer arithmetic shared by the grid-wide kernels
// (transfer.cu) and the single-CTA multigrid tail (mg.cu).  Evaluation trees
// restate transfers.py exactly: per axis, axis 0 first, one rounding per op.
#pragma once
#include "common.cuh"

namespace pl {

// one FW stencil along an axis: 0.25 * ((a + 2 b) + c)   transfers.py:30
__device__ __forceinline__ double fw3(double a, double b, double c) {
  return 0.25 * ((a + 2.0 * b) + c);
}

// FW value at coarse (jx, jy, jz) from fine field f (geometry gf).
template <int DIM>
__device__ __forceinline__ double fw_point(const double* __restrict__ f, const Geo& gf,
                                           int jx, int jy, int jz) {
  if (DIM == 1) return fw3(f[2 * jx], f[2 * jx + 1], f[2 * jx + 2]);
  if (DIM == 2) {
    double zx[3];
    for (int dx = 0; dx < 3; ++dx) {
      long long base = (long long)(2 * jy) * gf.sy + 2 * jx + dx;
      zx[dx] = fw3(f[base], f[base + gf.sy], f[base + 2 * gf.sy]);    // axis 0 (y)
    }
    return fw3(zx[0], zx[1], zx[2]);                                   // axis 1 (x)
  }
  double yx[3];
  for (int dx = 0; dx < 3; ++dx) {
    double zy[3];
    for (int dy = 0; dy < 3; ++dy) {
      long long base = (long long)(2 * jz) * gf.sz + (long long)(2 * jy + dy) * gf.sy +
                       2 * jx + dx;
      zy[dy] = fw3(f[base], f[base + gf.sz], f[base + 2 * gf.sz]);    // axis 0 (z)
    }
    yx[dx] = fw3(zy[0], zy[1], zy[2]);                                // axis 1 (y)
  }
  return fw3(yx[0], yx[1], yx[2]);                                     // axis 2 (x)
}

// Linear interpolation taps along one axis for fine array index i
// (transfers.py:40-45): odd i copies coarse (i-1)/2; even i averages coarse
// i/2-1 and i/2 with zero outside [0, nc1).
struct LinTap {
  int j0, j1;
  bool two;
};
__device__ __forceinline__ LinTap lin_tap(int i) {
  LinTap t;
  if (i & 1) {
    t.j0 = (i - 1) >> 1; t.j1 = -1; t.two = false;
  } else {
    t.j0 = (i >> 1) - 1; t.j1 = i >> 1; t.two = true;
  }
  return t;
}
__device__ __forceinline__ double lin_comb(double a, double b, bool two) {
  return two ? 0.5 * (a + b) : a;
}

template <int DIM>
__device__ __forceinline__ double lin_point(const double* __restrict__ c, const Geo& gc,
                                            int ix, int iy, int iz) {
  auto ld = [&](int jz, int jy, int jx) -> double {
    if (jx < 0 || jx >= gc.nx) return 0.0;
    if (DIM >= 2 && (jy < 0 || jy >= gc.ny)) return 0.0;
    if (DIM == 3 && (jz < 0 || jz >= gc.nz)) return 0.0;
    long long idx = jx;
    if (DIM >= 2) idx += (long long)jy * gc.sy;
    if (DIM == 3) idx += (long long)jz * gc.sz;
    return c[idx];
  };
  LinTap tx = lin_tap(ix);
  if (DIM == 1) return lin_comb(ld(0, 0, tx.j0), tx.two ? ld(0, 0, tx.j1) : 0.0, tx.two);
  LinTap ty = lin_tap(iy);
  if (DIM == 2) {
    // axis 0 (y) first, then x
    double a = lin_comb(ld(0, ty.j0, tx.j0), ty.two ? ld(0, ty.j1, tx.j0) : 0.0, ty.two);
    double b = 0.0;
    if (tx.two) b = lin_comb(ld(0, ty.j0, tx.j1), ty.two ? ld(0, ty.j1, tx.j1) : 0.0, ty.two);
    return lin_comb(a, b, tx.two);
  }
  // 3-D: all eight taps loaded unconditionally (out-of-range ones read as 0.0)
  // and combined by selects -- no lane-dependent loop trip counts, so a warp
  // whose lanes alternate odd/even x does not serialise the two tap paths.
  // lin_comb(a, b, false) == a for every b, so each result equals the
  // reference-order evaluation above bit for bit.
  LinTap tz = lin_tap(iz);
  double by[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int jx = a ? tx.j1 : tx.j0;
#pragma unroll
    for (int bidx = 0; bidx < 2; ++bidx) {
      const int jy = bidx ? ty.j1 : ty.j0;
      by[a][bidx] = lin_comb(ld(tz.j0, jy, jx), ld(tz.j1, jy, jx), tz.two);
    }
  }
  const double bx0 = lin_comb(by[0][0], by[0][1], ty.two);
  const double bx1 = lin_comb(by[1][0], by[1][1], ty.two);
  return lin_comb(bx0, bx1, tx.two);
}


}  // namespace pl
