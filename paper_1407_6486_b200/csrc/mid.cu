// Small-level V-cycle with ONE grid-wide phase per level and direction
// (3-D, order 2, jor-rb; multigrid.py:211-251 below the TMA threshold).
//
// The earlier cooperative kernel (k_mid in mg.cu) mapped every former kernel
// to a grid phase: red, black, residual, full weighting on the way down,
// prolongation, red, black on the way up -- seven grid barriers per level,
// each ~3 us of barrier plus L2 latency -- and ran the levels below 15^3 on
// one CTA.  Here each CTA owns a tile, stages it with a halo in shared
// memory and runs the whole level step locally (overlapped tiling):
//
//   down(l): tile = a block of coarse points; its fine footprint R (the
//            points full weighting reads) plus a halo of 2*pre + 1 is staged
//            (u, or zeros for a zero guess, and b); the pre sweeps run on
//            shrinking boxes (a red point needs the black ring around it, a
//            black point the red ring), the residual is evaluated on R in
//            place of b, full weighting writes the coarse right-hand side.
//            The smoothed u of the tile goes to the level's scratch t (other
//            CTAs still read u for their halos in this phase).
//   up(l):   tile = a block of fine points plus a halo of 2*post; the coarse
//            correction e is staged, u' = t + P_lin e is formed in shared
//            memory, the post sweeps run on shrinking boxes, the tile is
//            written to u.
//   bottom:  the 3^3 coarsest grid is one coarse tile of the last down
//            phase, so the CTA that computes its right-hand side also runs
//            the 27-unknown LU solve (LAPACK getrs order) right away.
//
// Phases: 2 * levels - 1 grid barriers (63^3 -> 3^3: 7, was 15 plus a
// 30-50 us single-CTA tail).  Halo points are recomputed by neighbouring
// tiles with the same expression tree on the same inputs, so every value is
// bit-identical to the separate kernels (k_rb / k_residual / k_fw /
// k_prolong and the reference's numpy).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"
#include "mg.h"
#include "transfer_dev.cuh"

namespace cg = cooperative_groups;

namespace pl {

namespace {

constexpr int M2_THREADS = 1024;
constexpr int M2_MAX = 8;
constexpr size_t M2_SMEM_MAX = 220 * 1024;

struct M2Level {
  double* u;   // level iterate (level 0: the caller's u; coarser: the correction e)
  double* b;   // right-hand side (coarser levels: written by the previous down phase)
  double* t;   // smoothed iterate between the down and the up phase
  Geo g;
  OpC c;
  double dval, dinv;   // constant shifted diagonal and RN(1 / dval)
};

struct M2Args {
  unsigned long long* trace;   // PL_MID_TRACE: %globaltimer per phase (or null)
  int nlev;                    // levels 0 .. nlev-1 on the grid; level nlev: 27-unknown LU
  M2Level lv[M2_MAX + 1];
  int pre, post;
  double omega, sigma;
  int zero;                    // level 0 starts from a zero guess
  const double* lu;            // 27 x 27 getrf factors (row-major) + 27 pivots
  int dt[3];                   // coarse tile of the down phase (x, y, z)
  int ut[3];                   // fine tile of the up phase
};

// correctly rounded a / b from y = RN(1/b) (see zmarch.cu div_const)
__device__ __noinline__ double m2_div_slow(double a, double b) { return a / b; }
__device__ __forceinline__ double m2_div(double a, double b, double y) {
  double q = a * y;
  double r = __fma_rn(-b, q, a);
  q = __fma_rn(r, y, q);
  r = __fma_rn(-b, q, a);
  q = __fma_rn(r, y, q);
  const double aa = fabs(a);
  if (__builtin_expect(!(aa >= 0x1p-960 && aa <= 0x1p960), 0)) q = m2_div_slow(a, b);
  return q;
}

template <bool POW2>
__device__ __forceinline__ double m2_dd2(double x, const OpC& c) {
  return POW2 ? x * c.inv_dx2 : x / c.dx2;
}

// nu * Lap at box index i (strides 1, sy, sz), heat.py:119-140 order: z, y, x
template <bool POW2>
__device__ __forceinline__ double m2_lap(const double* s, int i, int sy, int sz, const OpC& c) {
  const double c0 = s[i];
  double acc = 0.0;
  acc = acc + m2_dd2<POW2>((s[i - sz] - 2.0 * c0) + s[i + sz], c);
  acc = acc + m2_dd2<POW2>((s[i - sy] - 2.0 * c0) + s[i + sy], c);
  acc = acc + m2_dd2<POW2>((s[i - 1] - 2.0 * c0) + s[i + 1], c);
  return c.nu * acc;
}

// staged box: origin (ox, oy, oz) in level coordinates, extent (bx, by, bz)
struct Box {
  int ox, oy, oz, bx, by, bz;
  __device__ int vol() const { return bx * by * bz; }
  __device__ void decode(int p, int& x, int& y, int& z) const {
    const unsigned r = (unsigned)p / (unsigned)bx;
    x = p - (int)r * bx;
    z = (int)(r / (unsigned)by);
    y = (int)r - z * by;
  }
};

// cp.async 8-byte copy, zero-filled when !valid (src then unused)
__device__ __forceinline__ void m2_cpa8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void m2_cpa_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// stage box B of field f (geometry g) into s, zero outside the domain; one
// warp per box row (box rows are at most 32 wide), copies in flight together
__device__ __forceinline__ void m2_stage(double* s, const double* f, const Geo& g, const Box& B) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int rows = B.by * B.bz;
  for (int r = warp; r < rows; r += nw) {
    const int lz = r / B.by, ly = r - lz * B.by;
    const int y = B.oy + ly, z = B.oz + lz;
    const int x = B.ox + lane;
    const bool in = y >= 0 && z >= 0 && y < g.ny && z < g.nz && x >= 0 && x < g.nx;
    if (lane < B.bx) m2_cpa8(s + r * B.bx + lane, in ? f + g.at(x, y, z) : f, in);
  }
}
__device__ __forceinline__ void m2_zero(double* s, int n) {
  for (int p = threadIdx.x; p < n; p += blockDim.x) s[p] = 0.0;
}

// one colour of jor-rb on the box shrunk by `shrink` (in-domain points only).
// A warp takes two box rows, 16 lanes each; lane k owns the k-th point of
// the colour in its row (rows are at most 32 wide), so no lane idles on the
// other colour and no per-point division decodes the index.
template <bool POW2>
__device__ __forceinline__ void m2_colour(double* su, const double* sb, const Box& B,
                                          const M2Level& L, double sigma, double omega, int red,
                                          int shrink) {
  const int ix = B.bx - 2 * shrink, iy = B.by - 2 * shrink, iz = B.bz - 2 * shrink;
  if (ix <= 0 || iy <= 0 || iz <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int rows = iy * iz;
  const int sy = B.bx, sz = B.bx * B.by;
  const int xs = B.ox + shrink;
  for (int r2 = warp; 2 * r2 < rows; r2 += nw) {
    const int r = 2 * r2 + (lane >> 4);
    if (r >= rows) continue;
    const int lz = r / iy, ly = r - lz * iy;
    const int y = B.oy + shrink + ly, z = B.oz + shrink + lz;
    if (y < 0 || z < 0 || y >= L.g.ny || z >= L.g.nz) continue;
    // red: even 1-based coordinate sum (multigrid.py:167-175) <=> x + y + z odd
    const int want = red ? ((y + z + 1) & 1) : ((y + z) & 1);
    const int x = xs + ((want - xs) & 1) + 2 * (lane & 15);
    if (x >= xs + ix || x < 0 || x >= L.g.nx) continue;
    const int i = (lz + shrink) * sz + (ly + shrink) * sy + (x - B.ox);
    const double cc = su[i];
    const double rr = sb[i] - (cc - sigma * m2_lap<POW2>(su, i, sy, sz, L.c));
    su[i] = cc + m2_div(omega * rr, L.dval, L.dinv);
  }
}

// LAPACK getrs order for m = 27 (same chain as mg.cu ft_lu27): lane i holds
// x_i; A (factors + pivots) staged in shared memory
__device__ __forceinline__ void m2_lu27(const double* A, const double* b, double* u) {
  constexpr int m = 27;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const double* ar = A + (lane < m ? lane : m - 1) * m;
    const double* piv = A + m * m;
    int q = lane;
    for (int i = m - 1; i >= 0; --i) {
      const int pi = (int)piv[i];
      if (q == i) q = pi;
      else if (q == pi) q = i;
    }
    double v = lane < m ? b[q] : 0.0;
#pragma unroll
    for (int j = 0; j < m; ++j) {
      const double yj = __shfl_sync(0xffffffffu, v, j);
      if (lane > j && lane < m) v = __fma_rn(-yj, ar[j], v);
    }
#pragma unroll
    for (int j = m - 1; j >= 0; --j) {
      if (lane == j) v = v / ar[j];
      const double xj = __shfl_sync(0xffffffffu, v, j);
      if (lane < j) v = __fma_rn(-xj, ar[j], v);
    }
    if (lane < m) u[lane] = v;
  }
}

__device__ __forceinline__ void m2_trace(const M2Args& m, int& ph) {
  if (m.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (ph < 127) {
      m.trace[128 + ph] = clock64();
      m.trace[ph++] = t;
    }
  }
}

// ---- down(l): pre-smooth, residual, full weighting (+ LU at the bottom) ----
template <bool POW2>
__device__ void m2_down(const M2Args& m, int l, double* sm, int& ph) {
  const M2Level& L = m.lv[l];
  const M2Level& C = m.lv[l + 1];
  const bool zero = l > 0 || m.zero;
  const int H = 2 * m.pre + 1;
  const int tx = m.dt[0], ty = m.dt[1], tz = m.dt[2];
  const int ntx = (C.g.nx + tx - 1) / tx, nty = (C.g.ny + ty - 1) / ty,
            ntz = (C.g.nz + tz - 1) / tz;
  const int ntiles = ntx * nty * ntz;
  const bool bottom = l + 1 == m.nlev;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int kx = tile % ntx, ky = (tile / ntx) % nty, kz = tile / (ntx * nty);
    const int cx0 = kx * tx, cy0 = ky * ty, cz0 = kz * tz;
    const int cnx = min(tx, C.g.nx - cx0), cny = min(ty, C.g.ny - cy0),
              cnz = min(tz, C.g.nz - cz0);
    // fine footprint R = [2 c0, 2 (c0 + cn)] per axis, plus the halo H
    Box B;
    B.ox = 2 * cx0 - H; B.oy = 2 * cy0 - H; B.oz = 2 * cz0 - H;
    B.bx = 2 * cnx + 1 + 2 * H; B.by = 2 * cny + 1 + 2 * H; B.bz = 2 * cnz + 1 + 2 * H;
    const int vol = B.vol();
    double* su = sm;
    double* sb = sm + vol;
    if (zero) m2_zero(su, vol);
    else m2_stage(su, L.u, L.g, B);
    m2_stage(sb, L.b, L.g, B);
    m2_cpa_wait();
    __syncthreads();
    if (tile == (int)blockIdx.x) m2_trace(m, ph);
    for (int k = 0; k < m.pre; ++k) {
      m2_colour<POW2>(su, sb, B, L, m.sigma, m.omega, 1, 2 * k + 1);
      __syncthreads();
      if (tile == (int)blockIdx.x) m2_trace(m, ph);
      m2_colour<POW2>(su, sb, B, L, m.sigma, m.omega, 0, 2 * k + 2);
      __syncthreads();
      if (tile == (int)blockIdx.x) m2_trace(m, ph);
    }
    // residual on R, in place of b (k_residual arithmetic)
    {
      const int rx = 2 * cnx + 1, ry = 2 * cny + 1, rz = 2 * cnz + 1;
      const int sy = B.bx, sz = B.bx * B.by;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int r = warp; r < ry * rz; r += nw) {   // one warp per row (rx <= 32)
        const int lz = r / ry, ly = r - lz * ry;
        if (lane >= rx) continue;
        const int i = ((lz + H) * B.by + (ly + H)) * B.bx + (lane + H);
        sb[i] = sb[i] - (su[i] - m.sigma * m2_lap<POW2>(su, i, sy, sz, L.c));
      }
    }
    __syncthreads();
    if (tile == (int)blockIdx.x) m2_trace(m, ph);
    // full weighting (fw_point order: z, then y, then x) and the smoothed
    // iterate of the fine points this tile owns
    {
      Geo gs;   // shared-memory view with the box strides, origin at fine 0
      gs.dim = 3; gs.sy = B.bx; gs.sz = (long long)B.bx * B.by;
      const double* f0 = sb + ((2 * cz0 - B.oz) * gs.sz + (2 * cy0 - B.oy) * gs.sy +
                               (2 * cx0 - B.ox));
      for (int p = threadIdx.x; p < cnx * cny * cnz; p += blockDim.x) {
        const int jx = p % cnx, jy = (p / cnx) % cny, jz = p / (cnx * cny);
        C.b[C.g.at(cx0 + jx, cy0 + jy, cz0 + jz)] = fw_point<3>(f0, gs, jx, jy, jz);
      }
      // owned fine points: [2 c0, 2 (c0 + cn)), the last tile also 2 nc
      const int ex = 2 * cnx + (cx0 + cnx == C.g.nx ? 1 : 0);
      const int ey = 2 * cny + (cy0 + cny == C.g.ny ? 1 : 0);
      const int ez = 2 * cnz + (cz0 + cnz == C.g.nz ? 1 : 0);
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int r = warp; r < ey * ez; r += nw) {
        const int lz = r / ey, ly = r - lz * ey;
        if (lane >= ex) continue;
        const int i = ((lz + H) * B.by + (ly + H)) * B.bx + (lane + H);
        L.t[L.g.at(2 * cx0 + lane, 2 * cy0 + ly, 2 * cz0 + lz)] = su[i];
      }
    }
    __syncthreads();
    if (tile == (int)blockIdx.x) m2_trace(m, ph);
    if (bottom) {   // ntiles == 1 (checked on the host): the 3^3 LU right here
      double* cb = sm;
      double* cu = sm + 32;
      double* A = sm + 64;
      for (int p = threadIdx.x; p < 27 * 27 + 27; p += blockDim.x) m2_cpa8(A + p, m.lu + p, true);
      for (int p = threadIdx.x; p < 27; p += blockDim.x)
        cb[p] = C.b[C.g.at(p % 3, (p / 3) % 3, p / 9)];
      m2_cpa_wait();
      __syncthreads();
      m2_lu27(A, cb, cu);
      __syncthreads();
      for (int p = threadIdx.x; p < 27; p += blockDim.x)
        C.u[C.g.at(p % 3, (p / 3) % 3, p / 9)] = cu[p];
      __syncthreads();
    }
  }
}

// ---- up(l): u = t + P_lin e, post-smooth ------------------------------------
template <bool POW2>
__device__ void m2_up(const M2Args& m, int l, double* sm, int& ph) {
  const M2Level& L = m.lv[l];
  const M2Level& C = m.lv[l + 1];
  const int H = 2 * m.post;
  const int tx = m.ut[0], ty = m.ut[1], tz = m.ut[2];
  const int ntx = (L.g.nx + tx - 1) / tx, nty = (L.g.ny + ty - 1) / ty,
            ntz = (L.g.nz + tz - 1) / tz;
  const int ntiles = ntx * nty * ntz;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int kx = tile % ntx, ky = (tile / ntx) % nty, kz = tile / (ntx * nty);
    const int x0 = kx * tx, y0 = ky * ty, z0 = kz * tz;
    const int nx = min(tx, L.g.nx - x0), ny = min(ty, L.g.ny - y0), nz = min(tz, L.g.nz - z0);
    Box B;
    B.ox = x0 - H; B.oy = y0 - H; B.oz = z0 - H;
    B.bx = nx + 2 * H; B.by = ny + 2 * H; B.bz = nz + 2 * H;
    const int vol = B.vol();
    // coarse window read by lin_point for fine [lo, hi]: [lo/2 - 1, hi/2]
    Box E;
    E.ox = (B.ox >> 1) - 1; E.oy = (B.oy >> 1) - 1; E.oz = (B.oz >> 1) - 1;
    E.bx = ((B.ox + B.bx - 1) >> 1) - E.ox + 1;
    E.by = ((B.oy + B.by - 1) >> 1) - E.oy + 1;
    E.bz = ((B.oz + B.bz - 1) >> 1) - E.oz + 1;
    double* su = sm;
    double* sb = sm + vol;
    double* se = sm + 2 * vol;
    m2_stage(se, C.u, C.g, E);
    m2_stage(su, L.t, L.g, B);
    m2_stage(sb, L.b, L.g, B);
    m2_cpa_wait();
    __syncthreads();
    if (tile == (int)blockIdx.x) m2_trace(m, ph);
    Geo ge = C.g;   // domain bounds of the coarse grid, box strides
    ge.sy = E.bx;
    ge.sz = (long long)E.bx * E.by;
    const double* e0 = se - (E.oz * ge.sz + E.oy * ge.sy + E.ox);
    {   // u = t + P_lin e (k_prolong arithmetic), in-domain points
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int r = warp; r < B.by * B.bz; r += nw) {
        const int lz = r / B.by, ly = r - lz * B.by;
        const int x = B.ox + lane, y = B.oy + ly, z = B.oz + lz;
        if (lane >= B.bx || x < 0 || y < 0 || z < 0 || x >= L.g.nx || y >= L.g.ny ||
            z >= L.g.nz)
          continue;
        const int i = r * B.bx + lane;
        su[i] = su[i] + lin_point<3>(e0, ge, x, y, z);
      }
    }
    __syncthreads();
    if (tile == (int)blockIdx.x) m2_trace(m, ph);
    for (int k = 0; k < m.post; ++k) {
      m2_colour<POW2>(su, sb, B, L, m.sigma, m.omega, 1, 2 * k + 1);
      __syncthreads();
      if (tile == (int)blockIdx.x) m2_trace(m, ph);
      m2_colour<POW2>(su, sb, B, L, m.sigma, m.omega, 0, 2 * k + 2);
      __syncthreads();
      if (tile == (int)blockIdx.x) m2_trace(m, ph);
    }
    {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int r = warp; r < ny * nz; r += nw) {
        const int lz = r / ny, ly = r - lz * ny;
        if (lane < nx)
          L.u[L.g.at(x0 + lane, y0 + ly, z0 + lz)] =
              su[((lz + H) * B.by + (ly + H)) * B.bx + (lane + H)];
      }
    }
    __syncthreads();
  }
}

template <bool POW2>
__global__ void __launch_bounds__(M2_THREADS) k_mid2(M2Args m) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  int ph = 0;
  m2_trace(m, ph);
  for (int l = 0; l < m.nlev; ++l) {
    m2_down<POW2>(m, l, sm, ph);
    grid.sync();
    m2_trace(m, ph);
  }
  for (int l = m.nlev - 1; l >= 0; --l) {
    m2_up<POW2>(m, l, sm, ph);
    if (l > 0) {
      grid.sync();
      m2_trace(m, ph);
    }
  }
}

size_t down_smem(int tx, int ty, int tz, int pre) {
  const int H = 2 * pre + 1;
  const size_t v = (size_t)(2 * tx + 1 + 2 * H) * (2 * ty + 1 + 2 * H) * (2 * tz + 1 + 2 * H);
  return 8 * (2 * v > 27 * 27 + 27 + 64 ? 2 * v : 27 * 27 + 27 + 64);
}
size_t up_smem(int tx, int ty, int tz, int post) {
  const int H = 2 * post;
  const size_t v = (size_t)(tx + 2 * H) * (ty + 2 * H) * (tz + 2 * H);
  const size_t e = (size_t)((tx + 2 * H) / 2 + 3) * ((ty + 2 * H) / 2 + 3) * ((tz + 2 * H) / 2 + 3);
  return 8 * (2 * v + e);
}

}  // namespace

int g_mid2_enabled = 0;   // PL_OPT_MID2: one grid phase per level and direction (A/B; slower)
extern int g_mid_ctas;

// Can the one-phase-per-level kernel run levels l0 .. coarsest of P?
bool mid2_applies(const MgPlan* P, int l0) {
  if (!g_mid2_enabled || P->dim != 3 || P->order != 2 || P->smoother != SM_RB) return false;
  if (P->pre > 2 || P->post > 2 || P->m_lu != 27) return false;
  const int nl = (int)P->lv.size();
  if (nl - 1 - l0 < 1 || nl - 1 - l0 > M2_MAX) return false;
  if (!P->lv[nl - 1].coarsest || P->lv[nl - 1].g.N != 3) return false;
  for (int l = l0; l < nl; ++l)
    if (P->lv[l].c.pow2 != P->lv[l0].c.pow2) return false;
  return true;
}

int launch_mid2(MgPlan* P, int l0, double* u, const double* b, double sigma, int zero,
                const double* lu_dev, cudaStream_t s) {
  const int nl = (int)P->lv.size();
  M2Args m;
  std::memset(&m, 0, sizeof(m));
  m.nlev = nl - 1 - l0;
  m.pre = P->pre;
  m.post = P->post;
  m.omega = P->omega;
  m.sigma = sigma;
  m.zero = zero;
  m.lu = lu_dev;
  // tiles: the bottom coarse grid (3^3) must be a single down tile
  int dt[3] = {8, 8, 4}, ut[3] = {16, 16, 8};
  while (down_smem(dt[0], dt[1], dt[2], m.pre) > M2_SMEM_MAX) {
    int* big = dt[0] >= dt[1] && dt[0] >= dt[2] ? &dt[0] : (dt[1] >= dt[2] ? &dt[1] : &dt[2]);
    *big /= 2;
  }
  while (up_smem(ut[0], ut[1], ut[2], m.post) > M2_SMEM_MAX) {
    int* big = ut[0] >= ut[1] && ut[0] >= ut[2] ? &ut[0] : (ut[1] >= ut[2] ? &ut[1] : &ut[2]);
    *big /= 2;
  }
  if (2 * dt[0] + 1 + 2 * (2 * m.pre + 1) > 32 || ut[0] + 4 * m.post > 32) {
    set_error("mid2: box rows wider than a warp");
    return -2;
  }
  if (dt[0] < 3 || dt[1] < 3 || dt[2] < 3) {
    set_error("mid2: tiles do not fit shared memory");
    return -2;
  }
  std::memcpy(m.dt, dt, sizeof(dt));
  std::memcpy(m.ut, ut, sizeof(ut));
  double bytes = 0.0;
  for (int i = 0; i <= m.nlev; ++i) {
    const MgLevel& L = P->lv[l0 + i];
    M2Level& M = m.lv[i];
    M.u = i == 0 ? u : L.u;
    M.b = i == 0 ? const_cast<double*>(b) : L.b;
    M.t = L.t;
    M.g = L.g;
    M.c = L.c;
    double t = 0.0;
    t = t + L.c.d1_int;
    t = t + L.c.d1_int;
    t = t + L.c.d1_int;
    M.dval = 1.0 - sigma * (L.c.nu * t);   // shifted_diag<3> for order 2
    M.dinv = 1.0 / M.dval;
    if (i < m.nlev) {   // the unfused kernels' algorithmic bytes
      const double np = (double)L.g.npts, nc = (double)P->lv[l0 + i + 1].g.npts;
      bytes += np * (24.0 * (P->pre + P->post) + 24.0 + 8.0 + 16.0) + nc * 16.0;
    }
  }
  bytes += 8.0 * 27 * 2;
  const size_t smem = std::max(down_smem(dt[0], dt[1], dt[2], m.pre),
                               up_smem(ut[0], ut[1], ut[2], m.post));
  const bool pow2 = P->lv[l0].c.pow2 != 0;
  void* kern = pow2 ? (void*)k_mid2<true> : (void*)k_mid2<false>;
  static int grid[2] = {0, 0};
  static size_t attr_smem[2] = {0, 0};
  int& gsz = grid[pow2];
  if (attr_smem[pow2] < smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)M2_SMEM_MAX);
    attr_smem[pow2] = M2_SMEM_MAX;
  }
  if (gsz == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, M2_THREADS, M2_SMEM_MAX);
    if (per < 1) {
      set_error("mid2 kernel does not fit one CTA per SM");
      return 2;
    }
    gsz = sms;
  }
  static unsigned long long* trace = nullptr;
  static const bool tracing = std::getenv("PL_MID_TRACE") != nullptr;
  if (tracing && !trace) cudaMalloc(&trace, 256 * sizeof(unsigned long long));
  m.trace = tracing ? trace : nullptr;
  if (tracing) cudaMemsetAsync(trace, 0, 256 * sizeof(unsigned long long), s);
  void* args[] = {&m};
  PL_PRE(K_MID);
  cudaError_t e = cudaLaunchCooperativeKernel(kern, g_mid_ctas > 0 && g_mid_ctas < gsz ? g_mid_ctas : gsz,
                                              M2_THREADS, args, smem, s);
  if (e != cudaSuccess) return cuda_status(e, "cooperative mid2 launch");
  if (tracing) {
    unsigned long long h[256];
    cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "mid2 n=%d levels=%d:", P->lv[l0].g.N, m.nlev);
    for (int i = 1; i < 128 && h[i]; ++i) std::fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    std::fprintf(stderr, " us\n  SM MHz per phase:");
    for (int i = 1; i < 128 && h[i]; ++i)
      std::fprintf(stderr, " %.0f", (double)(h[128 + i] - h[127 + i]) / (double)(h[i] - h[i - 1]) * 1e3);
    std::fprintf(stderr, "\n");
  }
  PL_CHECK_LAUNCH(K_MID, bytes);
  return 0;
}

}  // namespace pl
