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
#include "transfer_dev.cuh"

namespace pl {

namespace {

constexpr int MAXN = 17;

struct NodeCoef {
  int rows;            // R <= MAXN
  int col[MAXN];       // source field index of compacted column k
  int addrow[MAXN];    // field index of `add` for output row m
  double a[MAXN * MAXN];   // R x K, row-major over compacted columns
};

// byte offsets of the compacted input columns and of the `add` rows, computed
// on the host (col[k] * stride * 8): a load address is one 64-bit add away
// from the point's base instead of a multiply by the field stride per load
struct ColOfs {
  long long f[MAXN];
  long long a[MAXN];
};
inline ColOfs col_offsets(const NodeCoef& c, int K, long long stride, long long add_stride) {
  ColOfs o;
  std::memset(&o, 0, sizeof(o));
  for (int k = 0; k < K && k < MAXN; ++k) o.f[k] = (long long)c.col[k] * stride * 8;
  for (int m = 0; m < MAXN; ++m) o.a[m] = (long long)c.addrow[m] * add_stride * 8;
  return o;
}

// the chain kernels index a field's points with 32 bits
inline bool small_field(long long npts) {
  if (npts < (1LL << 31)) return true;
  set_error("chain kernel: %lld points exceed 2^31", npts);
  return false;
}

// mode 0: out = scale*chain ; 1: out = scale*chain + add ; 2: out = add - scale*chain
template <int K>
__global__ void __launch_bounds__(256) k_chain(const double* __restrict__ in, ColOfs o,
                                               double* out, long long out_stride,
                                               NodeCoef c, double scale, long long npts,
                                               const double* add,   // may alias out
                                               int mode) {
  // fields have fewer than 2^31 elements (checked at launch): one 32-bit point
  // index, column / row addresses by 64-bit adds of host-computed byte offsets
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (unsigned)npts) return;
  const char* pin = reinterpret_cast<const char*>(in + i);
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = *reinterpret_cast<const double*>(pin + o.f[k]);
  char* po = reinterpret_cast<char*>(out + i);
  const char* pa = reinterpret_cast<const char*>(add + i);
  const long long ob = out_stride * 8;
#pragma unroll
  for (int m = 0; m < MAXN; ++m) {
    if (m >= c.rows) break;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc = __fma_rn(c.a[m * K + k], v[k], acc);
    double r = scale * acc;
    if (mode == 1) r = r + *reinterpret_cast<const double*>(pa + o.a[m]);
    else if (mode == 2) r = *reinterpret_cast<const double*>(pa + o.a[m]) - r;
    *reinterpret_cast<double*>(po) = r;
    po += ob;
  }
}

// sdc.py:117-124, max-reduced as IEEE bit patterns (non-negative doubles
// order like unsigned integers; NaN propagates like np.max).
// R > 0: the row count is a compile-time constant (R == q.rows), so every
// load of the point is issued before the first chain; R == 0: runtime rows
template <int K, int R = 0>
__global__ void __launch_bounds__(256) k_resmax(const double* __restrict__ Y,
                                                const double* __restrict__ F, ColOfs o,
                                                long long stride,
                                                const double* __restrict__ y0,
                                                const double* __restrict__ tau, NodeCoef q,
                                                double dt, long long npts,
                                                unsigned long long* out) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;   // < 2^31 (checked at launch)
  unsigned long long best = 0ull;
  if (i < (unsigned)npts) {
    const char* pf = reinterpret_cast<const char*>(F + i);
    double f[K];
#pragma unroll
    for (int k = 0; k < K; ++k) f[k] = *reinterpret_cast<const double*>(pf + o.f[k]);
    const double base = y0[i];
    constexpr int NR = R > 0 ? R : MAXN;
    const long long sb = stride * 8;
    const char* py = reinterpret_cast<const char*>(Y + i);
    const char* pt = reinterpret_cast<const char*>(tau + i);
    double yv[R > 0 ? R : 1];
    if constexpr (R > 0) {
#pragma unroll
      for (int m = 0; m < R; ++m) yv[m] = *reinterpret_cast<const double*>(py + m * sb);
    }
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      if (R > 0 || m < q.rows) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) acc = __fma_rn(q.a[m * K + k], f[k], acc);
        double r = (base + dt * acc) -
                   (R > 0 ? yv[R > 0 ? m : 0] : *reinterpret_cast<const double*>(py + m * sb));
        if (tau) r = r + *reinterpret_cast<const double*>(pt + m * sb);
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
                                                     ColOfs o, NodeCoef pt,
                                                     double* __restrict__ out,
                                                     long long out_stride, long long npts) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;   // < 2^31 (checked at launch)
  if (i >= (unsigned)npts) return;
  const char* pn = reinterpret_cast<const char*>(ynew + i);
  const char* po = reinterpret_cast<const char*>(yold + i);
  double d[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    d[k] = *reinterpret_cast<const double*>(pn + o.f[k]) -
           *reinterpret_cast<const double*>(po + o.f[k]);
  char* pout = reinterpret_cast<char*>(out + i);
  const long long ob = out_stride * 8;
#pragma unroll
  for (int m = 0; m < MAXN; ++m) {
    if (m >= pt.rows) break;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc = __fma_rn(pt.a[m * K + k], d[k], acc);
    *reinterpret_cast<double*>(pout) = acc;
    pout += ob;
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


// ---------------------------------------------------------------------------
// FAS node integrals fused into full weighting (hierarchy.py:102-108 then
// transfers.py:27-34): coarse[r] = FW(scale * chain_r(F) (+ add[addrow[r]]))
// for R selected rows, without writing the R fine integrals.  Layout and
// operation order are k_rfw's (zmarch.cu): a CTA owns a 16 x 8 coarse tile and
// the 33 x 17 fine window of its footprint; warp w owns window rows w and w+9,
// warp 8 also the last column; marching up the fine planes each thread
// evaluates k_chain's arithmetic at its points and folds it into fw3's z
// weights in registers (a, a + 2b, 0.25 (t + c)); the y pass runs one phase
// later and the x pass two, one barrier per plane.  The result is bit-identical
// to k_chain + k_fw.
// next-plane prefetch into L1: the plane loop issues its loads, waits for them
// and only then meets the barrier, so without it a CTA has one DRAM round trip
// per plane on its critical path (long scoreboard 10 warp-cycles per issued
// instruction).  restrict_state 272 -> 244 us, compute_fas 351 -> 341 us at
// 255^3; prefetching a second plane ahead into L2 as well is slower (261 /
// 375 us).
__device__ __forceinline__ void prefetch_plane(const double* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
constexpr int CF_TX = 32, CF_TY = 16, CF_RX = CF_TX + 1, CF_RY = CF_TY + 1;
constexpr int CF_PR = (CF_RX * CF_RY + 15) / 16 * 16;
constexpr int CF_NT = 288;

// IDENT (K == R): row r is input column r itself (restrict_state's full
// weighting of the selected nodes, several fields in one launch)
template <int K, int R, bool IDENT = false>
__global__ void __launch_bounds__(CF_NT, 3) k_chain_fw(const double* __restrict__ F,
                                                      ColOfs o, NodeCoef c, double scale,
                                                      const double* __restrict__ add, int mode,
                                                      double* __restrict__ coarse,
                                                      long long cstride, Geo gf, Geo gc,
                                                      int zcc) {
  extern __shared__ __align__(16) double cf_sm[];
  double* szb = cf_sm;                  // R z-weighted planes (CF_RX x CF_RY)
  double* syx = cf_sm + R * CF_PR;      // R y-weighted row sets (CF_RX x CF_TY/2)
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int w = tid >> 5, lane = tid & 31;
  const int x0 = blockIdx.x * CF_TX, y0 = blockIdx.y * CF_TY;
  const int jz0 = blockIdx.z * zcc, jz1 = min(jz0 + zcc, gc.nz);
  const int p0 = 2 * jz0, p1 = 2 * jz1;
  // ---- owned fine points: row w (q = 0), row w + 9 or (warp 8) the last column
  int r_k[2];
  bool r_on[2], r_ok[2];
  const double* r_f[2];                 // F at the point on plane p (column 0 of F)
  const double* r_a[2];                 // add (tau) at the point on plane p
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = q == 0 ? w * CF_RX + lane
                         : (w < 8 ? (w + 9) * CF_RX + lane : (lane < CF_RY ? lane * CF_RX + CF_TX : 0));
    const int ry = k / CF_RX, rx = k - ry * CF_RX;
    r_on[q] = q == 0 || w < 8 || lane < CF_RY;
    r_k[q] = k;
    r_ok[q] = r_on[q] && x0 + rx < gf.nx && y0 + ry < gf.ny;
    const long long g0 = r_ok[q] ? gf.at(x0 + rx, y0 + ry, p0) : 0;
    r_f[q] = F + g0;
    r_a[q] = add ? add + g0 : nullptr;
  }
  double acc[2][R];
  // ---- y pass: thread tid < 264 owns window entry (yy, xx) of every row set r
  constexpr int NYE = CF_RX * (CF_TY / 2);
  const bool ytask = tid < NYE;
  const int yy = tid / CF_RX, xx = tid - (tid / CF_RX) * CF_RX;
  const int y_src = 2 * yy * CF_RX + xx;
  // ---- x pass: entries e = tid + 288 i (< R * 128), coarse plane advanced per pass
  constexpr int NX = R * (CF_TX / 2) * (CF_TY / 2), NXI = (NX + CF_NT - 1) / CF_NT;
  // the chain values of plane p at the owned points (k_chain's arithmetic)
  auto values = [&](int q, long long off, double* v, bool pf) {
    if (!r_ok[q]) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = 0.0;
      return;
    }
    double f[K];
    const char* base = reinterpret_cast<const char*>(r_f[q] + off);
#pragma unroll
    for (int k = 0; k < K; ++k) f[k] = __ldcs(reinterpret_cast<const double*>(base + o.f[k]));
    if (pf) {
      const char* nxt = base + gf.sz * 8;
#pragma unroll
      for (int k = 0; k < K; ++k) prefetch_plane(reinterpret_cast<const double*>(nxt + o.f[k]));
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (IDENT) {
        v[r] = f[r];
      } else {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) a = __fma_rn(c.a[r * K + k], f[k], a);
        double t = scale * a;
        if (mode == 1)
          t = t + *reinterpret_cast<const double*>(reinterpret_cast<const char*>(r_a[q] + off) +
                                                   o.a[r]);
        v[r] = t;
      }
    }
  };
  // MODE 0: first plane of the chunk (a := v); 1: odd plane (t = a + 2 v);
  // 2: even plane (0.25 (t + v) -> szb, a := v)
  auto fold = [&](auto mode_tag, long long off, bool pf) {
    constexpr int MODE = decltype(mode_tag)::value;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!r_on[q]) continue;
      double v[R];
      values(q, off, v, pf);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (MODE == 0) {
          acc[q][r] = v[r];
        } else if (MODE == 1) {
          acc[q][r] = acc[q][r] + 2.0 * v[r];
        } else {
          szb[r * CF_PR + r_k[q]] = 0.25 * (acc[q][r] + v[r]);
          acc[q][r] = v[r];
        }
      }
    }
  };
  auto ypass = [&]() {
    if (!ytask) return;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double* zc = szb + r * CF_PR + y_src;
      syx[r * CF_PR + tid] = fw3(zc[0], zc[CF_RX], zc[2 * CF_RX]);
    }
  };
  int jz = jz0;
  auto xpass = [&]() {
#pragma unroll
    for (int it = 0; it < NXI; ++it) {
      const int e = tid + it * CF_NT;
      const int r = e >> 7, pt = e & 127;
      const int ex = pt & 15, ey = pt >> 4;
      const int gcx = x0 / 2 + ex, gcy = y0 / 2 + ey;
      if (e < NX && gcx < gc.nx && gcy < gc.ny) {
        const double* yr = syx + r * CF_PR + ey * CF_RX + 2 * ex;
        coarse[r * cstride + gc.at(gcx, gcy, jz)] = fw3(yr[0], yr[1], yr[2]);
      }
    }
    ++jz;
  };
  // phase p0, then pairs (odd plane: y pass of the coarse plane finished two
  // phases ago; even plane: x pass)
  long long off = 0;
  fold(std::integral_constant<int, 0>{}, off, p0 + 1 <= p1);
  __syncthreads();
  for (int p = p0 + 1; p <= p1 + 2; p += 2) {
    const int ph = p - p0;                     // odd
    off += gf.sz;
    if (p <= p1) fold(std::integral_constant<int, 1>{}, off, p + 1 <= p1);
    if (ph >= 3) ypass();                      // y pass of jz = (p - 3) / 2
    __syncthreads();
    off += gf.sz;
    if (p + 1 <= p1) fold(std::integral_constant<int, 2>{}, off, p + 2 <= p1);
    if (ph + 1 >= 4) xpass();                  // x pass of jz = (p - 3) / 2
    __syncthreads();
  }
}

// the same operation for many input fields (K x R large): the runtime plane
// loop keeps fewer values live (no spills at 72 registers)
template <int K, int R, bool IDENT = false>
__global__ void __launch_bounds__(CF_NT, 3) k_chain_fw_wide(const double* __restrict__ F,
                                                      ColOfs o, NodeCoef c, double scale,
                                                      const double* __restrict__ add, int mode,
                                                      double* __restrict__ coarse,
                                                      long long cstride, Geo gf, Geo gc,
                                                      int zcc) {
  extern __shared__ __align__(16) double cf_sm[];
  double* szb = cf_sm;                  // R z-weighted planes (CF_RX x CF_RY)
  double* syx = cf_sm + R * CF_PR;      // R y-weighted row sets (CF_RX x CF_TY/2)
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int w = tid >> 5, lane = tid & 31;
  const int x0 = blockIdx.x * CF_TX, y0 = blockIdx.y * CF_TY;
  const int jz0 = blockIdx.z * zcc, jz1 = min(jz0 + zcc, gc.nz);
  const int p0 = 2 * jz0, p1 = 2 * jz1;
  int r_k[2];
  bool r_ok[2];
  long long r_g[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = q == 0 ? w * CF_RX + lane
                         : (w < 8 ? (w + 9) * CF_RX + lane
                                  : (lane < CF_RY ? lane * CF_RX + CF_TX : CF_RX * CF_RY));
    const int ry = k / CF_RX, rx = k - ry * CF_RX;
    r_k[q] = k < CF_RX * CF_RY ? k : -1;
    r_ok[q] = r_k[q] >= 0 && x0 + rx < gf.nx && y0 + ry < gf.ny;
    r_g[q] = r_ok[q] ? gf.at(x0 + rx, y0 + ry, 0) : 0;
  }
  double acc[2][R];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[q][r] = 0.0;
  // y pass: thread tid < 264 owns window entry (yy, xx) of every row set r
  const bool ytask = tid < CF_RX * (CF_TY / 2);
  const int y_src = 2 * (tid / CF_RX) * CF_RX + (tid - (tid / CF_RX) * CF_RX);
  long long pofs = (long long)p0 * gf.sz * 8;      // byte offset of plane p
  for (int p = p0; p <= p1 + 2; ++p, pofs += gf.sz * 8) {
    const int ph = p - p0;
    if (p <= p1) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (r_k[q] < 0) continue;
        double v[R];
        if (r_ok[q]) {
          const char* base = reinterpret_cast<const char*>(F + r_g[q]) + pofs;
          double f[K];
#pragma unroll
          for (int k = 0; k < K; ++k)
            f[k] = __ldcs(reinterpret_cast<const double*>(base + o.f[k]));
          if (p < p1) {
            const char* nxt = base + gf.sz * 8;
#pragma unroll
            for (int k = 0; k < K; ++k) prefetch_plane(reinterpret_cast<const double*>(nxt + o.f[k]));
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {          // k_chain's arithmetic
            if constexpr (IDENT) {
              v[r] = f[r];
              continue;
            }
            double a = 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k) a = __fma_rn(c.a[r * K + k], f[k], a);
            double t = scale * a;
            if (mode == 1)
              t = t + *reinterpret_cast<const double*>(
                          reinterpret_cast<const char*>(add + r_g[q]) + pofs + o.a[r]);
            v[r] = t;
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = 0.0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (ph == 0) {
            acc[q][r] = v[r];
          } else if (ph & 1) {
            acc[q][r] = acc[q][r] + 2.0 * v[r];
          } else {
            szb[r * CF_PR + r_k[q]] = 0.25 * (acc[q][r] + v[r]);
            acc[q][r] = v[r];
          }
        }
      }
    }
    if ((ph & 1) == 1 && ph >= 3 && ytask) {          // y pass of jz = (p - 3) / 2
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double* zc = szb + r * CF_PR + y_src;
        syx[r * CF_PR + tid] = fw3(zc[0], zc[CF_RX], zc[2 * CF_RX]);
      }
    }
    if ((ph & 1) == 0 && ph >= 4) {          // x pass of jz = (p - 4) / 2
      for (int e = tid; e < R * (CF_TX / 2) * (CF_TY / 2); e += CF_NT) {
        const int r = e >> 7, pt = e & 127;
        const int ex = pt & 15, ey = pt >> 4;
        const int gcx = x0 / 2 + ex, gcy = y0 / 2 + ey;
        if (gcx < gc.nx && gcy < gc.ny) {
          const double* yr = syx + r * CF_PR + ey * CF_RX + 2 * ex;
          coarse[r * cstride + gc.at(gcx, gcy, (p - 4) / 2)] = fw3(yr[0], yr[1], yr[2]);
        }
      }
    }
    __syncthreads();
  }
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
  if (!small_field(npts)) return -1;
  const ColOfs ofs = col_offsets(c, K, in_stride, add_stride);
  const int blocks = ceil_div(npts, 256);
  PL_PRE(K_QUAD);
#define CALL(KK) \
  k_chain<KK><<<blocks, 256, 0, s>>>(in, ofs, out, out_stride, c, scale, npts, add, mode)
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
  if (!compact(q, c, K) || !small_field(npts)) return -1;
  const ColOfs ofs = col_offsets(c, K, stride, 0);
  cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(double), s);
  if (e != cudaSuccess) return cuda_status(e, "memset");
  const int blocks = ceil_div(npts, 256);
  unsigned long long* o = (unsigned long long*)out_dev;
  PL_PRE(K_RESMAX);
  if (c.rows == K + 1 && K >= 1 && K <= 8) {   // Q of M+1 nodes: K = M used columns
#define CALLR(KK) \
  k_resmax<KK, KK + 1><<<blocks, 256, 0, s>>>(Y, F, ofs, stride, y0, tau, c, dt, npts, o)
    switch (K) {
      case 1: CALLR(1); break; case 2: CALLR(2); break; case 3: CALLR(3); break;
      case 4: CALLR(4); break; case 5: CALLR(5); break; case 6: CALLR(6); break;
      case 7: CALLR(7); break; default: CALLR(8); break;
    }
#undef CALLR
  } else {
#define CALL(KK) \
  k_resmax<KK><<<blocks, 256, 0, s>>>(Y, F, ofs, stride, y0, tau, c, dt, npts, o)
    PL_K_DISPATCH(K, CALL);
#undef CALL
  }
  PL_CHECK_LAUNCH(K_RESMAX, 8.0 * npts * (K + q.rows + 1 + (tau ? q.rows : 0)));
  return 0;
}

int launch_delta_chain(const double* ynew, const double* yold, long long stride,
                       const Coef& pt, double* out, long long out_stride, long long npts,
                       cudaStream_t s) {
  NodeCoef c;
  int K;
  if (!compact(pt, c, K) || !small_field(npts)) return -1;
  const ColOfs ofs = col_offsets(c, K, stride, 0);
  const int blocks = ceil_div(npts, 256);
  PL_PRE(K_CORR);
#define CALL(KK) \
  k_delta_chain<KK><<<blocks, 256, 0, s>>>(ynew, yold, ofs, c, out, out_stride, npts)
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


int g_fuse_fas_fw = 1;   // PL_OPT_FUSE_FAS_FW

bool fw_select_ok(const Geo& gf, int nsel) {
  return g_fuse_fas_fw && gf.dim == 3 && gf.N >= 31 && zmarch_size_ok(gf.N) && nsel >= 1 &&
         nsel <= 5;
}

// coarse[j] = FW(fine[idx[j]]) for j < nsel in one launch (k_chain_fw<IDENT>)
int launch_fw_select(const double* fine, long long stride, const int* idx, int nsel,
                     double* coarse, long long cstride, const Geo& gf, cudaStream_t s) {
  NodeCoef c;
  std::memset(&c, 0, sizeof(c));
  c.rows = nsel;
  for (int j = 0; j < nsel; ++j) c.col[j] = idx[j];
  const ColOfs ofs = col_offsets(c, nsel, stride, 0);
  Geo gc = make_geo(3, (gf.N + 1) / 2);
  const int zcc = 8;
  dim3 grid(ceil_div(gf.nx, CF_TX), ceil_div(gf.ny, CF_TY), ceil_div(gc.nz, zcc));
  dim3 block(32, CF_NT / 32);
  PL_PRE(K_RESTRICT);
#define FS_CALL(RR)                                                                         \
  do {                                                                                      \
    size_t smem = sizeof(double) * 2 * RR * CF_PR;                                          \
    cudaFuncSetAttribute(k_chain_fw<RR, RR, true>,                                          \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);           \
    k_chain_fw<RR, RR, true><<<grid, block, smem, s>>>(fine, ofs, c, 1.0, nullptr, 0, coarse,  \
                                                       cstride, gf, gc, zcc);               \
  } while (0)
  switch (nsel) {
    case 1: FS_CALL(1); break; case 2: FS_CALL(2); break; case 3: FS_CALL(3); break;
    case 4: FS_CALL(4); break; default: FS_CALL(5); break;
  }
#undef FS_CALL
  PL_CHECK_LAUNCH(K_RESTRICT, (8.0 * gf.npts + 8.0 * gc.npts) * nsel);
  return 0;
}

bool chain_fw_ok(const Coef& a, const Geo& gf) {
  return g_fuse_fas_fw && gf.dim == 3 && gf.N >= 31 && zmarch_size_ok(gf.N) && a.rows >= 2 &&
         a.rows <= 5 &&
         a.cols <= 9;
}

int launch_chain_fw(const double* F, long long stride, const Coef& a, double scale,
                    const double* add, long long add_stride, const int* add_rows,
                    double* coarse, long long cstride, const Geo& gf, cudaStream_t s) {
  NodeCoef c;
  int K;
  if (!compact(a, c, K)) return -1;
  if (add_rows)
    for (int m = 0; m < a.rows; ++m) c.addrow[m] = add_rows[m];
  const ColOfs ofs = col_offsets(c, K, stride, add_stride);
  Geo gc = make_geo(3, (gf.N + 1) / 2);
  const int zcc = 8;
  dim3 grid(ceil_div(gf.nx, CF_TX), ceil_div(gf.ny, CF_TY), ceil_div(gc.nz, zcc));
  dim3 block(32, CF_NT / 32);
  const int mode = add ? 1 : 0;
  PL_PRE(K_FAS);
  // up to 25 chain coefficients per point the unrolled kernel keeps every
  // value in registers; wider FAS chains (K x R > 25) take the plane-loop form
#define CF_CALL(KK, RR)                                                                       \
  do {                                                                                        \
    size_t smem = sizeof(double) * 2 * RR * CF_PR;                                            \
    auto kern = KK * RR <= 25 ? k_chain_fw<KK, RR> : k_chain_fw_wide<KK, RR>;                 \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
    kern<<<grid, block, smem, s>>>(F, ofs, c, scale, add, mode, coarse, cstride, gf, gc, zcc); \
  } while (0)
#define CF_R(KK)                                   \
  switch (a.rows) {                                \
    case 2: CF_CALL(KK, 2); break;                 \
    case 3: CF_CALL(KK, 3); break;                 \
    case 4: CF_CALL(KK, 4); break;                 \
    default: CF_CALL(KK, 5); break;                \
  }
  switch (K) {
    case 1: CF_R(1); break; case 2: CF_R(2); break; case 3: CF_R(3); break;
    case 4: CF_R(4); break; case 5: CF_R(5); break; case 6: CF_R(6); break;
    case 7: CF_R(7); break; case 8: CF_R(8); break; default: CF_R(9); break;
  }
#undef CF_R
#undef CF_CALL
  // SURVEY 8(d) K13 for the fine part: read the K fine F fields (+ the
  // selected fine tau rows), write one coarse field per selected row
  PL_CHECK_LAUNCH(K_FAS, 8.0 * gf.npts * (K + (add ? a.rows : 0)) + 8.0 * gc.npts * a.rows);
  return 0;
}

}  // namespace pl
