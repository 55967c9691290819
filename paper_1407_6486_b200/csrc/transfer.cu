// Factor-2 grid transfers (transfers.py): full weighting, injection, linear
// and cubic interpolation.  Each restates the reference's per-axis numpy
// evaluation (axis 0 first, one rounding per operation) so results are
// bit-identical; the cubic weights go through a sequential FMA chain like the
// reference's dgemm (np.tensordot with the dense interpolation matrix).
#include <map>
#include <mutex>
#include <vector>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"
#include "transfer_dev.cuh"

namespace pl {

namespace {

template <int DIM>
__global__ void __launch_bounds__(256) k_fw(const double* __restrict__ f,
                                            double* __restrict__ cz, Geo gf, Geo gc) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= gc.npts) return;
  int jx, jy, jz;
  decode_point(gc, t, jx, jy, jz);
  cz[gc.at(jx, jy, jz)] = fw_point<DIM>(f, gf, jx, jy, jz);
}

template <int DIM>
__global__ void __launch_bounds__(256) k_inject(const double* __restrict__ f,
                                                double* __restrict__ cz, Geo gf, Geo gc) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= gc.npts) return;
  int jx, jy, jz;
  decode_point(gc, t, jx, jy, jz);
  long long idx = 2 * jx + 1;
  if (DIM >= 2) idx += (long long)(2 * jy + 1) * gf.sy;
  if (DIM == 3) idx += (long long)(2 * jz + 1) * gf.sz;
  cz[gc.at(jx, jy, jz)] = f[idx];
}

template <int DIM>
__global__ void __launch_bounds__(256) k_prolong(const double* __restrict__ c,
                                                 double* __restrict__ f, Geo gf, Geo gc,
                                                 int accumulate) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= gf.npts) return;
  int ix, iy, iz;
  decode_point(gf, t, ix, iy, iz);
  const long long o = gf.at(ix, iy, iz);
  double v = lin_point<DIM>(c, gc, ix, iy, iz);
  f[o] = accumulate ? f[o] + v : v;
}

// 3-D prolongation by coarse cell: thread (jx, jy, jz), 0 <= j <= nc, owns
// the fine points 2j and 2j+1 per axis (even: average of coarse j-1 and j;
// odd: copy of coarse j; transfers.py:40-45), reads the 2x2x2 coarse corners
// once (zero outside the domain) and moves fine x-pairs as 16-byte vectors.
// Per fine point the tree is lin_point's: z taps, then y, then x.
__global__ void __launch_bounds__(256) k_prolong3_cell(const double* __restrict__ c,
                                                       double* __restrict__ f, Geo gf, Geo gc,
                                                       int accumulate) {
  const int jx = blockIdx.x * 32 + threadIdx.x;
  const int jy = blockIdx.y * 8 + threadIdx.y;
  const int jz = blockIdx.z;
  const int nc = gc.nx;
  if (jx > nc || jy > nc) return;
  double cr[2][2][2];   // [z][y][x] corners at j-1, j
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const int z = jz - 1 + a, y = jy - 1 + b, x = jx - 1 + d;
        cr[a][b][d] = (z >= 0 && z < nc && y >= 0 && y < nc && x >= 0 && x < nc)
                          ? __ldg(c + (long long)z * gc.sz + (long long)y * gc.sy + x)
                          : 0.0;
      }
  const bool xo = jx < nc;   // fine 2j+1 exists along x
  // accumulate: the (up to) four fine pairs are loaded before any store, so
  // their DRAM latencies overlap (the compiler cannot prove the rows disjoint)
  double2 old[2][2];
#pragma unroll
  for (int pz = 0; pz < 2; ++pz)
#pragma unroll
    for (int py = 0; py < 2; ++py) {
      old[pz][py] = make_double2(0.0, 0.0);
      if (accumulate && (pz == 0 || jz < nc) && (py == 0 || jy < nc)) {
        const double* src = f + (long long)(2 * jz + pz) * gf.sz +
                            (long long)(2 * jy + py) * gf.sy + 2 * jx;
        if (xo) old[pz][py] = __ldcs(reinterpret_cast<const double2*>(src));
        else old[pz][py].x = __ldcs(src);
      }
    }
#pragma unroll
  for (int pz = 0; pz < 2; ++pz) {
    if (pz == 1 && jz >= nc) break;
    double zc[2][2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int d = 0; d < 2; ++d)
        zc[b][d] = pz == 0 ? 0.5 * (cr[0][b][d] + cr[1][b][d]) : cr[1][b][d];
#pragma unroll
    for (int py = 0; py < 2; ++py) {
      if (py == 1 && jy >= nc) break;
      const double y0 = py == 0 ? 0.5 * (zc[0][0] + zc[1][0]) : zc[1][0];
      const double y1 = py == 0 ? 0.5 * (zc[0][1] + zc[1][1]) : zc[1][1];
      const double ve = 0.5 * (y0 + y1), vo = y1;
      double* dst = f + (long long)(2 * jz + pz) * gf.sz + (long long)(2 * jy + py) * gf.sy +
                    2 * jx;
      if (xo) {
        double2 w = make_double2(ve, vo);
        if (accumulate) {
          const double2 o = old[pz][py];
          w.x = o.x + w.x;
          w.y = o.y + w.y;
        }
        *reinterpret_cast<double2*>(dst) = w;
      } else {
        dst[0] = accumulate ? old[pz][py].x + ve : ve;
      }
    }
  }
}

// One axis of the cubic interpolation (transfers.py:82-89): input viewed as
// (A, Bin, C) with strides (ia, ib, 1) -> output (A, Bout, C) with strides
// (oa, ob, 1), interpolating along B with sequential FMA over the taps
// (dgemm order).  Padded rows are processed whole (their zeros map to zeros).
__global__ void __launch_bounds__(256) k_cubic_axis(const double* __restrict__ in,
                                                    double* __restrict__ out, long long A,
                                                    int bout, long long C, long long ia,
                                                    long long ib, long long oa, long long ob,
                                                    const int* __restrict__ cnt,
                                                    const int* __restrict__ tidx,
                                                    const double* __restrict__ tw,
                                                    int accumulate) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A * bout * C) return;
  long long cc = t % C;
  long long r = t / C;
  int i = (int)(r % bout);
  long long a = r / bout;
  const double* src = in + a * ia + cc;
  double acc = 0.0;
  int nt = cnt[i];
  for (int q = 0; q < nt; ++q)
    acc = __fma_rn(tw[i * 4 + q], src[(long long)tidx[i * 4 + q] * ib], acc);
  double* dst = out + a * oa + (long long)i * ob + cc;
  *dst = accumulate ? *dst + acc : acc;
}

}  // namespace

#define PL_T_DISPATCH(g, KERNEL, grid, block, s, ...)                          \
  do {                                                                        \
    if ((g).dim == 1) KERNEL<1><<<grid, block, 0, s>>>(__VA_ARGS__);           \
    else if ((g).dim == 2) KERNEL<2><<<grid, block, 0, s>>>(__VA_ARGS__);      \
    else KERNEL<3><<<grid, block, 0, s>>>(__VA_ARGS__);                        \
  } while (0)

static Geo coarse_geo(const Geo& gf) { return make_geo(gf.dim, (gf.N + 1) / 2); }

int launch_fw(const double* fine, double* coarse, const Geo& gf, cudaStream_t s) {
  Geo gc = coarse_geo(gf);
  PL_PRE(K_RESTRICT);
  PL_T_DISPATCH(gf, k_fw, ceil_div(gc.npts, 256), 256, s, fine, coarse, gf, gc);
  PL_CHECK_LAUNCH(K_RESTRICT, 8.0 * gf.npts + 8.0 * gc.npts);
  return 0;
}

int launch_inject(const double* fine, double* coarse, const Geo& gf, cudaStream_t s) {
  Geo gc = coarse_geo(gf);
  PL_PRE(K_RESTRICT);
  PL_T_DISPATCH(gf, k_inject, ceil_div(gc.npts, 256), 256, s, fine, coarse, gf, gc);
  PL_CHECK_LAUNCH(K_RESTRICT, 16.0 * gc.npts);
  return 0;
}

int launch_prolong(const double* coarse, double* fine, const Geo& gf, int accumulate,
                   cudaStream_t s) {
  Geo gc = coarse_geo(gf);
  PL_PRE(K_PROLONG);
  if (gf.dim == 3 && (gf.sy % 2) == 0) {
    const int nc = gc.nx;
    dim3 grid(ceil_div(nc + 1, 32), ceil_div(nc + 1, 8), nc + 1);
    k_prolong3_cell<<<grid, dim3(32, 8), 0, s>>>(coarse, fine, gf, gc, accumulate);
  } else {
    PL_T_DISPATCH(gf, k_prolong, ceil_div(gf.npts, 256), 256, s, coarse, fine, gf, gc,
                  accumulate);
  }
  PL_CHECK_LAUNCH(K_PROLONG, (accumulate ? 16.0 : 8.0) * gf.npts + 8.0 * gc.npts);
  return 0;
}

// ---------------------------------------------------------------------------
// cubic taps (host restatement of transfers.py:53-79, weights in double with
// the reference's own float expression order)

static std::mutex g_taps_mu;
static std::map<int, CubicTaps*> g_taps;

const CubicTaps* cubic_taps(int nf) {
  std::lock_guard<std::mutex> lk(g_taps_mu);
  auto it = g_taps.find(nf);
  if (it != g_taps.end()) return it->second;
  int nc = nf / 2;
  int rows = nf - 1;
  std::vector<int> cnt(rows, 0), idx(rows * 4, 0);
  std::vector<double> w(rows * 4, 0.0);
  for (int i = 1; i < nf; ++i) {
    int r = i - 1;
    if (i % 2 == 0) {
      cnt[r] = 1;
      idx[r * 4] = i / 2 - 1;
      w[r * 4] = 1.0;
      continue;
    }
    double sp = i / 2.0;
    std::vector<int> pts;
    if (nc < 3) {
      for (int j = 0; j <= nc; ++j) pts.push_back(j);
    } else {
      int j0 = (int)std::floor(sp) - 1;
      if (j0 < 0) j0 = 0;
      if (j0 > nc - 3) j0 = nc - 3;
      for (int j = j0; j < j0 + 4; ++j) pts.push_back(j);
    }
    // the matrix row accumulates weights with += into zeros; columns are
    // then contracted in increasing order by the dgemm chain
    std::map<int, double> row;
    for (size_t a = 0; a < pts.size(); ++a) {
      double wt = 1.0;
      for (size_t b = 0; b < pts.size(); ++b)
        if (b != a) wt *= (sp - pts[b]) / (double)(pts[a] - pts[b]);
      if (pts[a] >= 1 && pts[a] <= nc - 1) {
        double& cell = row[pts[a] - 1];
        cell = cell + wt;
      }
    }
    int q = 0;
    for (auto& kv : row) {
      if (kv.second == 0.0) continue;
      idx[r * 4 + q] = kv.first;
      w[r * 4 + q] = kv.second;
      ++q;
    }
    cnt[r] = q;
  }
  CubicTaps* t = new CubicTaps;
  t->nf = nf;
  size_t bi = sizeof(int) * rows, bi4 = sizeof(int) * rows * 4, bw = sizeof(double) * rows * 4;
  if (cudaMalloc(&t->cnt, bi) != cudaSuccess || cudaMalloc(&t->idx, bi4) != cudaSuccess ||
      cudaMalloc(&t->w, bw) != cudaSuccess) {
    set_error("cudaMalloc failed for cubic taps");
    delete t;
    return nullptr;
  }
  cudaMemcpy(t->cnt, cnt.data(), bi, cudaMemcpyHostToDevice);
  cudaMemcpy(t->idx, idx.data(), bi4, cudaMemcpyHostToDevice);
  cudaMemcpy(t->w, w.data(), bw, cudaMemcpyHostToDevice);
  g_taps[nf] = t;
  return t;
}

long long cubic_scratch_doubles(const Geo& gf) {
  Geo gc = make_geo(gf.dim, (gf.N + 1) / 2);
  long long Nf = gf.N, Nc = gc.N;
  if (gf.dim == 1) return 0;
  if (gf.dim == 2) return Nf * gc.sy;
  return Nf * Nc * gc.sy + Nf * Nf * gc.sy;
}

int launch_cubic(const double* coarse, double* fine, const Geo& gf, int accumulate,
                 double* scratch, cudaStream_t s) {
  const CubicTaps* t = cubic_taps(gf.N + 1);
  if (!t) return 2;
  if (gf.dim == 3 && gf.N >= 31 && zmarch_size_ok(gf.N))
    return zlaunch_cubic(coarse, fine, gf, t->cnt, t->idx, t->w, accumulate, s);
  Geo gc = make_geo(gf.dim, (gf.N + 1) / 2);
  const long long Nf = gf.N, Nc = gc.N, pc = gc.sy, pf = gf.sy;
  auto pass = [&](const double* in, double* out, long long A, long long C, long long ia,
                  long long ib, long long oa, long long ob, int acc) {
    long long total = A * Nf * C;
    k_cubic_axis<<<ceil_div(total, 256), 256, 0, s>>>(in, out, A, (int)Nf, C, ia, ib, oa, ob,
                                                      t->cnt, t->idx, t->w, acc);
  };
  PL_PRE(K_INTERP);
  if (gf.dim == 1) {
    pass(coarse, fine, 1, 1, 0, 1, 0, 1, accumulate);
  } else if (gf.dim == 2) {
    // axis 0 (y): (Nc, pc) -> scratch (Nf, pc); axis 1 (x): rows of pc -> fine rows
    pass(coarse, scratch, 1, pc, 0, pc, 0, pc, 0);
    pass(scratch, fine, Nf, 1, pc, 1, pf, 1, accumulate);
  } else {
    double* s1 = scratch;                     // (Nf, Nc, pc)
    double* s2 = scratch + Nf * Nc * pc;      // (Nf, Nf, pc)
    pass(coarse, s1, 1, Nc * pc, 0, Nc * pc, 0, Nc * pc, 0);   // axis 0 (z)
    pass(s1, s2, Nf, pc, Nc * pc, pc, Nf * pc, pc, 0);         // axis 1 (y)
    pass(s2, fine, Nf * Nf, 1, pc, 1, pf, 1, accumulate);     // axis 2 (x)
  }
  double bytes = (accumulate ? 16.0 : 8.0) * gf.npts;
  if (gf.dim >= 2) bytes += 16.0 * (double)cubic_scratch_doubles(gf);
  PL_CHECK_LAUNCH(K_INTERP, bytes);
  return 0;
}

}  // namespace pl
