// 3-D order-2 stencil kernels with a cp.async plane pipeline ("z-marching").
//
// A CTA owns a 32 x 16 (x, y) tile and marches through a chunk of z planes.
// Each plane tile (with its 1- or 2-point halo; Dirichlet ghosts are the
// zero-fill of out-of-domain cp.async copies) is staged into a shared-memory
// ring PREF planes ahead of the plane being computed, so every SM keeps tens
// of KB of loads in flight (the naive one-point-per-thread kernels were
// latency-bound: <0.5 eligible warps per scheduler, see profiles/).  z
// neighbours come from the ring, x/y neighbours from the same smem plane;
// DRAM sees each input field once and each output field once.
//
// Fused sweeps (temporal blocking) run two dependent stages in one pass:
//   k_zrb   one full jor-rb sweep (red on plane z+1, black on plane z)
//   k_zjac2 two Jacobi sweeps (sweep 1 on plane z+1 over the halo-1 region,
//           sweep 2 on plane z over the tile)
// They read u and b once and write u once: 24 B/DOF for the whole fused
// pass instead of 24 B/DOF per stage.  Arithmetic is the reference's
// expression tree (common.cuh), so results are bit-identical to the
// unfused kernels.  Out-of-domain halo points are zero and stay zero: every
// stage forces its value to 0 outside the domain.
#include "common.cuh"
#include "kernels.cuh"

namespace pl {

namespace {

constexpr int TX = 32, TY = 16;           // output tile
constexpr int NTHR = 256;                 // 32 x 8 threads, 2 rows each

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// A W x H plane window with origin (gx0, gy0).  Each thread copies the same
// window elements for every plane, so their in-plane offsets (or "outside
// the domain" = -1, zero-filled) are computed once; a plane then costs one
// 64-bit add, one predicate and one cp.async per element.
template <int W, int H>
struct Window {
  static constexpr int N = W * H;
  static constexpr int PER = (N + NTHR - 1) / NTHR;
  int off[PER];

  __device__ __forceinline__ void init(const Geo& g, int gx0, int gy0, int tid) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      int i = tid + q * NTHR;
      int yy = i / W, xx = i - yy * W;
      int gx = gx0 + xx, gy = gy0 + yy;
      off[q] = (i < N && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny)
                   ? gy * (int)g.sy + gx : -1;
    }
  }
  __device__ __forceinline__ void load(double* dst, const double* src, const Geo& g, int gz,
                                       int tid) const {
    const bool zin = gz >= 0 && gz < g.nz;
    const double* plane = src + (long long)(zin ? gz : 0) * g.sz;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      int i = tid + q * NTHR;
      if (i < N) {
        bool ok = zin && off[q] >= 0;
        cp_async8(dst + i, ok ? plane + off[q] : src, ok);
      }
    }
  }
};

template <bool POW2>
__device__ __forceinline__ double dd2(double x, const OpC& c) {
  return POW2 ? x * c.inv_dx2 : x / c.dx2;
}

// nu * Lap at smem point: planes pm (z-1), pc (z), pp (z+1), row stride W
template <bool POW2, int W>
__device__ __forceinline__ double lap7(const double* pm, const double* pc, const double* pp,
                                       int i, const OpC& c) {
  const double c0 = pc[i];
  double acc = 0.0;
  acc = acc + dd2<POW2>((pm[i] - 2.0 * c0) + pp[i], c);
  acc = acc + dd2<POW2>((pc[i - W] - 2.0 * c0) + pc[i + W], c);
  acc = acc + dd2<POW2>((pc[i - 1] - 2.0 * c0) + pc[i + 1], c);
  return c.nu * acc;
}

enum { Z_APPLY = 0, Z_RESID = 1, Z_JAC = 2, Z_JAC0 = 3 };

// ---------------------------------------------------------------------------
// single-stage kernels: apply, residual, one Jacobi sweep

template <int OP, bool POW2, int PREF>
__global__ void __launch_bounds__(NTHR) k_z1(const double* __restrict__ u,
                                             const double* __restrict__ b,
                                             double* __restrict__ out, Geo g, OpC c,
                                             double sigma, double omega, double dval, int zc) {
  constexpr int HX = TX + 2, HY = TY + 2, PU = HX * HY, PB = TX * TY, RING = PREF + 3;
  constexpr bool NEED_U = OP != Z_JAC0;
  constexpr bool NEED_B = OP != Z_APPLY;
  extern __shared__ double sm[];
  double* su = sm;
  double* sb = sm + (NEED_U ? RING * PU : 0);
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, g.nz);

  Window<HX, HY> wu;
  Window<TX, TY> wb;
  if (NEED_U) wu.init(g, x0 - 1, y0 - 1, tid);
  if (NEED_B) wb.init(g, x0, y0, tid);
  auto load = [&](int zz) {
    if (zz <= z1) {
      int slot = (zz - z0 + 1) % RING;
      if (NEED_U) wu.load(su + slot * PU, u, g, zz, tid);
      if (NEED_B && zz < z1) wb.load(sb + slot * PB, b, g, zz, tid);
    }
    cp_commit();
  };
  if (NEED_U) {
    for (int k = -1; k <= PREF; ++k) load(z0 + k);
  } else {
    cp_commit();
    for (int k = 0; k <= PREF; ++k) load(z0 + k);
  }
  const int gx = x0 + threadIdx.x;
  for (int z = z0; z < z1; ++z) {
    cp_wait<PREF - 1>();
    __syncthreads();
    const int sc = (z - z0 + 1) % RING;
    const double* pc = su + sc * PU;
    const double* pm = su + ((z - z0) % RING) * PU;
    const double* pp = su + ((z - z0 + 2) % RING) * PU;
    const double* pb = sb + sc * PB;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int ly = threadIdx.y + 8 * r;
      const int gy = y0 + ly;
      if (gx < g.nx && gy < g.ny) {
        const long long gi = (long long)z * g.sz + (long long)gy * g.sy + gx;
        const int i = (ly + 1) * HX + threadIdx.x + 1;
        double v;
        if (OP == Z_JAC0) {
          v = 0.0 + ((omega * pb[ly * TX + threadIdx.x]) / dval);
        } else {
          double lap = lap7<POW2, HX>(pm, pc, pp, i, c);
          if (OP == Z_APPLY) {
            v = lap;
          } else {
            double au = pc[i] - sigma * lap;
            double bb = pb[ly * TX + threadIdx.x];
            v = OP == Z_RESID ? bb - au : pc[i] + ((omega * (bb - au)) / dval);
          }
        }
        out[gi] = v;
      }
    }
    __syncthreads();
    load(z + PREF + 1);
  }
  cp_wait<0>();
}

// ---------------------------------------------------------------------------
// fused two-stage kernels.  Input u window has halo 2, the intermediate stage
// (red-updated / once-smoothed u) halo 1.

template <bool RB, bool POW2, int PREF>
__global__ void __launch_bounds__(NTHR) k_z2(const double* __restrict__ u,
                                             const double* __restrict__ b,
                                             double* __restrict__ out, Geo g, OpC c,
                                             double sigma, double omega, double dval, int zc,
                                             int zero_in) {
  constexpr int UX = TX + 4, UY = TY + 4, PU = UX * UY;     // input, halo 2
  constexpr int HX = TX + 2, HY = TY + 2, PH = HX * HY;     // stage 1 + b, halo 1
  constexpr int RU = PREF + 3;    // u planes: the prologue stages z0-2 .. z0+PREF
  constexpr int RB_ = PREF + 1;   // b planes in flight / live (>= PREF)
  extern __shared__ double sm[];
  double* su = sm;                        // RU * PU
  double* sbb = su + RU * PU;             // RB_ * PH
  double* s1 = sbb + RB_ * PH;            // 3 * PH  stage-1 planes z-1, z, z+1
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, g.nz);

  // plane zz of u lives in slot (zz - z0 + 2) % RU (zz >= z0 - 2)
  // plane zz of b lives in slot (zz - z0 + 1) % RB_ (zz >= z0 - 1)
  Window<UX, UY> wu;
  Window<HX, HY> wb;
  wu.init(g, x0 - 2, y0 - 2, tid);
  wb.init(g, x0 - 1, y0 - 1, tid);
  auto load = [&](int zz) {            // u plane zz and b plane zz - 1
    if (zz <= z1 + 1 && !zero_in) wu.load(su + ((zz - z0 + 2) % RU) * PU, u, g, zz, tid);
    const int zb = zz - 1;
    if (zb >= z0 - 1 && zb <= z1) wb.load(sbb + ((zb - z0 + 1) % RB_) * PH, b, g, zb, tid);
    cp_commit();
  };
  // stage 1 at plane zz over the halo-1 window (value 0 outside the domain);
  // each thread owns the same <= 3 window points on every plane
  constexpr int PER1 = (PH + NTHR - 1) / NTHR;
  int e_k[PER1], e_i[PER1], e_par[PER1];
  bool e_in[PER1];
#pragma unroll
  for (int q = 0; q < PER1; ++q) {
    int k = tid + q * NTHR;
    int yy = k / HX, xx = k - yy * HX;
    int gxx = x0 - 1 + xx, gyy = y0 - 1 + yy;
    e_k[q] = k;
    e_i[q] = (yy + 1) * UX + xx + 1;
    e_in[q] = k < PH && gxx >= 0 && gxx < g.nx && gyy >= 0 && gyy < g.ny;
    e_par[q] = (gxx + gyy + 3) & 1;
  }
  auto stage1 = [&](int zz) {
    double* dst = s1 + ((zz - z0 + 3) % 3) * PH;
    const bool zin = zz >= 0 && zz < g.nz;
    const double* pm = su + ((zz - 1 - z0 + 2 + RU) % RU) * PU;
    const double* pc = su + ((zz - z0 + 2) % RU) * PU;
    const double* pp = su + ((zz + 1 - z0 + 2) % RU) * PU;
    const double* pb = sbb + ((zz - z0 + 1) % RB_) * PH;
#pragma unroll
    for (int q = 0; q < PER1; ++q) {
      const int k = e_k[q];
      if (k < PH) {
        double v = 0.0;
        if (zin && e_in[q]) {
          const int i = e_i[q];
          double bb = pb[k];
          if (RB) {
            bool red = ((e_par[q] + zz) & 1) == 0;
            if (red) {
              double r = bb - (pc[i] - sigma * lap7<POW2, UX>(pm, pc, pp, i, c));
              v = pc[i] + ((omega * r) / dval);
            } else {
              v = pc[i];
            }
          } else if (zero_in) {
            v = 0.0 + ((omega * bb) / dval);
          } else {
            double au = pc[i] - sigma * lap7<POW2, UX>(pm, pc, pp, i, c);
            v = pc[i] + ((omega * (bb - au)) / dval);
          }
        }
        dst[k] = v;
      }
    }
  };

  for (int k = -2; k <= PREF; ++k) load(z0 + k);     // u: z0-2..z0+PREF
  // prologue: stage-1 planes z0-1 and z0 need u up to z0+1 and b up to z0
  cp_wait<PREF - 1>();
  __syncthreads();
  stage1(z0 - 1);
  stage1(z0);
  const int gx = x0 + threadIdx.x;
  for (int z = z0; z < z1; ++z) {
    // stage 1 at z+1 needs u plane z+2 and b plane z+1: groups up to z+2
    cp_wait<PREF - 2>();
    __syncthreads();
    stage1(z + 1);
    __syncthreads();
    const double* qm = s1 + ((z - 1 - z0 + 3) % 3) * PH;
    const double* qc = s1 + ((z - z0 + 3) % 3) * PH;
    const double* qp = s1 + ((z + 1 - z0 + 3) % 3) * PH;
    const double* pb = sbb + ((z - z0 + 1) % RB_) * PH;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int ly = threadIdx.y + 8 * r;
      const int gy = y0 + ly;
      if (gx < g.nx && gy < g.ny) {
        const int i = (ly + 1) * HX + threadIdx.x + 1;
        double v;
        if (RB) {
          bool red = ((gx + gy + z + 3) & 1) == 0;
          if (red) {
            v = qc[i];
          } else {
            double rr = pb[i] - (qc[i] - sigma * lap7<POW2, HX>(qm, qc, qp, i, c));
            v = qc[i] + ((omega * rr) / dval);
          }
        } else {
          double au = qc[i] - sigma * lap7<POW2, HX>(qm, qc, qp, i, c);
          v = qc[i] + ((omega * (pb[i] - au)) / dval);
        }
        out[(long long)z * g.sz + (long long)gy * g.sy + gx] = v;
      }
    }
    __syncthreads();
    load(z + PREF + 1);
  }
  cp_wait<0>();
}

constexpr int PREF1 = 3;
constexpr int PREF2 = 3;

int pick_zc(const Geo& g) {
  // enough CTAs for several waves on 148 SMs; chunk halo planes cost
  // (2 or 4)/zc extra L2 reads
  long long tiles = (long long)ceil_div(g.nx, TX) * ceil_div(g.ny, TY);
  int zc = 64;
  while (zc > 16 && tiles * ceil_div(g.nz, zc) < 148 * 8) zc /= 2;
  return zc;
}

template <int OP>
int launch_z1(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
              double sigma, double omega, double dval, cudaStream_t s) {
  constexpr int HX = TX + 2, HY = TY + 2, RING = PREF1 + 3;
  size_t smem = sizeof(double) * RING *
                ((OP != Z_JAC0 ? HX * HY : 0) + (OP != Z_APPLY ? TX * TY : 0));
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc)), block(32, 8);
  auto kern = c.pow2 ? k_z1<OP, true, PREF1> : k_z1<OP, false, PREF1>;
  static bool set[2] = {false, false};
  if (!set[c.pow2]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    set[c.pow2] = true;
  }
  kern<<<grid, block, smem, s>>>(u, b, out, g, c, sigma, omega, dval, zc);
  return 0;
}

template <bool RB>
int launch_z2(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
              double sigma, double omega, double dval, int zero_in, cudaStream_t s) {
  constexpr int UX = TX + 4, UY = TY + 4, HX = TX + 2, HY = TY + 2;
  size_t smem = sizeof(double) * ((PREF2 + 3) * UX * UY + (PREF2 + 1) * HX * HY + 3 * HX * HY);
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc)), block(32, 8);
  auto kern = c.pow2 ? k_z2<RB, true, PREF2> : k_z2<RB, false, PREF2>;
  static bool set[2] = {false, false};
  if (!set[c.pow2]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    set[c.pow2] = true;
  }
  kern<<<grid, block, smem, s>>>(u, b, out, g, c, sigma, omega, dval, zc, zero_in);
  return 0;
}

}  // namespace

// host value of 1 - sigma * (nu * ((0 + d) + d + d)) for order 2 (constant)
double zdiag(const OpC& c, double sigma) {
  double t = 0.0;
  t = t + c.d1_int;
  t = t + c.d1_int;
  t = t + c.d1_int;
  return 1.0 - sigma * (c.nu * t);
}

int g_zmarch_enabled = 1;   // runtime knob (pl_set_option), for A/B tests

bool zmarch_ok(const Geo& g, const OpC& c) {
  return g_zmarch_enabled && g.dim == 3 && c.order == 2 && g.N >= 31;
}

int zlaunch_apply(const double* u, double* f, const Geo& g, const OpC& c, cudaStream_t s) {
  PL_PRE(K_APPLY);
  launch_z1<Z_APPLY>(u, nullptr, f, g, c, 0.0, 0.0, 1.0, s);
  PL_CHECK_LAUNCH(K_APPLY, 16.0 * g.npts);
  return 0;
}

int zlaunch_residual(const double* u, const double* b, double* r, const Geo& g, const OpC& c,
                     double sigma, cudaStream_t s) {
  PL_PRE(K_RESID);
  launch_z1<Z_RESID>(u, b, r, g, c, sigma, 0.0, 1.0, s);
  PL_CHECK_LAUNCH(K_RESID, 24.0 * g.npts);
  return 0;
}

int zlaunch_jacobi(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                   double sigma, double omega, int zero_in, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  PL_PRE(K_JACOBI);
  if (zero_in) launch_z1<Z_JAC0>(u, b, out, g, c, sigma, omega, dval, s);
  else launch_z1<Z_JAC>(u, b, out, g, c, sigma, omega, dval, s);
  PL_CHECK_LAUNCH(K_JACOBI, (zero_in ? 16.0 : 24.0) * g.npts);
  return 0;
}

int zlaunch_jacobi2(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                    double sigma, double omega, int zero_in, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  PL_PRE(K_JACOBI);
  launch_z2<false>(u, b, out, g, c, sigma, omega, dval, zero_in, s);
  // algorithmic bytes of the two unfused sweeps it replaces
  PL_CHECK_LAUNCH(K_JACOBI, (zero_in ? 40.0 : 48.0) * g.npts);
  return 0;
}

int zlaunch_rb(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
               double sigma, double omega, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  PL_PRE(K_RB);
  launch_z2<true>(u, b, out, g, c, sigma, omega, dval, 0, s);
  PL_CHECK_LAUNCH(K_RB, 24.0 * g.npts);
  return 0;
}

}  // namespace pl
