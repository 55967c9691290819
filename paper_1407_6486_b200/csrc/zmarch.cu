// 3-D order-2 stencil kernels fed by TMA ("z-marching").
//
// A CTA owns a 32 x 16 (x, y) tile and marches through a chunk of z planes.
// Each plane window (tile plus a 1- or 2-point halo) arrives in shared memory
// through one cp.async.bulk.tensor copy issued by a single thread; the
// tensor map covers only the interior points, so out-of-domain halo points
// -- the homogeneous Dirichlet ghosts -- are zero-filled by the TMA unit and
// the padded rows of the device layout are never read.  Copies run PREF
// planes ahead of the plane being computed and complete on per-slot
// mbarriers; no SM instruction is spent on address arithmetic for loads.
//
// Fused sweeps (temporal blocking) run two dependent stages in one pass:
//   k_z2<RB>  one full jor-rb sweep (red on plane z+1 over the halo-1 window,
//             black on plane z over the tile)
//   k_z2<Jac> two Jacobi sweeps (sweep 1 on plane z+1 over the halo-1 window,
//             sweep 2 on plane z)
// They read u and b once and write u once per pass.  Arithmetic is the
// reference's expression tree (common.cuh), bit-identical to the unfused
// kernels; out-of-domain stage-1 points are forced to zero.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace pl {

namespace {

constexpr int TX = 32, TY = 16;           // output tile
constexpr int NTHR = 256;                 // 32 x 8 threads, 2 rows each

// ---- TMA / mbarrier primitives --------------------------------------------

__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int x, int y, int z,
                                     unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(saddr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__host__ __device__ constexpr int align16(int n) { return (n + 15) / 16 * 16; }  // doubles -> 128 B

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
__global__ void __launch_bounds__(NTHR) k_z1(const __grid_constant__ CUtensorMap mu,
                                             const __grid_constant__ CUtensorMap mb,
                                             double* __restrict__ out, Geo g, OpC c,
                                             double sigma, double omega, double dval, int zc) {
  // TMA needs the innermost box start 16-byte aligned: windows start at the
  // even column x0-2 (one extra column on the left, unused)
  constexpr int HX = TX + 4, HY = TY + 2, PU = align16(HX * HY), PB = align16(TX * TY);
  constexpr int RING = PREF + 3;
  constexpr bool NEED_U = OP != Z_JAC0;
  constexpr bool NEED_B = OP != Z_APPLY;
  extern __shared__ __align__(128) double sm[];
  double* su = sm;
  double* sb = sm + (NEED_U ? RING * PU : 0);
  unsigned long long* bar = (unsigned long long*)(sb + (NEED_B ? RING * PB : 0));
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, g.nz);
  if (tid == 0) {
    for (int i = 0; i < RING; ++i) mbar_init(bar + i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  // plane p (z0-1 <= p <= z1) uses slot (p - z0 + 1) % RING, its k-th use
  // waits on parity k & 1.  Every plane in range arrives exactly once.
  auto issue = [&](int p) {
    if (p > z1) return;
    const int slot = (p - z0 + 1) % RING;
    const bool wu = NEED_U;
    const bool wb = NEED_B && p >= z0 && p < z1;
    if (!wu && !wb) {
      mbar_arrive(bar + slot);
      return;
    }
    mbar_expect(bar + slot, (wu ? HX * HY * 8u : 0u) + (wb ? TX * TY * 8u : 0u));
    if (wu) tma3(su + slot * PU, &mu, x0 - 2, y0 - 1, p, bar + slot);
    if (wb) tma3(sb + slot * PB, &mb, x0, y0, p, bar + slot);
  };
  auto wait = [&](int p) {
    const int k = p - z0 + 1;
    mbar_wait(bar + k % RING, (unsigned)((k / RING) & 1));
  };
  if (tid == 0)
    for (int p = z0 - 1; p <= z0 + PREF; ++p) issue(p);
  wait(z0 - 1);
  wait(z0);
  const int gx = x0 + threadIdx.x;
  for (int z = z0; z < z1; ++z) {
    wait(z + 1);
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
        const int i = (ly + 1) * HX + threadIdx.x + 2;
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
        out[g.at(gx, gy, z)] = v;
      }
    }
    __syncthreads();   // slot of plane z-1 is free
    if (tid == 0) issue(z + PREF + 1);
  }
}

// ---------------------------------------------------------------------------
// fused two-stage kernels.  Input u window has halo 2, stage 1 and b halo 1.

template <bool RB, bool POW2, int PREF>
__global__ void __launch_bounds__(NTHR) k_z2(const __grid_constant__ CUtensorMap mu,
                                             const __grid_constant__ CUtensorMap mb,
                                             double* __restrict__ out, Geo g, OpC c,
                                             double sigma, double omega, double dval, int zc,
                                             int zero_in) {
  constexpr int UX = TX + 4, UY = TY + 4, PU = align16(UX * UY);    // input, halo 2
  constexpr int HX = TX + 2, HY = TY + 2, PH = align16(HX * HY);    // stage 1, halo 1
  constexpr int NH = HX * HY;
  constexpr int BW = TX + 4, PBW = align16(BW * HY);   // b window from the even column x0-2
  constexpr int RU = PREF + 3;    // u planes z0-2 .. z0+PREF staged in the prologue
  constexpr int RBB = PREF + 1;   // b planes
  extern __shared__ __align__(128) double sm[];
  double* su = sm;                        // RU * PU
  double* sbb = su + RU * PU;             // RBB * PBW
  double* s1 = sbb + RBB * PBW;           // 3 * PH  stage-1 planes z-1, z, z+1
  unsigned long long* bu = (unsigned long long*)(s1 + 3 * PH);
  unsigned long long* bbar = bu + RU;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, g.nz);
  if (tid == 0) {
    for (int i = 0; i < RU; ++i) mbar_init(bu + i, 1);
    for (int i = 0; i < RBB; ++i) mbar_init(bbar + i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  // u plane p (z0-2 <= p <= z1+1): slot (p - z0 + 2) % RU
  // b plane q (z0-1 <= q <= z1):   slot (q - z0 + 1) % RBB
  auto issue = [&](int p) {          // u plane p and b plane p - 1
    if (p <= z1 + 1) {
      const int k = p - z0 + 2;
      if (zero_in) {
        mbar_arrive(bu + k % RU);
      } else {
        mbar_expect(bu + k % RU, UX * UY * 8u);
        tma3(su + (k % RU) * PU, &mu, x0 - 2, y0 - 2, p, bu + k % RU);
      }
    }
    const int q = p - 1;
    if (q >= z0 - 1 && q <= z1) {
      const int k = q - z0 + 1;
      mbar_expect(bbar + k % RBB, BW * HY * 8u);
      tma3(sbb + (k % RBB) * PBW, &mb, x0 - 2, y0 - 1, q, bbar + k % RBB);
    }
  };
  auto wait_u = [&](int p) {
    const int k = p - z0 + 2;
    mbar_wait(bu + k % RU, (unsigned)((k / RU) & 1));
  };
  auto wait_b = [&](int q) {
    const int k = q - z0 + 1;
    mbar_wait(bbar + k % RBB, (unsigned)((k / RBB) & 1));
  };

  // each thread owns the same <= 3 stage-1 window points on every plane
  constexpr int PER1 = (NH + NTHR - 1) / NTHR;
  int e_k[PER1], e_i[PER1], e_b[PER1], e_par[PER1];
  bool e_in[PER1];
#pragma unroll
  for (int q = 0; q < PER1; ++q) {
    int k = tid + q * NTHR;
    int yy = k / HX, xx = k - yy * HX;
    int gxx = x0 - 1 + xx, gyy = y0 - 1 + yy;
    e_k[q] = k;
    e_i[q] = (yy + 1) * UX + xx + 1;
    e_b[q] = yy * BW + xx + 1;
    e_in[q] = k < NH && gxx >= 0 && gxx < g.nx && gyy >= 0 && gyy < g.ny;
    e_par[q] = (gxx + gyy + 3) & 1;
  }
  auto stage1 = [&](int zz) {
    double* dst = s1 + ((zz - z0 + 3) % 3) * PH;
    const bool zin = zz >= 0 && zz < g.nz;
    const double* pm = su + ((zz - 1 - z0 + 2 + RU) % RU) * PU;
    const double* pc = su + ((zz - z0 + 2) % RU) * PU;
    const double* pp = su + ((zz + 1 - z0 + 2) % RU) * PU;
    const double* pb = sbb + ((zz - z0 + 1) % RBB) * PBW;
#pragma unroll
    for (int q = 0; q < PER1; ++q) {
      const int k = e_k[q];
      if (k < NH) {
        double v = 0.0;
        if (zin && e_in[q]) {
          const int i = e_i[q];
          double b = pb[e_b[q]];
          if (RB) {
            bool red = ((e_par[q] + zz) & 1) == 0;
            if (red) {
              double r = b - (pc[i] - sigma * lap7<POW2, UX>(pm, pc, pp, i, c));
              v = pc[i] + ((omega * r) / dval);
            } else {
              v = pc[i];
            }
          } else if (zero_in) {
            v = 0.0 + ((omega * b) / dval);
          } else {
            double au = pc[i] - sigma * lap7<POW2, UX>(pm, pc, pp, i, c);
            v = pc[i] + ((omega * (b - au)) / dval);
          }
        }
        dst[k] = v;
      }
    }
  };

  if (tid == 0)
    for (int p = z0 - 2; p <= z0 + PREF; ++p) issue(p);
  // prologue: stage-1 planes z0-1, z0 need u z0-2 .. z0+1 and b z0-1, z0
  for (int p = z0 - 2; p <= z0 + 1; ++p) wait_u(p);
  wait_b(z0 - 1);
  wait_b(z0);
  stage1(z0 - 1);
  stage1(z0);
  const int gx = x0 + threadIdx.x;
  for (int z = z0; z < z1; ++z) {
    wait_u(z + 2);
    wait_b(z + 1);
    stage1(z + 1);
    __syncthreads();
    const double* qm = s1 + ((z - 1 - z0 + 3) % 3) * PH;
    const double* qc = s1 + ((z - z0 + 3) % 3) * PH;
    const double* qp = s1 + ((z + 1 - z0 + 3) % 3) * PH;
    const double* pb = sbb + ((z - z0 + 1) % RBB) * PBW;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int ly = threadIdx.y + 8 * r;
      const int gy = y0 + ly;
      if (gx < g.nx && gy < g.ny) {
        const int i = (ly + 1) * HX + threadIdx.x + 1;
        const int ib = (ly + 1) * BW + threadIdx.x + 2;
        double v;
        if (RB) {
          bool red = ((gx + gy + z + 3) & 1) == 0;
          if (red) {
            v = qc[i];
          } else {
            double rr = pb[ib] - (qc[i] - sigma * lap7<POW2, HX>(qm, qc, qp, i, c));
            v = qc[i] + ((omega * rr) / dval);
          }
        } else {
          double au = qc[i] - sigma * lap7<POW2, HX>(qm, qc, qp, i, c);
          v = qc[i] + ((omega * (pb[ib] - au)) / dval);
        }
        out[g.at(gx, gy, z)] = v;
      }
    }
    __syncthreads();   // u plane z, b plane z and stage-1 plane z-1 are free
    if (tid == 0) issue(z + PREF + 1);
  }
}

// ---------------------------------------------------------------------------
// one full jor-rb sweep in one pass, divergence-free.  With the 7-point
// stencil a red point reads only black neighbours and its own old value, so
// the red update of plane z+1 is done IN PLACE in the staged u window (no
// copy of black points); the black update of plane z then reads the updated
// red neighbours straight from the window.  Red work is a dense list of the
// window's red points (17 per row); black work gives every thread one
// (black, red) x-pair of a tile row, so no warp branches on colour.

template <bool POW2, int PREF>
__global__ void __launch_bounds__(NTHR) k_zrb(const __grid_constant__ CUtensorMap mu,
                                              const __grid_constant__ CUtensorMap mb,
                                              double* __restrict__ out, Geo g, OpC c,
                                              double sigma, double omega, double dval, int zc) {
  constexpr int UX = TX + 4, UY = TY + 4, PU = align16(UX * UY);    // u window, halo 2
  constexpr int BW = TX + 4, BH = TY + 2, PB = align16(BW * BH);    // b window, halo 1
  constexpr int RU = PREF + 3, RBB = PREF + 1;
  constexpr int NRED = (TX + 2) / 2 * (TY + 2);                     // red points of halo-1
  constexpr int PERR = (NRED + NTHR - 1) / NTHR;
  extern __shared__ __align__(128) double sm[];
  double* su = sm;
  double* sbb = su + RU * PU;
  unsigned long long* bu = (unsigned long long*)(sbb + RBB * PB);
  unsigned long long* bbar = bu + RU;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, g.nz);
  if (tid == 0) {
    for (int i = 0; i < RU; ++i) mbar_init(bu + i, 1);
    for (int i = 0; i < RBB; ++i) mbar_init(bbar + i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int p) {          // u plane p and b plane p - 1
    if (p <= z1 + 1) {
      const int k = p - z0 + 2;
      mbar_expect(bu + k % RU, UX * UY * 8u);
      tma3(su + (k % RU) * PU, &mu, x0 - 2, y0 - 2, p, bu + k % RU);
    }
    const int q = p - 1;
    if (q >= z0 - 1 && q <= z1) {
      const int k = q - z0 + 1;
      mbar_expect(bbar + k % RBB, BW * BH * 8u);
      tma3(sbb + (k % RBB) * PB, &mb, x0 - 2, y0 - 1, q, bbar + k % RBB);
    }
  };
  auto wait_u = [&](int p) {
    const int k = p - z0 + 2;
    mbar_wait(bu + k % RU, (unsigned)((k / RU) & 1));
  };
  auto wait_b = [&](int q) {
    const int k = q - z0 + 1;
    mbar_wait(bbar + k % RBB, (unsigned)((k / RBB) & 1));
  };
  // red list: window point j -> (yy, xx) with xx = 2 (j % 17) + ((yy + zz + 1) & 1)
  // (x0, y0 even); per plane parity: u-window index, b-window index, in-domain
  int r_iu[2][PERR], r_ib[2][PERR];
  bool r_in[2][PERR];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int q = 0; q < PERR; ++q) {
      int j = tid + q * NTHR;
      int yy = j / ((TX + 2) / 2), xr = j - yy * ((TX + 2) / 2);
      int xx = 2 * xr + ((yy + par + 1) & 1);
      int gx = x0 - 1 + xx, gy = y0 - 1 + yy;
      r_iu[par][q] = (yy + 1) * UX + xx + 1;
      r_ib[par][q] = yy * BW + xx + 1;
      r_in[par][q] = j < NRED && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny;
    }
  // black pair: tile row `row`, x = 2 px + {0, 1}; black x has (x + row + z) even
  const int px = tid & 15, row = tid >> 4;
  const int gy = y0 + row;
  auto red_update = [&](int zz) {
    if (zz < 0 || zz >= g.nz) return;       // ghost planes stay zero
    const int par = zz & 1;
    double* pc = su + ((zz - z0 + 2) % RU) * PU;
    const double* pm = su + ((zz - 1 - z0 + 2 + RU) % RU) * PU;
    const double* pp = su + ((zz + 1 - z0 + 2) % RU) * PU;
    const double* pb = sbb + ((zz - z0 + 1) % RBB) * PB;
#pragma unroll
    for (int q = 0; q < PERR; ++q) {
      if (r_in[par][q]) {
        const int i = r_iu[par][q];
        const double r = pb[r_ib[par][q]] - (pc[i] - sigma * lap7<POW2, UX>(pm, pc, pp, i, c));
        pc[i] = pc[i] + ((omega * r) / dval);
      }
    }
  };

  if (tid == 0)
    for (int p = z0 - 2; p <= z0 + PREF; ++p) issue(p);
  // prologue: red planes z0-1 (needs u z0-2..z0, b z0-1) and z0
  for (int p = z0 - 2; p <= z0 + 1; ++p) wait_u(p);
  wait_b(z0 - 1);
  wait_b(z0);
  red_update(z0 - 1);
  __syncthreads();
  red_update(z0);
  for (int z = z0; z < z1; ++z) {
    wait_u(z + 2);
    wait_b(z + 1);
    __syncthreads();                          // red planes <= z complete
    red_update(z + 1);
    __syncthreads();
    const int par = (row + z) & 1;
    const int xb = 2 * px + par, xr = 2 * px + 1 - par;
    const double* pm = su + ((z - 1 - z0 + 2 + RU) % RU) * PU;
    const double* pc = su + ((z - z0 + 2) % RU) * PU;
    const double* pp = su + ((z + 1 - z0 + 2) % RU) * PU;
    const double* pb = sbb + ((z - z0 + 1) % RBB) * PB;
    if (gy < g.ny) {
      const int gxb = x0 + xb, gxr = x0 + xr;
      const int ib = (row + 2) * UX + xb + 2;
      if (gxb < g.nx) {
        const double rr =
            pb[(row + 1) * BW + xb + 2] - (pc[ib] - sigma * lap7<POW2, UX>(pm, pc, pp, ib, c));
        out[g.at(gxb, gy, z)] = pc[ib] + ((omega * rr) / dval);
      }
      if (gxr < g.nx) out[g.at(gxr, gy, z)] = pc[(row + 2) * UX + xr + 2];
    }
    __syncthreads();   // u plane z-1 and b plane z are free
    if (tid == 0) issue(z + PREF + 1);
  }
}

constexpr int PREF1 = 3;
constexpr int PREF2 = 3;

// ---- host: tensor maps -----------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_encode_mu;

int get_encode() {
  std::lock_guard<std::mutex> lk(g_encode_mu);
  if (g_encode) return 0;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 2;
  }
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return 0;
}

int make_map(CUtensorMap* m, const double* base, const Geo& g, int bw, int bh) {
  PL_TRY(get_encode());
  cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz};
  cuuint64_t strides[2] = {(cuuint64_t)g.sy * 8, (cuuint64_t)g.sz * 8};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): base %p pitch %lld", (int)r, (void*)base,
              (long long)g.sy);
    return 2;
  }
  return 0;
}

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
  constexpr int HX = TX + 4, HY = TY + 2, RING = PREF1 + 3;
  CUtensorMap mu, mb;
  std::memset(&mu, 0, sizeof(mu));
  std::memset(&mb, 0, sizeof(mb));
  if (OP != Z_JAC0) PL_TRY(make_map(&mu, u, g, HX, HY));
  if (OP != Z_APPLY) PL_TRY(make_map(&mb, b, g, TX, TY));
  size_t smem = sizeof(double) * RING *
                    ((OP != Z_JAC0 ? align16(HX * HY) : 0) +
                     (OP != Z_APPLY ? align16(TX * TY) : 0)) +
                8 * RING;
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc)), block(32, 8);
  auto kern = c.pow2 ? k_z1<OP, true, PREF1> : k_z1<OP, false, PREF1>;
  static bool set[2] = {false, false};
  if (!set[c.pow2]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    set[c.pow2] = true;
  }
  kern<<<grid, block, smem, s>>>(mu, mb, out, g, c, sigma, omega, dval, zc);
  return 0;
}

template <bool RB>
int launch_z2(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
              double sigma, double omega, double dval, int zero_in, cudaStream_t s) {
  constexpr int UX = TX + 4, UY = TY + 4, HX = TX + 2, HY = TY + 2, BW = TX + 4;
  CUtensorMap mu, mb;
  std::memset(&mu, 0, sizeof(mu));
  if (!zero_in) PL_TRY(make_map(&mu, u, g, UX, UY));
  PL_TRY(make_map(&mb, b, g, BW, HY));
  size_t smem = sizeof(double) * ((PREF2 + 3) * align16(UX * UY) +
                                  (PREF2 + 1) * align16(BW * HY) + 3 * align16(HX * HY)) +
                8 * ((PREF2 + 3) + (PREF2 + 1));
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc)), block(32, 8);
  auto kern = c.pow2 ? k_z2<RB, true, PREF2> : k_z2<RB, false, PREF2>;
  static bool set[2] = {false, false};
  if (!set[c.pow2]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    set[c.pow2] = true;
  }
  kern<<<grid, block, smem, s>>>(mu, mb, out, g, c, sigma, omega, dval, zc, zero_in);
  return 0;
}

int launch_zrb(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
               double sigma, double omega, double dval, cudaStream_t s) {
  constexpr int UX = TX + 4, UY = TY + 4, BW = TX + 4, BH = TY + 2;
  CUtensorMap mu, mb;
  PL_TRY(make_map(&mu, u, g, UX, UY));
  PL_TRY(make_map(&mb, b, g, BW, BH));
  size_t smem = sizeof(double) * ((PREF2 + 3) * align16(UX * UY) + (PREF2 + 1) * align16(BW * BH)) +
                8 * ((PREF2 + 3) + (PREF2 + 1));
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc)), block(32, 8);
  auto kern = c.pow2 ? k_zrb<true, PREF2> : k_zrb<false, PREF2>;
  static bool set[2] = {false, false};
  if (!set[c.pow2]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    set[c.pow2] = true;
  }
  kern<<<grid, block, smem, s>>>(mu, mb, out, g, c, sigma, omega, dval, zc);
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
  // TMA needs 16-byte row and plane strides: the padded device layout
  return g_zmarch_enabled && g.dim == 3 && c.order == 2 && g.N >= 31 && (g.sy % 2) == 0;
}

int zlaunch_apply(const double* u, double* f, const Geo& g, const OpC& c, cudaStream_t s) {
  PL_PRE(K_APPLY);
  PL_TRY(launch_z1<Z_APPLY>(u, nullptr, f, g, c, 0.0, 0.0, 1.0, s));
  PL_CHECK_LAUNCH(K_APPLY, 16.0 * g.npts);
  return 0;
}

int zlaunch_residual(const double* u, const double* b, double* r, const Geo& g, const OpC& c,
                     double sigma, cudaStream_t s) {
  PL_PRE(K_RESID);
  PL_TRY(launch_z1<Z_RESID>(u, b, r, g, c, sigma, 0.0, 1.0, s));
  PL_CHECK_LAUNCH(K_RESID, 24.0 * g.npts);
  return 0;
}

int zlaunch_jacobi(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                   double sigma, double omega, int zero_in, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  PL_PRE(K_JACOBI);
  if (zero_in) PL_TRY(launch_z1<Z_JAC0>(u, b, out, g, c, sigma, omega, dval, s));
  else PL_TRY(launch_z1<Z_JAC>(u, b, out, g, c, sigma, omega, dval, s));
  PL_CHECK_LAUNCH(K_JACOBI, (zero_in ? 16.0 : 24.0) * g.npts);
  return 0;
}

int zlaunch_jacobi2(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                    double sigma, double omega, int zero_in, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  PL_PRE(K_JACOBI);
  PL_TRY(launch_z2<false>(u, b, out, g, c, sigma, omega, dval, zero_in, s));
  // algorithmic bytes of the two unfused sweeps it replaces
  PL_CHECK_LAUNCH(K_JACOBI, (zero_in ? 40.0 : 48.0) * g.npts);
  return 0;
}

int zlaunch_rb(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
               double sigma, double omega, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  PL_PRE(K_RB);
  PL_TRY(launch_zrb(u, b, out, g, c, sigma, omega, dval, s));
  PL_CHECK_LAUNCH(K_RB, 24.0 * g.npts);
  return 0;
}

}  // namespace pl
