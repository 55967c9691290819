// 3-D order-2 stencil kernels fed by TMA ("z-marching").
//
// A CTA owns a 32 x 16 (x, y) tile and marches through a chunk of z planes.
// Each plane window (tile plus halo) arrives in shared memory through one
// cp.async.bulk.tensor copy issued by a single thread; the tensor map covers
// only the interior points, so out-of-domain halo points -- the homogeneous
// Dirichlet ghosts -- are zero-filled by the TMA unit and the padded rows of
// the device layout are never read.  Copies run PREF planes ahead of the
// plane being computed and complete on per-slot mbarriers.  TMA requires the
// innermost box start to be 16-byte aligned, so every window starts at the
// even column x0-2.
//
// Kernels
//   k_z1<op>     one stage: heat apply, residual, or one Jacobi sweep
//   k_z2<PRO>    two fused Jacobi sweeps (sweep 1 on plane z+1 over the halo-1
//                window, sweep 2 on plane z)
//   k_zrb<PRO>   one fused jor-rb sweep: red points of plane z+1 are updated
//                in place in the staged window (a red point reads only black
//                neighbours and itself), black points of plane z then read
//                the updated reds -- no colour divergence inside a warp
// With PRO (prolongation fused, multigrid.py:250) every staged u plane first
// receives u += P_lin e_c in shared memory, the coarse correction planes
// arriving by TMA on the same barriers, so the post-smoother replaces the
// separate prolongation pass.  Arithmetic is the reference's expression tree
// (common.cuh / transfer_dev.cuh), bit-identical to the unfused kernels.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <vector>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "transfer_dev.cuh"

namespace pl {

extern int g_zrb_ring;   // PL_OPT_ZRB_RING: 0 8+4 plane rings (3 CTAs/SM), 1 6+3 (4 CTAs/SM)

namespace {

constexpr int TX = 32, TY = 16;           // output tile
constexpr int NTHR = 256;                 // k_z1 / k_z2: 32 x 8 threads, 2 rows each

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

__host__ __device__ constexpr int align16(int n) { return (n + 15) / 16 * 16; }  // 128 B

// z-chunk of this CTA.  A negative chunk length asks for the reverse chunk
// order: a kernel that streams a field right after another kernel streamed
// it forwards then starts on the planes still resident in the 126 MB L2.
__device__ __forceinline__ int zchunk_block(int& zc) {
  if (zc < 0) {
    zc = -zc;
    return gridDim.z - 1 - blockIdx.z;
  }
  return blockIdx.z;
}

// acc + ((m - 2 c0) + p) / dx^2, one axis of the order-2 Laplacian.  For a
// power-of-two dx^2 <= 1 (OpC::pow2) the scaling by 1 / dx^2 is exact, hence
// fma(t, 1 / dx^2, acc) == acc + t / dx^2 bit for bit (short of overflow):
// the reference's value with one dependent operation less per axis.  (Folding
// m - 2 c0 into an FMA as well is just as exact but costs the red-black sweep
// registers: 116 instead of 24 bytes of spill loads.)
template <bool POW2>
__device__ __forceinline__ double axis_acc(double acc, double m, double c0, double p,
                                           const OpC& c) {
  const double t = (m - 2.0 * c0) + p;
  return POW2 ? __fma_rn(t, c.inv_dx2, acc) : acc + t / c.dx2;
}

// nu * Lap at smem point: planes pm (z-1), pc (z), pp (z+1), row stride W
template <bool POW2, int W>
__device__ __forceinline__ double lap7(const double* pm, const double* pc, const double* pp,
                                       int i, const OpC& c) {
  const double c0 = pc[i];
  double acc = 0.0;
  acc = axis_acc<POW2>(acc, pm[i], c0, pp[i], c);
  acc = axis_acc<POW2>(acc, pc[i - W], c0, pc[i + W], c);
  acc = axis_acc<POW2>(acc, pc[i - 1], c0, pc[i + 1], c);
  return c.nu * acc;
}

enum { Z_APPLY = 0, Z_RESID = 1, Z_JAC = 2, Z_JAC0 = 3, Z_APPLY_RHS = 4 };

// Z_APPLY_RHS epilogue operands: the next sub-step's right-hand side
// r = (y - dtm f_next) + s (+ (t1 - t0)) from the same u plane (sdc.py:102-104)
struct RhsArgs {
  const double* fn;
  const double* s;
  const double* t0;
  const double* t1;
  double* r;
  double dtm;
};

// ---- shared machinery of the halo-2 kernels -------------------------------

constexpr int UX = TX + 4, UY = TY + 4, PU = align16(UX * UY);   // u window (halo 2)
constexpr int BW = TX + 4, BH = TY + 2, PB = align16(BW * BH);   // b window (halo 1)
constexpr int CW = TX / 2 + 4, CH = TY / 2 + 3, PC = align16(CW * CH);   // coarse e window
constexpr int RC = 6;                                                    // coarse ring

// linear interpolation tap along one axis for fine index i (transfers.py:40-45)
__device__ __forceinline__ void ltap(int i, int& j0, int& j1, bool& two) {
  if (i & 1) {
    j0 = (i - 1) >> 1; j1 = j0; two = false;
  } else {
    j0 = (i >> 1) - 1; j1 = i >> 1; two = true;
  }
}
__device__ __forceinline__ double lcomb(double a, double b, bool two) {
  return two ? 0.5 * (a + b) : a;
}

// u += P_lin e on a staged window plane, separably and in the tree order of
// transfer_dev.cuh::lin_point (z, then y, then x):
//   pass B: Y(yy, cx) = lcomb(Z(jy0, cx), Z(jy1, cx), yt(gy)) with
//           Z(jy, cx) = lcomb(c0[jy][cx], c1[jy][cx], zt)   for the 20 window rows
//   pass C: w(yy, xx) += lcomb(Y(yy, jx0), Y(yy, jx1), xt(gx))
// Each thread owns fixed window entries (the (x, y) geometry does not change
// between planes), precomputed once by ProlongGeo::init.
constexpr int NYC = UY * CW;      // pass-B entries (fine window rows x coarse window cols)

template <int NT>
struct ProlongGeo {
  static constexpr int PB_ = (NYC + NT - 1) / NT;
  static constexpr int PC_ = (UX * UY + NT - 1) / NT;
  short b_row[PB_], b_c0[PB_], b_c1[PB_], b_k[PB_];   // Y entry, Z rows (local)
  bool b_two[PB_], b_ok[PB_];
  short c_k[PC_], c_y[PC_], c_x0[PC_], c_x1[PC_];
  bool c_two[PC_], c_ok[PC_];

  __device__ __forceinline__ void init(const Geo& g, int x0, int y0, int cy0, int cx0, int tid) {
#pragma unroll
    for (int q = 0; q < PB_; ++q) {
      const int k = tid + q * NT;
      const int yy = k / CW;
      const int gy = y0 - 2 + yy;
      int j0, j1;
      bool two;
      ltap(gy, j0, j1, two);
      b_k[q] = (short)k;
      b_row[q] = (short)yy;
      b_c0[q] = (short)(j0 - cy0);
      b_c1[q] = (short)(j1 - cy0);
      b_two[q] = two;
      b_ok[q] = k < NYC && gy >= 0 && gy < g.ny;
    }
#pragma unroll
    for (int q = 0; q < PC_; ++q) {
      const int k = tid + q * NT;
      const int yy = k / UX, xx = k - yy * UX;
      const int gx = x0 - 2 + xx, gy = y0 - 2 + yy;
      int j0, j1;
      bool two;
      ltap(gx, j0, j1, two);
      c_k[q] = (short)k;
      c_y[q] = (short)yy;
      c_x0[q] = (short)(j0 - cx0);
      c_x1[q] = (short)(j1 - cx0);
      c_two[q] = two;
      c_ok[q] = k < UX * UY && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny;
    }
  }

  // two passes with a barrier between; the caller syncs after
  __device__ __forceinline__ void apply(double* w, double* ybuf, const double* c0,
                                        const double* c1, bool zt) const {
#pragma unroll
    for (int q = 0; q < PB_; ++q) {
      if (b_k[q] < NYC) {
        double v = 0.0;
        if (b_ok[q]) {
          const int cx = b_k[q] - b_row[q] * CW;
          const int i0 = b_c0[q] * CW + cx, i1 = b_c1[q] * CW + cx;
          const double z0 = lcomb(c0[i0], zt ? c1[i0] : 0.0, zt);
          const double z1 = b_two[q] ? lcomb(c0[i1], zt ? c1[i1] : 0.0, zt) : 0.0;
          v = lcomb(z0, z1, b_two[q]);
        }
        ybuf[b_k[q]] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PC_; ++q) {
      if (c_ok[q]) {
        const double* yr = ybuf + c_y[q] * CW;
        const double v = lcomb(yr[c_x0[q]], c_two[q] ? yr[c_x1[q]] : 0.0, c_two[q]);
        w[c_k[q]] = w[c_k[q]] + v;
      }
    }
  }
};

// ---------------------------------------------------------------------------
// single-stage kernels: apply, residual, one Jacobi sweep (halo-1 window)

template <int OP, bool POW2, int PREF>
__global__ void __launch_bounds__(NTHR) k_z1(const __grid_constant__ CUtensorMap mu,
                                             const __grid_constant__ CUtensorMap mb,
                                             double* __restrict__ out, Geo g, OpC c,
                                             double sigma, double omega, double dval, int zc,
                                             RhsArgs ra) {
  constexpr int HX = TX + 4, HY = TY + 2, P1 = align16(HX * HY), P0 = align16(TX * TY);
  constexpr int RING = PREF + 3;
  constexpr bool NEED_U = OP != Z_JAC0;
  constexpr bool NEED_B = OP != Z_APPLY && OP != Z_APPLY_RHS;
  extern __shared__ __align__(128) double sm[];
  double* su = sm;
  double* sb = sm + (NEED_U ? RING * P1 : 0);
  unsigned long long* bar = (unsigned long long*)(sb + (NEED_B ? RING * P0 : 0));
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int bz = zchunk_block(zc);
  const int z0 = bz * zc, z1 = min(z0 + zc, g.nz);
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
    if (wu) tma3(su + slot * P1, &mu, x0 - 2, y0 - 1, p, bar + slot);
    if (wb) tma3(sb + slot * P0, &mb, x0, y0, p, bar + slot);
  };
  auto wait = [&](int p) {
    const int k = p - z0 + 1;
    mbar_wait(bar + k % RING, (unsigned)((k / RING) & 1));
  };
  if (tid == 0)
    for (int p = z0 - 1; p <= z0 + PREF; ++p) issue(p);
  wait(z0 - 1);
  wait(z0);
  // ---- per-thread constants: two points (rows ty and ty + 8) of column tx.
  // Window indices, validity and the 32-bit element offset of the point on
  // plane z (every field here has fewer than 2^31 elements: checked at launch)
  // are computed once; the plane loop advances them by additions only, the
  // ring slot of plane z+1 and its barrier parity incrementally, and carries
  // the points' own z column (u on planes z-1, z) in registers.
  const int gx = x0 + threadIdx.x;
  const int i0 = (threadIdx.y + 1) * HX + threadIdx.x + 2;
  constexpr int DI = 8 * HX;                          // second point: 8 rows down
  const bool ok0 = gx < g.nx && y0 + (int)threadIdx.y < g.ny;
  const bool ok1 = gx < g.nx && y0 + (int)threadIdx.y + 8 < g.ny;
  unsigned gi = (unsigned)g.at(gx < g.nx ? gx : 0, min(y0 + (int)threadIdx.y, g.ny - 1), z0);
  const unsigned dgi = 8u * (unsigned)g.sy, gsz = (unsigned)g.sz;
  const int ib0 = threadIdx.y * TX + threadIdx.x;     // b window (no halo)
  int sn = 2;                                         // slot of plane z+1 (z = z0: plane z0+1)
  unsigned pn = 0;                                    // its barrier parity
  const double* pm = su;                              // planes z-1, z: slots 0, 1
  const double* pc = su + P1;
  const double* pbc = sb + P0;                        // b of plane z
  double um0 = 0.0, um1 = 0.0, uc0 = 0.0, uc1 = 0.0;
  if constexpr (NEED_U) {
    um0 = pm[i0]; um1 = pm[i0 + DI];
    uc0 = pc[i0]; uc1 = pc[i0 + DI];
  }
  // Z_APPLY_RHS: f_next, s (and tau) of plane z+1 are loaded into registers
  // while plane z computes, so their DRAM latency overlaps a whole plane
  constexpr bool RHS = OP == Z_APPLY_RHS;
  constexpr int NR = RHS ? 2 : 1;
  double cf[NR], cs[NR], ct[NR];
  auto rhs_load = [&](bool live, unsigned o, double* f, double* sv, double* t) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      f[r] = sv[r] = t[r] = 0.0;
      if (live && (r ? ok1 : ok0)) {
        const unsigned q = o + (r ? dgi : 0u);
        f[r] = __ldcs(ra.fn + q);
        sv[r] = __ldcs(ra.s + q);
        if (ra.t0) t[r] = __ldcs(ra.t1 + q) - __ldcs(ra.t0 + q);
      }
    }
  };
  if constexpr (RHS) rhs_load(true, gi, cf, cs, ct);
  // lap7's expression tree with the own column from registers
  auto lap = [&](const double* qc, const double* qp, int i, double m, double c0) {
    double acc = 0.0;
    acc = axis_acc<POW2>(acc, m, c0, qp[i], c);
    acc = axis_acc<POW2>(acc, qc[i - HX], c0, qc[i + HX], c);
    acc = axis_acc<POW2>(acc, qc[i - 1], c0, qc[i + 1], c);
    return c.nu * acc;
  };
  for (int z = z0; z < z1; ++z, gi += gsz) {
    double nf[NR], ns[NR], nt[NR];
    if constexpr (RHS) rhs_load(z + 1 < z1, gi + gsz, nf, ns, nt);
    mbar_wait(bar + sn, pn);
    const double* pp = su + sn * P1;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = i0 + r * DI;
      double& um = r ? um1 : um0;
      double& uc = r ? uc1 : uc0;
      double up = 0.0;
      if constexpr (NEED_U) up = pp[i];
      if (r ? ok1 : ok0) {
        const unsigned q = gi + (r ? dgi : 0u);
        double v;
        if constexpr (OP == Z_APPLY_RHS) {
          // sdc.py:112 f refresh of this node, then sdc.py:102-104 for the next
          double rr = (uc - ra.dtm * cf[r & (NR - 1)]) + cs[r & (NR - 1)];
          if (ra.t0) rr = rr + ct[r & (NR - 1)];
          ra.r[q] = rr;
          v = lap(pc, pp, i, um, uc);
        } else if (OP == Z_JAC0) {
          v = 0.0 + ((omega * pbc[ib0 + r * 8 * TX]) / dval);
        } else {
          const double l = lap(pc, pp, i, um, uc);
          if (OP == Z_APPLY) {
            v = l;
          } else {
            const double au = uc - sigma * l;
            const double bb = pbc[ib0 + r * 8 * TX];
            v = OP == Z_RESID ? bb - au : uc + ((omega * (bb - au)) / dval);
          }
        }
        out[q] = v;
      }
      um = uc;
      uc = up;
    }
    __syncthreads();   // slot of plane z-1 is free
    if (tid == 0) issue(z + PREF + 1);
    pm = pc;
    pc = pp;
    pbc = sb + sn * P0;
    if (++sn == RING) { sn = 0; pn ^= 1u; }
    if constexpr (RHS) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        cf[r] = nf[r];
        cs[r] = ns[r];
        ct[r] = nt[r];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fused two-stage kernels (halo-2 u window, halo-1 b window)
//
// u plane p (z0-2 <= p <= z1+1): slot (p - z0 + 2) % RU
// b plane q (z0-1 <= q <= z1):   slot (q - z0 + 1) % RBB, arrives with u plane q+1
// coarse plane j: slot (j - jlo) % RC, arrives with u plane 2j (and the
//                 first plane z0-2 also brings j = jlo = (z0-2)/2 - 1)

template <int NT, bool PRO, int PREF>
struct Stager {
  static constexpr int RU = PREF + 3, RBB = PREF + 1;
  double *su, *sbb, *se, *ybuf;
  ProlongGeo<NT> pg;
  unsigned long long *bu, *bbar;
  const CUtensorMap *mu, *mb, *me;
  int x0, y0, z0, z1, jlo, cx0, cy0;

  __device__ __forceinline__ void setup(double* sm, const CUtensorMap* mu_,
                                        const CUtensorMap* mb_, const CUtensorMap* me_, int zc,
                                        const Geo& g, int tid) {
    su = sm;
    sbb = su + RU * PU;
    se = sbb + RBB * PB;
    ybuf = se + (PRO ? RC * PC : 0);
    bu = (unsigned long long*)(ybuf + (PRO ? align16(NYC) : 0));
    bbar = bu + RU;
    mu = mu_;
    mb = mb_;
    me = me_;
    x0 = blockIdx.x * TX;
    y0 = blockIdx.y * TY;
    z0 = blockIdx.z * zc;
    z1 = min(z0 + zc, g.nz);
    jlo = (z0 - 2) / 2 - 1;    // z0 is even: exact
    cx0 = x0 / 2 - 2;
    cy0 = y0 / 2 - 2;
    if (PRO) pg.init(g, x0, y0, cy0, cx0, tid);
    if (tid == 0) {
      for (int i = 0; i < RU; ++i) mbar_init(bu + i, 1);
      for (int i = 0; i < RBB; ++i) mbar_init(bbar + i, 1);
      fence_barrier_init();
    }
    __syncthreads();
  }
  __device__ __forceinline__ double* uplane(int p) const { return su + ((p - z0 + 2) % RU) * PU; }
  __device__ __forceinline__ const double* bplane(int q) const {
    return sbb + ((q - z0 + 1) % RBB) * PB;
  }
  __device__ __forceinline__ const double* eplane(int j) const {
    return se + ((j - jlo) % RC) * PC;
  }
  __device__ __forceinline__ void issue(int p, bool zero_u) {   // thread 0 only
    if (p <= z1 + 1) {
      const int k = p - z0 + 2;
      unsigned bytes = zero_u ? 0u : UX * UY * 8u;
      int ne = 0, js[2];
      if (PRO && !zero_u && (p & 1) == 0) {
        if (p == z0 - 2) js[ne++] = jlo;
        js[ne++] = p / 2;
        bytes += ne * CW * CH * 8u;
      }
      if (bytes == 0) {
        mbar_arrive(bu + k % RU);
      } else {
        mbar_expect(bu + k % RU, bytes);
        if (!zero_u) tma3(su + (k % RU) * PU, mu, x0 - 2, y0 - 2, p, bu + k % RU);
        for (int e = 0; e < ne; ++e)
          tma3(se + ((js[e] - jlo) % RC) * PC, me, cx0, cy0, js[e], bu + k % RU);
      }
    }
    const int q = p - 1;
    if (q >= z0 - 1 && q <= z1) {
      const int k = q - z0 + 1;
      mbar_expect(bbar + k % RBB, BW * BH * 8u);
      tma3(sbb + (k % RBB) * PB, mb, x0 - 2, y0 - 1, q, bbar + k % RBB);
    }
  }
  __device__ __forceinline__ void wait_u(int p) const {
    const int k = p - z0 + 2;
    mbar_wait(bu + k % RU, (unsigned)((k / RU) & 1));
  }
  __device__ __forceinline__ void wait_b(int q) const {
    const int k = q - z0 + 1;
    mbar_wait(bbar + k % RBB, (unsigned)((k / RBB) & 1));
  }
  // prolongation of staged u plane p (after wait_u(p), before any use)
  // prolongation of staged u plane p (after wait_u(p), before any use); all
  // threads, contains a barrier -- the plane is usable after the next one
  __device__ __forceinline__ void prolong(int p, const Geo& g) {
    if (!PRO || p < 0 || p >= g.nz) return;
    int jz0, jz1;
    bool zt;
    ltap(p, jz0, jz1, zt);
    pg.apply(uplane(p), ybuf, eplane(jz0), eplane(jz1), zt);
  }
  __host__ __device__ static constexpr size_t smem_doubles() {
    return (size_t)RU * PU + RBB * PB + (PRO ? RC * PC + align16(NYC) : 0);
  }
  __host__ __device__ static constexpr size_t smem_bytes() { return smem_doubles() * 8 + 8 * (RU + RBB); }
};

// two fused Jacobi sweeps (optionally after the prolongation)
template <bool POW2, bool PRO, int PREF>
__global__ void __launch_bounds__(NTHR) k_z2(const __grid_constant__ CUtensorMap mu,
                                             const __grid_constant__ CUtensorMap mb,
                                             const __grid_constant__ CUtensorMap me,
                                             double* __restrict__ out, Geo g, OpC c,
                                             double sigma, double omega, double dval, int zc,
                                             int zero_in) {
  constexpr int HX = TX + 2, HY = TY + 2, PH = align16(HX * HY), NH = HX * HY;
  using S = Stager<NTHR, PRO, PREF>;
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  S st;
  st.setup(sm, &mu, &mb, &me, zc, g, tid);
  double* s1 = sm + S::smem_doubles() + 16;     // after the (<= 16) barriers
  const int x0 = st.x0, y0 = st.y0, z0 = st.z0, z1 = st.z1;

  constexpr int PER1 = (NH + NTHR - 1) / NTHR;
  int e_k[PER1], e_i[PER1], e_b[PER1];
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
  }
  // sweep 1 at plane zz over the halo-1 window (0 outside the domain)
  auto stage1 = [&](int zz) {
    double* dst = s1 + ((zz - z0 + 3) % 3) * PH;
    const bool zin = zz >= 0 && zz < g.nz;
    const double* pm = st.uplane(zz - 1);
    const double* pc = st.uplane(zz);
    const double* pp = st.uplane(zz + 1);
    const double* pb = st.bplane(zz);
#pragma unroll
    for (int q = 0; q < PER1; ++q) {
      const int k = e_k[q];
      if (k < NH) {
        double v = 0.0;
        if (zin && e_in[q]) {
          const int i = e_i[q];
          const double b = pb[e_b[q]];
          if (zero_in) {
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
    for (int p = z0 - 2; p <= z0 + PREF; ++p) st.issue(p, zero_in);
  for (int p = z0 - 2; p <= z0 + 1; ++p) {
    st.wait_u(p);
    __syncthreads();
    st.prolong(p, g);
  }
  st.wait_b(z0 - 1);
  st.wait_b(z0);
  __syncthreads();
  stage1(z0 - 1);
  stage1(z0);
  const int gx = x0 + threadIdx.x;
  for (int z = z0; z < z1; ++z) {
    st.wait_u(z + 2);
    st.wait_b(z + 1);
    if (PRO) {
      st.prolong(z + 2, g);
      __syncthreads();
    }
    stage1(z + 1);
    __syncthreads();
    const double* qm = s1 + ((z - 1 - z0 + 3) % 3) * PH;
    const double* qc = s1 + ((z - z0 + 3) % 3) * PH;
    const double* qp = s1 + ((z + 1 - z0 + 3) % 3) * PH;
    const double* pb = st.bplane(z);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int ly = threadIdx.y + 8 * r;
      const int gy = y0 + ly;
      if (gx < g.nx && gy < g.ny) {
        const int i = (ly + 1) * HX + threadIdx.x + 1;
        const int ib = (ly + 1) * BW + threadIdx.x + 2;
        double au = qc[i] - sigma * lap7<POW2, HX>(qm, qc, qp, i, c);
        out[g.at(gx, gy, z)] = qc[i] + ((omega * (pb[ib] - au)) / dval);
      }
    }
    __syncthreads();   // u plane z-1, b plane z and stage-1 plane z-1 are free
    if (tid == 0) st.issue(z + PREF + 1, zero_in);
  }
}

// ---------------------------------------------------------------------------
// helpers of the fused red-black sweep (k_zrb3)

constexpr int NTHR_RB2 = 256;


__device__ __forceinline__ double2 lds2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
// shared-window (32-bit) addressing for the sweep's plane loop: address
// arithmetic stays one integer add and the offsets fold into the instruction
template <int OFF>
__device__ __forceinline__ double sld1(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ double2 sld2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v.x), "=d"(v.y) : "r"(a), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ void sst1(unsigned a, double v) {
  asm volatile("st.shared.f64 [%0+%1], %2;" ::"r"(a), "n"(OFF), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// k_zrb3: one fused jor-rb sweep (multigrid.py:225-233) with one CTA barrier
// per TWO planes.  Phase z updates the red points of plane z+2 and the black
// points of plane z: a red point reads only black neighbours (old values) and
// its own centre, a black point reads the red points of planes z-1..z+1,
// final since phases z-3..z-1 -- the two sets touch disjoint data, and a red
// value written in phase z is first read by another thread in phase z+2.
// Thread (row, px) owns the point pair (x0+2px, x0+2px+1) of its row on every
// plane and carries that pair for planes z-1..z+2 (plus the plane it loads)
// and the black member of b for z, z+1 in registers, so the centre and
// z-neighbours come from registers and only x/y neighbours are shared-memory
// loads; the 50 red points of the tile's halo ring are updated by threads
// 0..49.  Warp w owns tile rows 4(w/2) + (w&1) and that + 2, so (y + z) has
// one parity per warp and plane: the phase code is instantiated per parity
// (no selects) and the plane loop is unrolled by four, which rotates the four
// register pairs and the four ring offsets by name.  u plane p is read from
// shared memory in phases p-3 .. p, b plane q in phase q-2 only.  The
// division by the constant diagonal is the correctly rounded Markstein
// quotient (div_const's); everything else is the reference's expression tree,
// so the sweep is bit-identical to the one-colour kernels.

// Ring slots carry their own mbarrier: slot s of the u ring is the USL doubles
// at su + s * USL, the window first and the barrier word at element PU, so a
// slot offset is all a phase needs (no slot index, no modulo).  The b ring
// (half as many slots, same stride) follows the u ring.
constexpr int USL = PU + 16;              // slot stride (a multiple of 128 bytes)
static_assert(BW == UX && PB <= PU, "the b window shares the u window's row pitch and slot");

struct RbCtx {
  double* su;
  double* sb;
  int z0, R;
  int iu, ib;           // own pair (first member) in the u / b windows
  bool va, vb;          // pair members in the domain
  double* optr;         // global address of the pair on plane 0
  long long sz;
  int hu0, hu1;         // halo red point per plane parity (b: the same - UX)
  bool hv0, hv1;
  OpC c;
  double sigma, omega, dval, dinv;
};

template <int RU>
__device__ __forceinline__ double* rb_u(const RbCtx& k, int p) {
  return k.su + ((unsigned)(p - k.z0 + 2) % RU) * USL;
}
template <int RB>
__device__ __forceinline__ double* rb_b(const RbCtx& k, int q) {
  return k.sb + ((unsigned)(q - k.z0 + 3) % RB) * USL;   // the slot of u plane q+1, mod RB
}
template <int O>
__device__ __forceinline__ double mem(const double2& v) { return O ? v.y : v.x; }
template <int O>
__device__ __forceinline__ void set_mem(double2& v, double x) {
  if (O) v.y = x; else v.x = x;
}
template <bool POW2>
__device__ __forceinline__ double rb_relax(const RbCtx& k, double zm, double zp, double ym,
                                           double yp, double xm, double xp, double cc,
                                           double bv) {
  double acc = 0.0;
  acc = axis_acc<POW2>(acc, zm, cc, zp, k.c);
  acc = axis_acc<POW2>(acc, ym, cc, yp, k.c);
  acc = axis_acc<POW2>(acc, xm, cc, xp, k.c);
  const double lp = k.c.nu * acc;
  const double r = bv - (cc - k.sigma * lp);
  return cc + div_const(k.omega * r, k.dval, k.dinv);
}

// branch-free part of a relaxation: a = omega * r and the Markstein quotient
// (valid when in_range(a)); the caller finishes with cc + quotient
struct Relax {
  double cc, a, q;
};
// UNIT: nu = omega = 1, whose multiplications are exact and skipped
template <bool POW2, bool UNIT = false>
__device__ __forceinline__ Relax rb_fast(const RbCtx& k, double zm, double zp, double ym,
                                         double yp, double xm, double xp, double cc, double bv) {
  double acc = 0.0;
  acc = axis_acc<POW2>(acc, zm, cc, zp, k.c);
  acc = axis_acc<POW2>(acc, ym, cc, yp, k.c);
  acc = axis_acc<POW2>(acc, xm, cc, xp, k.c);
  const double lp = UNIT ? acc : k.c.nu * acc;
  const double r = bv - (cc - k.sigma * lp);
  Relax o;
  o.cc = cc;
  o.a = UNIT ? r : k.omega * r;
  double q = o.a * k.dinv;
  double e = __fma_rn(-k.dval, q, o.a);
  q = __fma_rn(e, k.dinv, q);
  e = __fma_rn(-k.dval, q, o.a);
  o.q = __fma_rn(e, k.dinv, q);
  return o;
}
// 2^-960 <= |a| < 2^960 from the biased exponent (integer pipe; both paths
// are correctly rounded, so the exact cut only picks the method)
__device__ __forceinline__ bool quot_ok(double a) {
  const unsigned e = ((unsigned)__double2hiint(a) >> 20) & 0x7ffu;
  return e - 63u <= 1919u;
}

// update member O of the own pair on plane q (pl); um/uc/up = own pair on
// planes q-1, q, q+1 (uc updated), bq = b pair on q.  Returns the new value.
template <bool POW2, int O>
__device__ __forceinline__ double rb_point(const RbCtx& k, const double* pl, const double2& um,
                                           const double2& uc, const double2& up,
                                           const double2& bq) {
  const double xm = O ? uc.x : pl[k.iu - 1];
  const double xp = O ? pl[k.iu + 2] : uc.y;
  return rb_relax<POW2>(k, mem<O>(um), mem<O>(up), pl[k.iu - UX + O], pl[k.iu + UX + O], xm, xp,
                        mem<O>(uc), mem<O>(bq));
}
// the same from the thread's own pair address `own` on that plane, with the z
// neighbours and b as scalars; branch-free part only
template <bool POW2, int O, bool UNIT>
__device__ __forceinline__ Relax rb_own(const RbCtx& k, const double* own, double zm, double zp,
                                        const double2& uc, double bq) {
  const double xm = O ? uc.x : own[-1];
  const double xp = O ? own[2] : uc.y;
  return rb_fast<POW2, UNIT>(k, zm, zp, own[-UX + O], own[UX + O], xm, xp, mem<O>(uc), bq);
}

// halo red point (threads < 50) on plane q of parity P, shared memory only
template <bool POW2, int RU, int RB, int P>
__device__ __forceinline__ void rb_halo(const RbCtx& k, int q) {
  const bool hv = P ? k.hv1 : k.hv0;
  if (!hv || q > k.R || q < 0) return;
  const int i = P ? k.hu1 : k.hu0;
  double* pl = rb_u<RU>(k, q);
  const double* pm = rb_u<RU>(k, q - 1);
  const double* pp = rb_u<RU>(k, q + 1);
  pl[i] = rb_relax<POW2>(k, pm[i], pp[i], pl[i - UX], pl[i + UX], pl[i - 1], pl[i + 1], pl[i],
                         rb_b<RB>(k, q)[i - UX]);
}

// both quotient numerators in [2^-960, 2^960): one unsigned compare of the
// shifted high words (sign dropped, biased exponent 63 .. 1982)
__device__ __forceinline__ bool quots_ok(double a, double b) {
  const unsigned ha = ((unsigned)__double2hiint(a) << 1) - (63u << 21);
  const unsigned hb = ((unsigned)__double2hiint(b) << 1) - (63u << 21);
  return max(ha, hb) <= ((1919u << 21) | 0x1fffffu);
}
template <bool POW2, int RU, int RB, int MINB, bool UNIT>
__global__ void __launch_bounds__(NTHR_RB2, MINB) k_zrb3(const __grid_constant__ CUtensorMap mu,
                                                      const __grid_constant__ CUtensorMap mb,
                                                      double* __restrict__ out, Geo g, OpC c,
                                                      double sigma, double omega, double dval,
                                                      double dinv, int zc) {
  static_assert(RU >= 6 && RU == 2 * RB, "rings");
  extern __shared__ __align__(128) double sm[];
  RbCtx k;
  k.su = sm;
  k.sb = sm + RU * USL;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, g.nz);
  k.z0 = z0;
  k.R = min(z1, g.nz - 1);
  const int uhi = k.R + 1, bhi = k.R;
  k.c = c;
  k.sigma = sigma;
  k.omega = omega;
  k.dval = dval;
  k.dinv = dinv;
  // b plane q rides with u plane q+1: it sits in the b slot "u slot of plane
  // q+1, mod RB" and completes on that u slot's barrier, which is armed for the
  // bytes of both copies -- one wait per phase covers the two planes it needs
  auto ubar = [&](int s) { return (unsigned long long*)(k.su + s * USL + PU); };
  if (tid == 0) {
    for (int i = 0; i < RU; ++i) mbar_init(ubar(i), 1);
    fence_barrier_init();
  }
  __syncthreads();
  // TMA copy of u plane p / b plane q into the slot at element offset o
  // TMA copy of u plane p into the slot at element offset o; its barrier also
  // expects b plane p-1 when that plane exists (p >= z0; p <= uhi <=> p-1 <= bhi)
  auto load_u = [&](int p, int o) {
    if (p > uhi) return;
    unsigned long long* bar = (unsigned long long*)(k.su + o + PU);
    mbar_expect(bar, UX * UY * 8u + (p >= z0 ? BW * BH * 8u : 0u));
    tma3(k.su + o, &mu, x0 - 2, y0 - 2, p, bar);
  };
  // TMA copy of b plane q into the b slot of the u slot at element offset o
  // (the slot of u plane q+1), completing on that u slot's barrier
  auto load_b = [&](int q, int o) {
    if (q > bhi) return;
    unsigned long long* bar = (unsigned long long*)(k.su + o + PU);
    tma3(k.sb + (o >= RB * USL ? o - RB * USL : o), &mb, x0 - 2, y0 - 1, q, bar);
  };
  auto issue_u = [&](int p) { load_u(p, (int)((unsigned)(p - z0 + 2) % RU) * USL); };
  auto issue_b = [&](int q) { load_b(q, (int)((unsigned)(q - z0 + 3) % RU) * USL); };
  auto wait_u = [&](int p) {      // u plane p and b plane p-1
    const int i = p - z0 + 2;
    mbar_wait(ubar((unsigned)i % RU), ((unsigned)i / RU) & 1u);
  };
  if (tid == 0) {
    for (int p = z0 - 2; p < z0 - 2 + RU; ++p) issue_u(p);
    for (int q = z0 - 1; q < z0 - 1 + RB; ++q) issue_b(q);
  }
  // rows 4(w/2) + (w&1) (lanes 0-15) and +2 (lanes 16-31): one parity per warp
  const int row = 4 * (warp >> 1) + (warp & 1) + 2 * (lane >> 4), px = lane & 15;
  const int gy = y0 + row, gxa = x0 + 2 * px;
  k.va = gy < g.ny && gxa < g.nx;
  k.vb = gy < g.ny && gxa + 1 < g.nx;
  k.iu = (row + 2) * UX + 2 * px + 2;
  k.ib = (row + 1) * BW + 2 * px + 2;
  k.optr = out + (long long)gy * g.sy + gxa;
  k.sz = g.sz;
  // halo red ids: threads 0..49
  const int hid = tid;
  const bool is_halo = hid < 50;
  {
    int hu[2];
    bool hv[2];
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      int xx, yy;
      if (hid < 17) { yy = -1; xx = -1 + 2 * hid + (1 - P); }
      else if (hid < 34) { yy = TY; xx = -1 + 2 * (hid - 17) + P; }
      else if (hid < 42) { xx = -1; yy = 2 * (hid - 34) + P; }
      else { xx = TX; yy = 2 * (hid - 42) + (1 - P); }
      hu[P] = (yy + 2) * UX + xx + 2;
      hv[P] = hid >= 0 && hid < 50 && x0 + xx >= 0 && x0 + xx < g.nx && y0 + yy >= 0 &&
              y0 + yy < g.ny;
    }
    k.hu0 = hu[0]; k.hu1 = hu[1];
    k.hv0 = hv[0]; k.hv1 = hv[1];
  }
  const int wpar = (y0 + row) & 1;   // = warp & 1 (y0 even)

  // ---- prologue: reds of planes z0-1 (if >= 0), z0, z0+1 (if <= R)
  for (int p = z0 - 2; p <= min(z0 + 2, uhi); ++p) wait_u(p);
  const double2 zero2 = make_double2(0.0, 0.0);
  double2 Um2 = lds2(rb_u<RU>(k, z0 - 2) + k.iu);
  double2 W0 = lds2(rb_u<RU>(k, z0 - 1) + k.iu);
  double2 W1 = lds2(rb_u<RU>(k, z0) + k.iu);
  double2 W2 = lds2(rb_u<RU>(k, z0 + 1) + k.iu);
  double2 W3 = z0 + 2 <= uhi ? lds2(rb_u<RU>(k, z0 + 2) + k.iu) : zero2;
  const double2 Bm1 = lds2(rb_b<RB>(k, z0 - 1) + k.ib);
  const double2 B0 = lds2(rb_b<RB>(k, z0) + k.ib);
  // plane p red member: 1 - ((y + p) & 1); z0 even, so plane z0 has parity wpar
  auto pro_red = [&](int q, const double2& um, double2& uc, const double2& up,
                     const double2& bq, int par) {
    if (q < 0 || q > k.R) return;
    double* pl = rb_u<RU>(k, q);
    if (par) {
      const double v = c.pow2 ? rb_point<true, 0>(k, pl, um, uc, up, bq)
                              : rb_point<false, 0>(k, pl, um, uc, up, bq);
      if (k.va) { pl[k.iu] = v; uc.x = v; }
    } else {
      const double v = c.pow2 ? rb_point<true, 1>(k, pl, um, uc, up, bq)
                              : rb_point<false, 1>(k, pl, um, uc, up, bq);
      if (k.vb) { pl[k.iu + 1] = v; uc.y = v; }
    }
  };
  pro_red(z0 - 1, Um2, W0, W1, Bm1, 1 - wpar);
  pro_red(z0, W0, W1, W2, B0, wpar);
  if (is_halo) {
    rb_halo<POW2, RU, RB, 1>(k, z0 - 1);
    rb_halo<POW2, RU, RB, 0>(k, z0);
  }
  const double2 B1 = z0 + 1 <= bhi ? lds2(rb_b<RB>(k, z0 + 1) + k.ib) : zero2;
  pro_red(z0 + 1, W1, W2, W3, B1, 1 - wpar);
  if (is_halo) rb_halo<POW2, RU, RB, 1>(k, z0 + 1);
  __syncthreads();
  if (tid == 0) {       // u planes z0-2, z0-1 and b planes z0-1 .. z0+1 are dead
    issue_u(z0 - 2 + RU);
    issue_u(z0 - 1 + RU);
    for (int q = z0 - 1; q <= z0 + 1; ++q) issue_b(q + RB);
  }

  // ---- main loop, four planes per trip.  In phase z the registers A, B, C, D
  // hold the own pair on planes z-1 .. z+2 and plane z+3 is loaded over A once
  // A's last use is done; four phases rotate the four names back, so no
  // register moves.  The ring offsets (bytes) of planes z .. z+3 rotate the
  // same way (advanced by one slot with a compare for the wrap); b plane z+2
  // sits in the b slot "u slot of z+3, mod RB", whose barrier parity is which
  // half of the u ring that slot is in.  The b plane's black member waits two
  // phases in ba / bb.
  constexpr int SB = USL * 8;                          // slot stride in bytes
  constexpr int HB = (RU * USL - UX) * 8;              // u-ring point -> same point of the b ring
  const unsigned smb = saddr(sm);
  const unsigned tub = smb + k.iu * 8;                 // own pair in slot 0 of the u ring
  // halo point per plane parity
  const unsigned hb0 = smb + k.hu0 * 8, hb1 = smb + k.hu1 * 8;
  // bit 0: a thread that issues copies -- the first lanes of warps 4..7 (no
  // halo points there), one of the four copies of a refill each (bits 3-4), so
  // the copies start in parallel right after the barrier (88.3 vs 89.5 us at
  // 255^3, 22.7 vs 23.7 at 127^3); bit 1 / 2: halo thread with a point on even
  // / odd planes
  const int flags = ((tid & 31) == 0 && tid >= NTHR_RB2 / 2 ? 1 | ((tid - NTHR_RB2 / 2) >> 5) << 3
                                                            : 0) |
                    (is_halo && k.hv0 ? 2 : 0) | (is_halo && k.hv1 ? 4 : 0);
  auto run = [&](auto par_tag) {
    constexpr int PA = decltype(par_tag)::value, PB_ = 1 - PA;
    int o0 = 2 * SB, o1 = 3 * SB, o2 = 4 * SB, o3 = 5 * SB;   // planes z0 .. z0+3
    unsigned pu = 0;                               // mbarrier parity of plane z+3's copy
    double* dst = k.optr + (long long)z0 * k.sz;   // own pair on plane z
    double ba = mem<PA>(B0), bb = mem<PB_>(B1);    // black members of b on z, z+1
    // one phase: red of plane z+2 (if <= R), black of plane z.  PAR = (y + z) & 1
    // of this warp's rows: red member 1 - PAR, black member PAR.  Both updates
    // are evaluated branch-free (independent chains the scheduler interleaves);
    // one warp-wide test sends out-of-range quotients to the IEEE division.
    //
    // SYNC: the phase ends with the CTA barrier and the refill of the slots the
    // last two phases freed.  Reds written in phase z are first read by other
    // threads in phase z+2, so one barrier per two phases orders every
    // shared-memory dependence.
    auto next_u = [](int o) { return o == (RU - 1) * SB ? 0 : o + SB; };
    auto phase = [&](auto ptag, auto sync_tag, int z, double2& A, double2& B, const double2& C,
                     double2& D, double& bk, int& oa, int o_b, int o_c, int o_d) {
      constexpr int PAR = decltype(ptag)::value;
      constexpr bool SYNC = decltype(sync_tag)::value;
      constexpr int ZP = PAR ^ PA;                   // parity of plane z (z0 is even)
      const int q = z + 2;
      const bool hi = o_d >= RB * SB;                // b slot round = half of the u ring
      const int ob = (hi ? o_d - RB * SB : o_d);     // b plane z+2's slot
      if (q <= k.R) mbar_wait_s(smb + o_d + PU * 8, pu);
      const double2 N = sld2<0>(tub + o_d);          // plane z+3 (stale beyond R: unused)
      const double2 B2 = sld2<HB>(tub + ob);         // b on plane z+2
      const unsigned ar = tub + o_c, ak = tub + oa;  // own pair on planes z+2, z
      Relax rr, rk;
      {
        constexpr int O = 1 - PAR;
        const double xm = O ? D.x : sld1<-8>(ar);
        const double xp = O ? sld1<16>(ar) : D.y;
        rr = rb_fast<POW2, UNIT>(k, mem<O>(C), mem<O>(N), sld1<(O - UX) * 8>(ar),
                                 sld1<(O + UX) * 8>(ar), xm, xp, mem<O>(D), mem<O>(B2));
      }
      {
        constexpr int O = PAR;
        const double xm = O ? B.x : sld1<-8>(ak);
        const double xp = O ? sld1<16>(ak) : B.y;
        rk = rb_fast<POW2, UNIT>(k, mem<O>(A), mem<O>(C), sld1<(O - UX) * 8>(ak),
                                 sld1<(O + UX) * 8>(ak), xm, xp, mem<O>(B), bk);
      }
      if (__builtin_expect(!quots_ok(rr.a, rk.a), 0)) {
        if (!quot_ok(rr.a)) rr.q = div_slow(rr.a, k.dval);
        if (!quot_ok(rk.a)) rk.q = div_slow(rk.a, k.dval);
      }
      const double vr = rr.cc + rr.q, vk = rk.cc + rk.q;
      if (q <= k.R && (PAR ? k.va : k.vb)) {
        sst1<(1 - PAR) * 8>(ar, vr);
        set_mem<1 - PAR>(D, vr);
      }
      set_mem<PAR>(B, vk);
      if (k.vb) *reinterpret_cast<double2*>(dst) = B;   // vb implies va
      else if (k.va) dst[0] = B.x;
      dst += k.sz;
      A = N;
      bk = mem<PAR>(B2);
      if ((flags & (ZP ? 4 : 2)) && q <= k.R) {      // halo reds of plane z+2
        const unsigned h = ZP ? hb1 : hb0;
        const unsigned hc = h + o_c;
        const double cc = sld1<0>(hc);
        sst1<0>(hc, rb_relax<POW2>(k, sld1<0>(h + o_b), sld1<0>(h + o_d), sld1<-UX * 8>(hc),
                                   sld1<UX * 8>(hc), sld1<-8>(hc), sld1<8>(hc), cc,
                                   sld1<HB>(h + ob)));
      }
      // plane z+4 takes the slot after plane z+3's
      const bool wu = o_d == (RU - 1) * SB;
      oa = wu ? 0 : o_d + SB;
      pu ^= wu ? 1u : 0u;
      if (SYNC) {
        __syncthreads();
        if (flags & 1) {
          // u planes z-1, z and b planes z+1, z+2 are dead.  oa is the slot
          // of u plane z+4; plane z-1+RU follows it RU-5 slots on.  b plane
          // q sits in the b slot "u slot of q+1, mod RB".
          int u1 = oa, t = oa;
#pragma unroll
          for (int i = 0; i < RU - 5; ++i) u1 = next_u(u1);
#pragma unroll
          for (int i = 0; i < RB - 2; ++i) t = next_u(t);   // u plane z+2+RB
          const int role = (flags >> 3) & 3;
          if (role == 0) load_u(z - 1 + RU, u1 >> 3);
          else if (role == 1) load_b(z + 1 + RB, t >> 3);
          else if (role == 2) load_u(z + RU, next_u(u1) >> 3);
          else load_b(z + 2 + RB, next_u(t) >> 3);
        }
      }
    };
    using TA = std::integral_constant<int, PA>;
    using TB = std::integral_constant<int, PB_>;
    using S0 = std::false_type;
    using S1 = std::true_type;
    for (int z = z0;; z += 4) {
      phase(TA{}, S0{}, z, W0, W1, W2, W3, ba, o0, o1, o2, o3);
      if (z + 1 >= z1) break;
      phase(TB{}, S1{}, z + 1, W1, W2, W3, W0, bb, o1, o2, o3, o0);
      if (z + 2 >= z1) break;
      phase(TA{}, S0{}, z + 2, W2, W3, W0, W1, ba, o2, o3, o0, o1);
      if (z + 3 >= z1) break;
      phase(TB{}, S1{}, z + 3, W3, W0, W1, W2, bb, o3, o0, o1, o2);
      if (z + 4 >= z1) break;
    }
  };
  if (wpar) run(std::integral_constant<int, 1>{});
  else run(std::integral_constant<int, 0>{});
}

// ---------------------------------------------------------------------------
// fine (+)= P_cubic coarse for 3-D (transfers.py:82-89).  The coarse planes a
// fine plane needs arrive by TMA (20 x 12 windows); per fine plane three
// separable passes in shared memory -- z taps over the coarse window, y taps
// onto the tile rows, x taps onto the tile -- each a sequential FMA chain in
// increasing tap order, exactly the per-axis dgemm order of the reference.

constexpr int QW = TX / 2 + 4, QH = TY / 2 + 4, PQ = align16(QW * QH);   // coarse window

// k_rfw: coarse b = FW(b - (I - sigma A) u) in one pass (multigrid.py:245-246;
// transfers.py:27-34).  A CTA owns a 16 x 8 coarse tile and marches up the
// fine planes of its z chunk; each fine residual of the 33 x 17 window (fine
// x0..x0+32, y0..y0+16) is evaluated from TMA-staged u (halo 1) and b windows
// and folded into the z weights in registers in fw3's operation order
// (0.25 * ((a + 2 b) + c): a at plane 2jz, t = a + 2 b at 2jz+1,
// 0.25 * (t + c) at 2jz+2, which is also the next coarse plane's a).  The
// z-weighted plane goes to shared memory; its y pass runs in the next phase
// and the x pass in the one after -- one barrier per fine plane, and the fine
// residual is never stored.  Nine warps: warp w owns residual rows w and w+9
// of x0..x0+31, warp 8 also the column x0+32, so each thread evaluates at
// most two residuals per plane and a warp's loads are 32 consecutive doubles.
// The plane loop is unrolled by two (odd and even planes of the chunk carry
// different z weights and passes), the u / b ring slots and their mbarrier
// phases advance incrementally, and every per-thread index is precomputed:
// the integer work per plane is a few adds.  ν = 1 has its own instantiation.
// Residual arithmetic is k_z1<Z_RESID>'s and the weights fw_point's: the
// coarse right-hand side is bit-identical to residual + full_weighting.
constexpr int RX = TX + 1, RY = TY + 1, PR = align16(RX * RY);     // residual window
constexpr int FUX = TX + 4, FUY = TY + 3, PFU = align16(FUX * FUY);  // u window
constexpr int FBX = TX + 2, FBY = TY + 1, PFB = align16(FBX * FBY);  // b window
constexpr int RFW_RU = 5, RFW_RB = 3, RFW_NT = 288;
constexpr int RFW_SMEM = sizeof(double) * (RFW_RU * PFU + RFW_RB * PFB + 2 * PR) + 8 * RFW_RU;

template <bool POW2, bool UNIT>
__global__ void __launch_bounds__(RFW_NT, 4) k_rfw(const __grid_constant__ CUtensorMap mu,
                                                    const __grid_constant__ CUtensorMap mb,
                                                    double* __restrict__ coarse, Geo gf, Geo gc,
                                                    OpC c, double sigma, int zcc) {
  extern __shared__ __align__(128) double sm[];
  double* su = sm;                            // RFW_RU u windows
  double* sb = su + RFW_RU * PFU;             // RFW_RB b windows
  double* szb = sb + RFW_RB * PFB;            // z-weighted plane (RX x RY)
  double* syx = szb + PR;                     // y-weighted rows (RX x TY/2)
  unsigned long long* bu = (unsigned long long*)(syx + PR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int rfw_issuer = RFW_NT - 32;     // warp 8: fewest residual points, no x pass
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int bz = zchunk_block(zcc);
  const int jz0 = bz * zcc, jz1 = min(jz0 + zcc, gc.nz);
  const int p0 = 2 * jz0, p1 = 2 * jz1;       // residual planes p0 .. p1
  const int ulo = p0 - 1, uhi = p1 + 1;       // u planes
  if (tid == 0) {
    for (int i = 0; i < RFW_RU; ++i) mbar_init(bu + i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  // b plane p is needed in the same phase as u plane p+1 and completes on
  // that u slot's barrier, armed for the bytes of both copies: one wait per
  // plane.  (Only the issuing thread computes slots by modulo.)
  auto issue_u = [&](int p) {
    if (p > uhi) return;
    const int s = (p - ulo) % RFW_RU;
    mbar_expect(bu + s, FUX * FUY * 8u + (p > p0 ? FBX * FBY * 8u : 0u));
    tma3(su + s * PFU, &mu, x0 - 2, y0 - 1, p, bu + s);
  };
  auto issue_b = [&](int p) {
    if (p > p1) return;
    const int s = (p - p0) % RFW_RB;
    tma3(sb + s * PFB, &mb, x0, y0, p, bu + (p + 1 - ulo) % RFW_RU);
  };
  if (tid == 0) {
    for (int p = ulo; p < ulo + RFW_RU; ++p) issue_u(p);
    for (int p = p0; p < p0 + RFW_RB; ++p) issue_b(p);
  }
  // ---- owned residual points (q = 0: row w; q = 1: row w + 9, or for warp 8
  // the column x0 + 32 of rows 0..16)
  int r_iu[2], r_ib[2], r_k[2];
  bool r_ok[2], r_on[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = q == 0 ? warp * RX + lane
                         : (warp < 8 ? (warp + 9) * RX + lane : (lane < RY ? lane * RX + TX : 0));
    const int ry = k / RX, rx = k - ry * RX;
    r_on[q] = q == 0 || warp < 8 || lane < RY;
    r_k[q] = k;
    r_iu[q] = (ry + 1) * FUX + rx + 2;
    r_ib[q] = ry * FBX + rx;
    r_ok[q] = r_on[q] && x0 + rx < gf.nx && y0 + ry < gf.ny;
  }
  double acc[2], cm_[2], cc_[2];             // z fold; u of the own column at p-1, p
  // ---- y pass entry (threads < RX * TY/2): syx[yy][xx] from szb rows 2yy..2yy+2
  const bool ytask = tid < RX * (TY / 2);
  const int yy = tid / RX, xx = tid - (tid / RX) * RX;
  const int yo = ytask ? 2 * yy * RX + xx : 0, yd = ytask ? tid : 0;
  // ---- x pass entry (threads < 128): coarse point (cx, cy) of the tile
  const int cx = tid & 15, cy = tid >> 4;
  const int gcx = x0 / 2 + cx, gcy = y0 / 2 + cy;
  const bool c_ok = tid < (TX / 2) * (TY / 2) && gcx < gc.nx && gcy < gc.ny;
  const int xo = cy * RX + 2 * cx;
  double* cdst = coarse + (c_ok ? gc.at(gcx, gcy, jz0) : 0);
  // ---- u / b ring position of plane p+1 (u) and p (b), advanced per plane
  int us = 2, up_ = 0;          // slot and phase bit of u plane p+1 (= ulo + 2 at p = p0)
  int bs = 0;                   // slot of b plane p
  const double* pm = su;        // u planes p-1, p (slots 0, 1 at p = p0)
  const double* pc = su + PFU;
  // residual of plane p folded into the weights; FIRST: the chunk's first
  // plane (a := v), ODD: t = a + 2 v, else 0.25 (t + v) -> szb, a := v
  auto resid = [&](auto mode_tag, int p) {
    constexpr int MODE = decltype(mode_tag)::value;   // 0 first, 1 odd, 2 even
    mbar_wait(bu + us, (unsigned)up_);   // u plane p+1 and b plane p
    const double* pp = su + us * PFU;
    const double* pb = sb + bs * PFB;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!r_on[q]) continue;
      const int i = r_iu[q];
      if (MODE == 0) {
        cm_[q] = pm[i];
        cc_[q] = pc[i];
      }
      const double zcp = pp[i];
      double v = 0.0;
      if (r_ok[q]) {
        // lap7's expression tree with the column's centre values in registers
        const double c0 = cc_[q];
        double lacc = 0.0;
        lacc = axis_acc<POW2>(lacc, cm_[q], c0, zcp, c);
        lacc = axis_acc<POW2>(lacc, pc[i - FUX], c0, pc[i + FUX], c);
        lacc = axis_acc<POW2>(lacc, pc[i - 1], c0, pc[i + 1], c);
        const double lap = UNIT ? lacc : c.nu * lacc;
        const double au = c0 - sigma * lap;
        v = pb[r_ib[q]] - au;
      }
      cm_[q] = cc_[q];
      cc_[q] = zcp;
      if (MODE == 0) {
        acc[q] = v;
      } else if (MODE == 1) {
        acc[q] = acc[q] + 2.0 * v;
      } else {
        szb[r_k[q]] = 0.25 * (acc[q] + v);
        acc[q] = v;
      }
    }
    pm = pc;
    pc = pp;
    if (++us == RFW_RU) { us = 0; up_ ^= 1; }
    if (++bs == RFW_RB) bs = 0;
  };
  auto ypass = [&]() {
    if (ytask) syx[yd] = fw3(szb[yo], szb[yo + RX], szb[yo + 2 * RX]);
  };
  auto xpass = [&]() {
    if (c_ok) {
      *cdst = fw3(syx[xo], syx[xo + 1], syx[xo + 2]);
      cdst += gc.sz;
    }
  };
  auto after = [&](int p) {    // plane p's residuals done: u plane p-1 and b plane p are free
    __syncthreads();
    if (p <= p1) {      // the two copies start together: warp 8 issues u, warp 7 b
      if (tid == rfw_issuer) issue_u(p - 1 + RFW_RU);
      else if (tid == rfw_issuer - 32) issue_b(p + RFW_RB);
    }
  };
  // phase p0: a of coarse plane jz0
  mbar_wait(bu + 0, 0u);
  mbar_wait(bu + 1, 0u);
  resid(std::integral_constant<int, 0>{}, p0);
  after(p0);
  // phases (p0 + 2i + 1, p0 + 2i + 2): odd plane (t, y pass of the coarse
  // plane finished two phases ago), even plane (c and the next a, x pass)
  for (int p = p0 + 1; p <= p1 + 2; p += 2) {
    const int ph = p - p0;                         // odd
    if (p <= p1) resid(std::integral_constant<int, 1>{}, p);
    if (ph >= 3) ypass();                          // y pass of jz = (p - 3) / 2
    after(p);
    if (p + 1 > p1 + 2) break;
    if (p + 1 <= p1) resid(std::integral_constant<int, 2>{}, p + 1);
    if (ph + 1 >= 4) xpass();                      // x pass of jz = (p - 3) / 2
    after(p + 1);
  }
}

// Shared pieces of the 3-D cubic interpolation kernel: coarse windows arrive
// by TMA (zero-filled outside the domain) into an 8-slot ring, issued as soon
// as a slot's plane is no longer needed; every tap is loaded from a safe index
// and accumulated by a predicated FMA, so the chains are branch-free and skip
// absent taps exactly like the reference's sparse rows.
constexpr int RQ4 = 8;

// acc = chain_{u < n} w[u] * v[u] in tap order (v loaded for every u).
// g_cubic_pad: absent taps carry weight 0 and are chained too -- the
// reference's dense tensordot adds those zero products as well, and for
// finite values acc + 0 * v == acc (acc is never -0: the chain starts from
// +0), so the result is the same bit for bit and the chain has no branches.
template <bool PAD>
__device__ __forceinline__ double tap_chain(int n, const double (&w)[4], double v0, double v1,
                                            double v2, double v3) {
  double acc = __fma_rn(w[0], v0, 0.0);
  if (PAD || n > 1) acc = __fma_rn(w[1], v1, acc);
  if (PAD || n > 2) acc = __fma_rn(w[2], v2, acc);
  if (PAD || n > 3) acc = __fma_rn(w[3], v3, acc);
  return acc;
}

constexpr int PF4 = TX * TY;

// k_cubic5: fine (+)= P_cubic coarse for 3-D (transfers.py:82-89) with the
// coincident rows, columns and planes specialised.  A fine index on a coarse
// point has the single weight 1 in the reference's dense interpolation
// matrix, so its dgemm chain fma(1, v, 0) + 0 * ... is exactly v + 0.0 for
// finite v; the other fine indices keep the 4-tap FMA chain in tap
// order.  Fine x columns and y rows alternate between the two kinds, so every
// thread owns one of each -- an x task is one column pair of one row, a y
// task one row pair of one coarse column -- and no warp diverges; fine z
// planes alternate too, and a coincident plane skips the z pass (its y pass
// reads the coarse window straight from the TMA ring).  Skewed three-stage
// pipeline (z pass of plane t, y pass of t-1, x pass of t-2), one
// barrier per plane; coarse windows (20 x 12) and, in accumulate mode, the
// old fine tiles arrive by TMA.  Bit-identical to the per-axis pass kernels.
constexpr int PYB5 = align16(QW * TY);
constexpr int NT5 = 256;
constexpr int RF5 = 6;                       // fine-tile ring (accumulate mode)
static_assert((TX / 2) * TY == NT5 && (TY / 2) * QW <= NT5 && QW * QH <= NT5, "task layout");

__global__ void __launch_bounds__(NT5, 4) k_cubic5(const __grid_constant__ CUtensorMap mc,
                                                   const __grid_constant__ CUtensorMap mf,
                                                   double* __restrict__ fine, Geo gf,
                                                   const int* __restrict__ tcnt,
                                                   const int* __restrict__ tidx,
                                                   const double* __restrict__ tw, int zc,
                                                   int accumulate) {
  __shared__ __align__(128) double sc[RQ4 * PQ];
  __shared__ __align__(128) double zb[PQ];
  __shared__ __align__(128) double yb[2 * PYB5];
  __shared__ __align__(8) unsigned long long bar[RQ4];
  __shared__ __align__(8) unsigned long long fbar[RF5];
  __shared__ double s_zw[64 * 4];
  __shared__ int s_zj[64 * 4], s_zn[64];
  extern __shared__ __align__(128) double sfine[];   // RF5 fine tiles (accumulate)
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, gf.nz);
  const int n = z1 - z0;
  const int cx0 = x0 / 2 - 2, cy0 = y0 / 2 - 2;
  auto first_tap = [&](int iz) { return __ldg(tidx + iz * 4); };
  auto last_tap = [&](int iz) { return __ldg(tidx + iz * 4 + __ldg(tcnt + iz) - 1); };
  const int jlo = n > 1 ? min(first_tap(z0), first_tap(z0 + 1)) : first_tap(z0);
  const int jtop = n > 1 ? max(last_tap(z1 - 1), last_tap(z1 - 2)) : last_tap(z1 - 1);
  if (tid == 0) {
    for (int i = 0; i < RQ4; ++i) mbar_init(bar + i, 1);
    for (int i = 0; i < RF5; ++i) mbar_init(fbar + i, 1);
    fence_barrier_init();
  }
  if (tid < n) {
    const int iz = z0 + tid, nt = __ldg(tcnt + iz);
    s_zn[tid] = nt;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s_zj[tid * 4 + u] = __ldg(tidx + iz * 4 + min(u, nt - 1));
      s_zw[tid * 4 + u] = u < nt ? __ldg(tw + iz * 4 + u) : 0.0;
    }
  }
  __syncthreads();
  constexpr int cissuer = NT5 - 32;
  auto issue_fine = [&](int p) {
    if (!accumulate || p >= z1) return;
    const int sl = (p - z0) % RF5;
    mbar_expect(fbar + sl, PF4 * 8u);
    tma3(sfine + sl * PF4, &mf, x0, y0, p, fbar + sl);
  };
  if (tid == cissuer)
    for (int p = z0; p < z0 + RF5; ++p) issue_fine(p);
  int issued = jlo;
  auto issue_upto = [&](int live_lo) {
    for (; issued <= jtop && issued < live_lo + RQ4; ++issued) {
      const int sl = (issued - jlo) & (RQ4 - 1);
      mbar_expect(bar + sl, QW * QH * 8u);
      tma3(sc + sl * PQ, &mc, cx0, cy0, issued, bar + sl);
    }
  };
  if (tid == cissuer) issue_upto(jlo);
  int waited = jlo;
  // ---- y task: coarse column ycx; fine rows y0+2q (4-tap, table taps) and
  // y0+2q+1 (coincident with coarse row y0/2+q, window row q+2)
  const bool yt = tid < (TY / 2) * QW;
  const int yq = tid / QW, ycx = tid - (tid / QW) * QW;
  int yi[4];
  double yw[4];
  {
    const int gy = y0 + 2 * yq;
    const bool ok = yt && gy < gf.ny;
    const int yn = ok ? __ldg(tcnt + gy) : 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      yi[u] = ok ? (__ldg(tidx + gy * 4 + min(u, yn - 1)) - cy0) * QW + ycx : ycx;
      yw[u] = ok && u < yn ? __ldg(tw + gy * 4 + u) : 0.0;
    }
  }
  const int yci = (yq + 2) * QW + ycx;
  const int yo = (2 * yq) * QW + ycx;
  // ---- x task: row xr, columns x0+2xp (4-tap) and x0+2xp+1 (coincident with
  // coarse column x0/2+xp, window column xp+2)
  const int xr = tid >> 4, xp = tid & 15;
  const int gx = x0 + 2 * xp, gy = y0 + xr;
  int xi[4];
  double xw[4];
  {
    const bool ok = gx < gf.nx;
    const int xn = ok ? __ldg(tcnt + gx) : 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      xi[u] = xr * QW + (ok ? __ldg(tidx + gx * 4 + min(u, xn - 1)) - cx0 : 0);
      xw[u] = ok && u < xn ? __ldg(tw + gx * 4 + u) : 0.0;
    }
  }
  const int xci = xr * QW + xp + 2;
  const bool in0 = gx < gf.nx && gy < gf.ny, in1 = gx + 1 < gf.nx && gy < gf.ny;
  const int fo = xr * TX + 2 * xp;
  double* fp = fine + (in0 ? gf.at(gx, gy, 0) : 0) + (long long)z0 * gf.sz;
  // z0 is even (even chunks): window planes t alternate 4-tap (t even: fine
  // array index even) and coincident (t odd).  Phase t runs the z pass of
  // plane t (4-tap planes only), the y pass of t-1 and the x pass of t-2, so
  // an even phase writes yb[1] and reads yb[0], an odd phase the reverse, and
  // one z buffer suffices (written in even phases, read in the next odd one).
  int fslot = 0, fphase = 0;   // fine-tile ring slot / phase of the x-pass plane
  auto wait_coarse = [&](int jmax) {
    for (; waited <= jmax; ++waited) {
      const int k = waited - jlo;
      mbar_wait(bar + (k & (RQ4 - 1)), (unsigned)((k / RQ4) & 1));
    }
  };
  auto xpass = [&](const double* ys, bool coincident_plane) {
    double a0 = tap_chain<true>(4, xw, ys[xi[0]], ys[xi[1]], ys[xi[2]], ys[xi[3]]);
    double a1 = ys[xci] + 0.0;
    (void)coincident_plane;
    if (accumulate) {
      mbar_wait(fbar + fslot, (unsigned)fphase);
      const double2 o = *reinterpret_cast<const double2*>(sfine + fslot * PF4 + fo);
      a0 = o.x + a0;
      a1 = o.y + a1;
    }
    if (++fslot == RF5) { fslot = 0; fphase ^= 1; }
    if (in1) *reinterpret_cast<double2*>(fp) = make_double2(a0, a1);
    else if (in0) fp[0] = a0;
    fp += gf.sz;
  };
  auto issue_after = [&](int t) {   // phase t done
    if (tid != cissuer) return;
    if (t >= 2) issue_fine(z0 + t - 2 + RF5);   // x pass of plane t-2 done: slot free
    int lo = jtop + 1;                  // coarse planes still read: z pass of t+1, t+2,
    if (t < n && s_zn[t] == 1) lo = min(lo, s_zj[t * 4]);   // y pass of a coincident t
    if (t + 1 < n) lo = min(lo, s_zj[(t + 1) * 4]);
    if (t + 2 < n) lo = min(lo, s_zj[(t + 2) * 4]);
    issue_upto(lo);
  };
  for (int t = 0; t < n + 2; t += 2) {
    // ---- even phase: z pass of 4-tap plane t, y pass of coincident t-1,
    // x pass of 4-tap t-2
    if (t < n) {
      int zj[4];
      double zw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { zj[u] = s_zj[t * 4 + u]; zw[u] = s_zw[t * 4 + u]; }
      wait_coarse(zj[3]);
      if (tid < QW * QH) {
        const double* s0 = sc + ((zj[0] - jlo) & (RQ4 - 1)) * PQ + tid;
        const double* s1 = sc + ((zj[1] - jlo) & (RQ4 - 1)) * PQ + tid;
        const double* s2 = sc + ((zj[2] - jlo) & (RQ4 - 1)) * PQ + tid;
        const double* s3 = sc + ((zj[3] - jlo) & (RQ4 - 1)) * PQ + tid;
        zb[tid] = tap_chain<true>(4, zw, *s0, *s1, *s2, *s3);
      }
    }
    if (t >= 1 && t - 1 < n && yt) {
      const double* zs = sc + ((s_zj[(t - 1) * 4] - jlo) & (RQ4 - 1)) * PQ;
      double* yd = yb + PYB5;
      yd[yo] = tap_chain<true>(4, yw, zs[yi[0]], zs[yi[1]], zs[yi[2]], zs[yi[3]]);
      yd[yo + QW] = zs[yci] + 0.0;
    }
    if (t >= 2) xpass(yb, false);
    __syncthreads();
    issue_after(t);
    if (t + 1 >= n + 2) break;
    // ---- odd phase: (coincident plane t+1 needs its coarse plane next
    // phase), y pass of 4-tap plane t, x pass of coincident t-1
    if (t + 1 < n) wait_coarse(s_zj[(t + 1) * 4]);
    if (t < n && yt) {
      double* yd = yb;
      yd[yo] = tap_chain<true>(4, yw, zb[yi[0]], zb[yi[1]], zb[yi[2]], zb[yi[3]]);
      yd[yo + QW] = zb[yci] + 0.0;
    }
    if (t >= 1) xpass(yb + PYB5, true);
    __syncthreads();
    issue_after(t + 1);
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

}  // namespace
int g_zrev_mask = 3;   // PL_OPT_ZREV: reverse z-chunk order of 1 apply / apply+rhs, 2 k_rfw
int g_zc_floor = 16;  // PL_OPT_ZC_FLOOR (A/B): smallest z chunk (4 and 8 measured slower at 127^3)
int g_zc_ctas = 148 * 8;   // PL_OPT_ZC_CTAS (A/B): CTA count the z chunking aims for
int g_zc_fit = 1;          // PL_OPT_ZC_FIT: wave-aware z chunks (pick_zc_fit)
namespace {
int pick_zc(const Geo& g) {
  // enough CTAs for several waves on 148 SMs; chunk halo planes cost
  // (2 or 4)/zc extra (L2) reads; zc even (the prolongation pairs planes).
  // Grids below ~2^24 points are L2-resident: short chunks are cheap there
  // and keep all SMs busy.
  long long tiles = (long long)ceil_div(g.nx, TX) * ceil_div(g.ny, TY);
  int zc = 64;
  while (zc > g_zc_floor && tiles * ceil_div(g.nz, zc) < g_zc_ctas) zc /= 2;
  return zc;
}

template <typename K>
void raise_smem(K kern, size_t bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// resident CTAs of one kernel configuration on the whole device (cached)
template <typename K>
int resident_ctas(K kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  auto key = std::make_tuple((const void*)kern, threads, smem, dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem);
  const int r = sms * (per > 0 ? per : 1);
  cache[key] = r;
  return r;
}

// Wave-aware z chunk (PL_OPT_ZC_FIT): the CTAs of a z-marching kernel (tiles
// x chunks, dispatched in blockIdx order) are list-scheduled on the device's
// resident slots, each taking (planes + extra) plane-phases, where extra is
// the pipeline fill and the per-CTA prologue; the chunk length in [zmin, zmax]
// (a multiple of step) with the shortest makespan wins, ties to the longer
// chunk.  At 255^3 with 4 CTAs per SM the power-of-two chunks give 1.7 or 3.5
// waves; e.g. 30-plane chunks give 1,152 CTAs = 1.95 waves.
int pick_zc_fit(const Geo& g, int slots, int step, int extra, int zmin, int zmax) {
  if (!g_zc_fit) return pick_zc(g);
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int, int>, int> cache;
  const long long tiles = (long long)ceil_div(g.nx, TX) * ceil_div(g.ny, TY);
  auto key = std::make_tuple(g.nz, (int)tiles, slots, step, extra, zmin, zmax);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int best = zmax;
  long long best_t = -1;
  std::vector<long long> fin;
  for (int zc = zmax; zc >= zmin; zc -= step) {
    fin.assign(slots, 0);
    std::make_heap(fin.begin(), fin.end(), std::greater<long long>());
    long long end = 0;
    for (int z = 0; z < g.nz; z += zc) {
      const long long d = std::min(zc, g.nz - z) + extra;
      for (long long t = 0; t < tiles; ++t) {
        std::pop_heap(fin.begin(), fin.end(), std::greater<long long>());
        fin.back() += d;
        end = std::max(end, fin.back());
        std::push_heap(fin.begin(), fin.end(), std::greater<long long>());
      }
    }
    if (best_t < 0 || end < best_t) {
      best_t = end;
      best = zc;
    }
  }
  cache[key] = best;
  return best;
}

template <int OP>
int launch_z1(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
              double sigma, double omega, double dval, cudaStream_t s,
              const RhsArgs& ra = RhsArgs{}) {
  constexpr int HX = TX + 4, HY = TY + 2, RING = PREF1 + 3;
  if (g.nstore >= (1LL << 31)) {     // the kernel indexes a field with 32-bit element offsets
    set_error("k_z1: field of %lld elements exceeds 2^31", g.nstore);
    return 2;
  }
  CUtensorMap mu, mb;
  std::memset(&mu, 0, sizeof(mu));
  std::memset(&mb, 0, sizeof(mb));
  if (OP != Z_JAC0) PL_TRY(make_map(&mu, u, g, HX, HY));
  constexpr bool NB = OP != Z_APPLY && OP != Z_APPLY_RHS;
  if (NB) PL_TRY(make_map(&mb, b, g, TX, TY));
  size_t smem = sizeof(double) * RING *
                    ((OP != Z_JAC0 ? align16(HX * HY) : 0) + (NB ? align16(TX * TY) : 0)) +
                8 * RING;
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc)), block(32, 8);
  auto kern = c.pow2 ? k_z1<OP, true, PREF1> : k_z1<OP, false, PREF1>;
  raise_smem(kern, smem);
  const bool rev = (OP == Z_APPLY || OP == Z_APPLY_RHS) && (g_zrev_mask & 1);
  kern<<<grid, block, smem, s>>>(mu, mb, out, g, c, sigma, omega, dval, rev ? -zc : zc, ra);
  return 0;
}

// e (coarse correction, geometry gc) non-null: prolongation fused
int launch_z2(const double* u, const double* b, const double* e, const Geo& gc, double* out,
              const Geo& g, const OpC& c, double sigma, double omega, double dval, int zero_in,
              cudaStream_t s) {
  constexpr int HX = TX + 2, HY = TY + 2;
  CUtensorMap mu, mb, me;
  std::memset(&mu, 0, sizeof(mu));
  std::memset(&me, 0, sizeof(me));
  if (!zero_in) PL_TRY(make_map(&mu, u, g, UX, UY));
  PL_TRY(make_map(&mb, b, g, BW, BH));
  if (e) PL_TRY(make_map(&me, e, gc, CW, CH));
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc)), block(32, 8);
#define PL_Z2(P2, PRO)                                                                  \
  do {                                                                                 \
    size_t smem = (Stager<NTHR, PRO, PREF2>::smem_doubles() + 16 + 3 * align16(HX * HY)) * 8; \
    auto kern = k_z2<P2, PRO, PREF2>;                                                  \
    raise_smem(kern, smem);                                                            \
    kern<<<grid, block, smem, s>>>(mu, mb, me, out, g, c, sigma, omega, dval, zc, zero_in); \
  } while (0)
  if (c.pow2) {
    if (e) PL_Z2(true, true); else PL_Z2(true, false);
  } else {
    if (e) PL_Z2(false, true); else PL_Z2(false, false);
  }
#undef PL_Z2
  return 0;
}

int launch_zrb3(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
                double sigma, double omega, double dval, cudaStream_t s) {
  CUtensorMap mu, mb;
  PL_TRY(make_map(&mu, u, g, UX, UY));
  PL_TRY(make_map(&mb, b, g, BW, BH));
  int zc = pick_zc(g);
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(g.nz, zc));
  const double dinv = 1.0 / dval;
  const bool unit = c.nu == 1.0 && omega == 1.0;   // exact multiplications skipped
  // default (0): 6 u + 3 b planes from 255^3 up, in z chunks of >= 32 planes
  // (1,024 CTAs at 255^3, 1.7 waves of 4 per SM: 91 vs 97 us); the 8 + 4
  // rings at 3 CTAs per SM below, where they are faster (26 vs 27 us at 127^3)
  const bool big = g_zrb_ring == 0 && g.N >= 255;
  if (big) zc = zc < 32 ? 32 : zc;
  if (g_zrb_ring == 1 || big) {   // 6 u + 3 b planes, 4 CTAs per SM (register cap 64)
    size_t smem = (size_t)(6 + 3) * USL * 8;
    auto kern = c.pow2 ? (unit ? k_zrb3<true, 6, 3, 4, true> : k_zrb3<true, 6, 3, 4, false>)
                       : (unit ? k_zrb3<false, 6, 3, 4, true> : k_zrb3<false, 6, 3, 4, false>);
    raise_smem(kern, smem);
    // even chunks (the phase code assumes an even z0)
    if (g_zc_fit) zc = pick_zc_fit(g, resident_ctas(kern, NTHR_RB2, smem), 2, 5, 16, 64);
    grid.z = ceil_div(g.nz, zc);
    kern<<<grid, dim3(NTHR_RB2), smem, s>>>(mu, mb, out, g, c, sigma, omega, dval, dinv, zc);
    return 0;
  }
  size_t smem = (size_t)(8 + 4) * USL * 8;
  auto kern = c.pow2 ? (unit ? k_zrb3<true, 8, 4, 3, true> : k_zrb3<true, 8, 4, 3, false>)
                     : (unit ? k_zrb3<false, 8, 4, 3, true> : k_zrb3<false, 8, 4, 3, false>);
  raise_smem(kern, smem);
  // (wave-fitted shorter chunks are faster for a lone sweep on the L2-resident
  // levels -- 35 vs 38 us at 127^3 with 10 planes, 25 vs 30 us at 63^3 with 2 --
  // but not inside the rank-stream wavefront: 7.04-7.18 vs 7.20-7.23 time-steps/s)
  kern<<<grid, dim3(NTHR_RB2), smem, s>>>(mu, mb, out, g, c, sigma, omega, dval, dinv, zc);
  return 0;
}

int launch_rfw(const double* u, const double* b, double* coarse, const Geo& g, const OpC& c,
               double sigma, cudaStream_t s) {
  Geo gc = make_geo(3, (g.N + 1) / 2);
  CUtensorMap mu, mb;
  PL_TRY(make_map(&mu, u, g, FUX, FUY));
  PL_TRY(make_map(&mb, b, g, FBX, FBY));
  const int zcc = pick_zc(g) / 2 < 4 ? 4 : pick_zc(g) / 2;
  dim3 grid(ceil_div(g.nx, TX), ceil_div(g.ny, TY), ceil_div(gc.nz, zcc));
  auto kern = c.pow2 ? (c.nu == 1.0 ? k_rfw<true, true> : k_rfw<true, false>)
                     : (c.nu == 1.0 ? k_rfw<false, true> : k_rfw<false, false>);
  raise_smem(kern, RFW_SMEM);
  kern<<<grid, RFW_NT, RFW_SMEM, s>>>(mu, mb, coarse, g, gc, c, sigma,
                                      (g_zrev_mask & 2) ? -zcc : zcc);
  return 0;
}

}  // namespace
namespace {

int launch_cubic5(const double* coarse, double* fine, const Geo& gf, const int* cnt,
                  const int* idx, const double* w, int accumulate, cudaStream_t s) {
  Geo gc = make_geo(3, (gf.N + 1) / 2);
  const int zc = pick_zc(gf);
  dim3 grid(ceil_div(gf.nx, TX), ceil_div(gf.ny, TY), ceil_div(gf.nz, zc));
  CUtensorMap mc;
  PL_TRY(make_map(&mc, coarse, gc, QW, QH));
  CUtensorMap mf;
  std::memset(&mf, 0, sizeof(mf));
  if (accumulate) PL_TRY(make_map(&mf, fine, gf, TX, TY));
  const size_t smem5 = accumulate ? sizeof(double) * RF5 * PF4 : 0;
  raise_smem(k_cubic5, smem5);
  const int zc5 = pick_zc_fit(gf, resident_ctas(k_cubic5, NT5, smem5), 2, 5, 8, 64);
  grid.z = ceil_div(gf.nz, zc5);
  k_cubic5<<<grid, NT5, smem5, s>>>(mc, mf, fine, gf, cnt, idx, w, zc5, accumulate);
  return 0;
}

}  // namespace

int zlaunch_cubic(const double* coarse, double* fine, const Geo& gf, const int* cnt,
                  const int* idx, const double* w, int accumulate, cudaStream_t s) {
  PL_PRE(K_INTERP);
  PL_TRY(launch_cubic5(coarse, fine, gf, cnt, idx, w, accumulate, s));
  Geo gc = make_geo(3, (gf.N + 1) / 2);
  PL_CHECK_LAUNCH(K_INTERP, (accumulate ? 16.0 : 8.0) * gf.npts + 8.0 * gc.npts);
  return 0;
}

// host value of 1 - sigma * (nu * ((0 + d) + d + d)) for order 2 (constant)
double zdiag(const OpC& c, double sigma) {
  double t = 0.0;
  t = t + c.d1_int;
  t = t + c.d1_int;
  t = t + c.d1_int;
  return 1.0 - sigma * (c.nu * t);
}

int g_zmarch_enabled = 1;   // runtime knob (pl_set_option), for A/B tests
int g_zrb_ring = 0;
int g_fuse_prolong = 0;     // Jacobi: prolongation fused into the first post-sweep pair (k_z2)
bool zmarch_fuse_prolong() { return g_fuse_prolong != 0; }
// smallest interior size for the TMA kernels: below it a CTA would march many
// planes for few CTAs (latency-bound); the one-point-per-thread kernels win
int g_zmarch_min_n = 127;
bool zmarch_enabled() { return g_zmarch_enabled != 0; }
bool zmarch_size_ok(int N) { return g_zmarch_enabled && N >= g_zmarch_min_n; }

bool zmarch_ok(const Geo& g, const OpC& c) {
  // TMA needs 16-byte row and plane strides: the padded device layout
  return g_zmarch_enabled && g.dim == 3 && c.order == 2 && g.N >= g_zmarch_min_n && g.N >= 31 &&
         (g.sy % 2) == 0;
}

int g_rfw_enabled = 1;     // PL_OPT_RFW: fused residual + full weighting
bool zmarch_rfw() { return g_rfw_enabled != 0; }

int zlaunch_rfw(const double* u, const double* b, double* coarse, const Geo& g, const OpC& c,
                double sigma, cudaStream_t s) {
  Geo gc = make_geo(3, (g.N + 1) / 2);
  PL_PRE(K_RESTRICT);
  PL_TRY(launch_rfw(u, b, coarse, g, c, sigma, s));
  // read u, b (16 B per fine point), write the coarse rhs
  PL_CHECK_LAUNCH(K_RESTRICT, 16.0 * g.npts + 8.0 * gc.npts);
  return 0;
}

int zlaunch_apply(const double* u, double* f, const Geo& g, const OpC& c, cudaStream_t s) {
  PL_PRE(K_APPLY);
  PL_TRY(launch_z1<Z_APPLY>(u, nullptr, f, g, c, 0.0, 0.0, 1.0, s));
  PL_CHECK_LAUNCH(K_APPLY, 16.0 * g.npts);
  return 0;
}

int zlaunch_apply_rhs(const double* u, double* f, const double* fnext, const double* sm,
                      const double* tau0, const double* tau1, double dtm, double* rhs,
                      const Geo& g, const OpC& c, cudaStream_t s) {
  RhsArgs ra{fnext, sm, tau0, tau1, rhs, dtm};
  PL_PRE(K_APPLY_RHS);
  PL_TRY(launch_z1<Z_APPLY_RHS>(u, nullptr, f, g, c, 0.0, 0.0, 1.0, s, ra));
  // the unfused passes it replaces: apply (16 B) + rhs (32 B, 48 B with tau),
  // minus the shared read of u
  PL_CHECK_LAUNCH(K_APPLY_RHS, (tau0 ? 56.0 : 40.0) * g.npts);
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
                    double sigma, double omega, int zero_in, const double* e, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  Geo gc = make_geo(3, (g.N + 1) / 2);
  PL_PRE(K_JACOBI);
  PL_TRY(launch_z2(u, b, e, gc, out, g, c, sigma, omega, dval, zero_in, s));
  // algorithmic bytes of the unfused passes it replaces (two sweeps, prolongation)
  PL_CHECK_LAUNCH(K_JACOBI, (zero_in ? 40.0 : 48.0) * g.npts +
                                (e ? 16.0 * g.npts + 8.0 * gc.npts : 0.0));
  return 0;
}

int zlaunch_rb(const double* u, const double* b, double* out, const Geo& g, const OpC& c,
               double sigma, double omega, cudaStream_t s) {
  double dval = zdiag(c, sigma);
  if (!diag_div_ok(dval)) {   // outside div_const's range: the one-colour kernels
    PL_TRY(launch_rb(u, b, out, g, c, sigma, omega, 1, s));
    return launch_rb(out, b, out, g, c, sigma, omega, 0, s);
  }
  PL_PRE(K_RB);
  PL_TRY(launch_zrb3(u, b, out, g, c, sigma, omega, dval, s));
  PL_CHECK_LAUNCH(K_RB, 24.0 * g.npts);
  return 0;
}

}  // namespace pl
