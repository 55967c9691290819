// Lexicographic Gauss-Seidel sweeps on the grid-wide levels (multigrid.py:
// 219-224), bit-identical to scipy.linalg.solve_banded (see gs.cuh).
//
// One sweep = the residual kernel (r = b - A_sigma u into the scratch t) and
// one cooperative launch that walks the hyperplanes s = x + y + z in order:
// every point of hyperplane s reads the final y of its lower neighbours
// (hyperplanes s-1, s-2), overwrites its r with y and adds y / D to u; a
// grid-wide barrier separates the hyperplanes.  1-D is a single recurrence
// and runs on one thread.  The smoother is inherently sequential along the
// hyperplanes (3N - 2 barriers per 3-D sweep); no BASELINE configuration
// uses it, the reference's CLI presets and tests do.
#include <cooperative_groups.h>

#include "gs.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace pl {

namespace {

constexpr int GS_THREADS = 512;

template <int DIM>
__device__ __forceinline__ void gs_update(double* u, double* t, const Geo& g, const OpC& c,
                                          double sigma, int x, int y, int z) {
  const long long idx = g.at(x, y, z);
  const double yi = gs_lower_point<DIM>(t, t[idx], g, c, sigma, x, y, z, idx);
  t[idx] = yi;
  u[idx] = u[idx] + yi / shifted_diag<DIM>(g, c, sigma, x, y, z);
}

template <int DIM>
__global__ void __launch_bounds__(GS_THREADS) k_gs_wave(double* u, double* t, Geo g, OpC c,
                                                        double sigma) {
  cg::grid_group grid = cg::this_grid();
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  const int smax = (g.nx - 1) + (DIM >= 2 ? g.ny - 1 : 0) + (DIM == 3 ? g.nz - 1 : 0);
  for (int s = 0; s <= smax; ++s) {
    if (DIM == 2) {
      const int ylo = max(0, s - (g.nx - 1)), yhi = min(g.ny - 1, s);
      for (long long k = gt; k <= yhi - ylo; k += gs) {
        const int y = ylo + (int)k;
        gs_update<2>(u, t, g, c, sigma, s - y, y, 0);
      }
    } else {
      const int zlo = max(0, s - (g.nx - 1) - (g.ny - 1)), zhi = min(g.nz - 1, s);
      const long long cand = (long long)(zhi - zlo + 1) * g.ny;
      for (long long k = gt; k < cand; k += gs) {
        const int z = zlo + (int)(k / g.ny), y = (int)(k % g.ny);
        const int x = s - y - z;
        if (x < 0 || x >= g.nx) continue;
        gs_update<3>(u, t, g, c, sigma, x, y, z);
      }
    }
    grid.sync();
  }
}

__global__ void k_gs_line(double* u, double* t, Geo g, OpC c, double sigma) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int x = 0; x < g.nx; ++x) gs_update<1>(u, t, g, c, sigma, x, 0, 0);
}

}  // namespace

int launch_gs(double* u, const double* b, double* t, const Geo& g, const OpC& c, double sigma,
              int count, cudaStream_t s) {
  for (int k = 0; k < count; ++k) {
    PL_TRY(launch_residual(u, b, t, g, c, sigma, s));
    PL_PRE(K_GS);
    if (g.dim == 1) {
      k_gs_line<<<1, 32, 0, s>>>(u, t, g, c, sigma);
    } else {
      void* kern = g.dim == 2 ? (void*)k_gs_wave<2> : (void*)k_gs_wave<3>;
      // resident grid, cached per device and dimension
      static int grid_of[64][4] = {};
      int dev = 0;
      cudaGetDevice(&dev);
      int* grid = grid_of[dev & 63];
      if (grid[g.dim] == 0) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, GS_THREADS, 0);
        if (per < 1) {
          set_error("gauss-seidel wavefront kernel does not fit one CTA per SM");
          return 2;   // PL_ERR_CUDA
        }
        grid[g.dim] = sms * (per < 2 ? per : 2);
      }
      // enough threads for the widest hyperplane, at most the resident grid
      const long long width = g.dim == 2 ? g.ny : (long long)g.ny * g.nz;
      int blocks = (int)((width + GS_THREADS - 1) / GS_THREADS);
      blocks = blocks < 1 ? 1 : (blocks > grid[g.dim] ? grid[g.dim] : blocks);
      Geo gg = g;
      OpC cc = c;
      double sg = sigma;
      void* args[] = {&u, &t, &gg, &cc, &sg};
      cudaError_t e = cudaLaunchCooperativeKernel(kern, blocks, GS_THREADS, args, 0, s);
      if (e != cudaSuccess) return cuda_status(e, "gauss-seidel wavefront");
    }
    // algorithmic bytes of the triangular solve pass: read r, u; write y, u
    PL_CHECK_LAUNCH(K_GS, 32.0 * g.npts);
  }
  return 0;
}

}  // namespace pl
