// Minimal TMA probe: copy one box of a padded 3-D fp64 field to smem, write it back.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int bw, int bh, int x, int y, int z) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(&bar)), "r"(bw * bh * 8) : "memory");
    if (VARIANT == 0)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                   ::"r"(saddr(sm)), "l"(&map), "r"(x), "r"(y), "r"(z), "r"(saddr(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                   ::"r"(saddr(sm)), "l"(&map), "r"(x), "r"(y), "r"(z), "r"(saddr(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(saddr(&bar)) : "memory");
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  int bw = argc > 2 ? atoi(argv[2]) : 34, bh = argc > 3 ? atoi(argv[3]) : 18;
  int cx = argc > 4 ? atoi(argv[4]) : -1, cy = argc > 5 ? atoi(argv[5]) : -1, cz = argc > 6 ? atoi(argv[6]) : 3;
  int dt = argc > 7 ? atoi(argv[7]) : 0;
  const int N = 31, P = 32;
  std::vector<double> h((size_t)N * N * P, 0.0);
  for (int z = 0; z < N; ++z) for (int y = 0; y < N; ++y) for (int x = 0; x < N; ++x)
    h[(size_t)z * N * P + y * P + x] = 1 + x + 100 * y + 10000 * z;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 4096 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap map; memset(&map, 0, sizeof(map));
  cuuint64_t dims[3] = {N, N, N};
  cuuint64_t strides[2] = {P * 8, (cuuint64_t)N * P * 8};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&map, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d q=%d\n", (int)r, (int)q);
  size_t smem = bw * bh * 8;
  if (variant == 0) k<0><<<1, 128, smem>>>(map, o, bw, bh, cx, cy, cz);
  else k<1><<<1, 128, smem>>>(map, o, bw, bh, cx, cy, cz);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d: %s\n", variant, cudaGetErrorString(e));
  std::vector<double> out(bw * bh);
  cudaMemcpy(out.data(), o, out.size() * 8, cudaMemcpyDeviceToHost);
  printf("row0: %g %g %g ... row1: %g %g\n", out[0], out[1], out[2], out[bw], out[bw + 1]);
  return 0;
}
