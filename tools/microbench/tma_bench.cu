// Microbenchmark: TMA load throughput per SM for different box shapes (all CTAs busy).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int RANK>
__global__ void k(const __grid_constant__ CUtensorMap map, int iters, int box_bytes, int ncoord, int v0, long long* out) {
  const int mode = 0;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    uint32_t phase[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; it++) {
      int s = it & 3;
      if (it >= 4) {
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar[s])), "r"(phase[s]));
        phase[s] ^= 1;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(box_bytes));
      int c = (blockIdx.x * 7 + it) % ncoord;
      uint32_t dst = smem_u32(base + s * 32768);
      if (mode == 0)
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                     ::"r"(dst), "l"((uint64_t)&map), "r"(smem_u32(&bar[s])), "r"(0), "r"(v0), "r"(0), "r"(c) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(dst), "l"((uint64_t)&map), "r"(smem_u32(&bar[s])), "r"(0), "r"(c * 128) : "memory");
    }
    for (int s = 0; s < 4; s++)
      asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D2;\nbra W2;\nD2:\n}" ::"r"(smem_u32(&bar[s])), "r"(phase[s]));
    out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  size_t bytes = 1100ull << 20;
  uint8_t* g;
  cudaMalloc(&g, bytes);
  cudaMemset(g, 1, bytes);
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  cuuint32_t es[4] = {1, 1, 1, 1};
  struct Cfg { const char* name; int inner, P, rows; CUtensorMapSwizzle sw; int vdim = 256; int v0 = 0; } cfgs[] = {
      {"4d inner64 P64 rows4 sw64 OOB v=-1,W=56", 64, 64, 4, CU_TENSOR_MAP_SWIZZLE_64B, 56, -1},
      {"4d inner64 P64 rows4 sw64 W=56 v=0", 64, 64, 4, CU_TENSOR_MAP_SWIZZLE_64B, 56, 0},
      {"4d inner64 P64 rows4 sw64 W=64 v=-1", 64, 64, 4, CU_TENSOR_MAP_SWIZZLE_64B, 64, -1},
      {"4d inner16 P64 rows4 (v1 planes)", 16, 64, 4, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"4d inner64 P64 rows4 sw64 (v2)", 64, 64, 4, CU_TENSOR_MAP_SWIZZLE_64B},
      {"4d inner64 P64 rows4 noswz", 64, 64, 4, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"4d inner128 P64 rows4 sw128", 128, 64, 4, CU_TENSOR_MAP_SWIZZLE_128B},
      {"4d inner64 P256 rows1 sw64", 64, 256, 1, CU_TENSOR_MAP_SWIZZLE_64B},
  };
  for (auto& c : cfgs) {
    CUtensorMap m;
    // dims (c=inner, v=56.., u, n)
    cuuint64_t dims[4] = {(cuuint64_t)c.inner, (cuuint64_t)c.vdim, 64, 128};
    cuuint64_t str[3] = {(cuuint64_t)c.inner, (cuuint64_t)c.inner * 256, (cuuint64_t)c.inner * 256 * 64};
    cuuint32_t box[4] = {(cuuint32_t)c.inner, (cuuint32_t)c.P, (cuuint32_t)c.rows, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, r); continue; }
    int box_bytes = c.inner * c.P * c.rows;
    int iters = 400;
    k<4><<<148, 32, 140 * 1024>>>(m, iters, box_bytes, 128, c.v0, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; i++) avg += h[i];
    avg /= 148;
    double cyc = avg / iters;
    printf("%-36s box %6d B: %7.1f cycles/box  %6.1f B/cycle/SM  rows=%d -> %.1f cyc/row  %s\n", c.name, box_bytes, cyc,
           box_bytes / cyc, c.P * c.rows, cyc / (c.P * c.rows), e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
}
