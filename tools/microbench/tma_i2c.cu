// Microbenchmark: TMA im2col load throughput per SM (148 CTAs, one thread issuing, 4-deep ring).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap map, int iters, int box_bytes, int Q, int P, int N, int taps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    uint32_t phase[8] = {0};
    for (int it = 0; it < iters; it++) {
      int s = it & 7;
      if (it >= 8) {
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar[s])), "r"(phase[s]));
        phase[s] ^= 1;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(box_bytes));
      long long m = ((long long)(blockIdx.x + 148 * (it / taps)) * 128) % ((long long)N * P * Q);
      int tap = it % taps;
      int n = m / (P * Q), rem = m % (P * Q), x = rem / Q, y = rem % Q;
      uint32_t dst = smem_u32(base + s * 16384);
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
          "l"((uint64_t)&map), "r"(smem_u32(&bar[s])), "r"(0), "r"(y), "r"(x), "r"(n), "h"((uint16_t)(tap % 3)), "h"((uint16_t)(tap / 3))
          : "memory");
    }
    for (int s = 0; s < 8; s++)
      asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D2;\nbra W2;\nD2:\n}" ::"r"(smem_u32(&bar[s])), "r"(phase[s]));
    out[blockIdx.x] = clock64() - t0;
  }
}
int main(int argc, char** argv) {
  int only = argc > 1 ? atoi(argv[1]) : -1;
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeIm2col_v12000)fn;
  uint8_t* g; cudaMalloc(&g, 1ull << 30); cudaMemset(g, 1, 1ull << 30);
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  struct C { const char* name; int ch; int N, H, W; int pix; CUtensorMapSwizzle sw; int stride; } cs[] = {
    {"C64  56x56 b128 (27MB) sw64", 64, 128, 56, 56, 128, CU_TENSOR_MAP_SWIZZLE_64B, 64},
    {"C64  56x56 b8 (L2) sw64", 64, 8, 56, 56, 128, CU_TENSOR_MAP_SWIZZLE_64B, 64},
    {"C128 28x28 b128 sw128", 128, 128, 28, 28, 128, CU_TENSOR_MAP_SWIZZLE_128B, 128},
    {"C128 28x28 b8 (L2) sw128", 128, 8, 28, 28, 128, CU_TENSOR_MAP_SWIZZLE_128B, 128},
    {"C64 overlapping stride16 (fold) b128", 64, 128, 115, 112, 128, CU_TENSOR_MAP_SWIZZLE_64B, 16},
    {"C64 overlapping stride16 (fold) b8", 64, 8, 115, 112, 128, CU_TENSOR_MAP_SWIZZLE_64B, 16},
    {"C64 56x56 b128 pix64 sw64", 64, 128, 56, 56, 64, CU_TENSOR_MAP_SWIZZLE_64B, 64},
  };
  int ci = -1;
  for (auto& c : cs) {
    if (++ci != only && only >= 0) continue;
    CUtensorMap m;
    cuuint64_t dim[4] = {(cuuint64_t)c.ch, (cuuint64_t)c.W, (cuuint64_t)c.H, (cuuint64_t)c.N};
    cuuint64_t str[3] = {(cuuint64_t)c.stride, (cuuint64_t)c.stride * (c.W + (c.stride == 16 ? 3 : 0)), (cuuint64_t)c.stride * (c.W + 3) * c.H};
    int lower[2] = {-1, -1}, upper[2] = {-1, -1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, g, dim, str, lower, upper, c.ch, c.pix, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("%s: encode %d\n", c.name, r); continue; }
    int iters = 2000, taps = 9;
    int box = c.ch * c.pix;
    for (int rep = 0; rep < 2; rep++) {
      k<<<148, 32, 140 * 1024>>>(m, iters, box, c.W, c.H, c.N, taps, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; i++) avg += h[i]; avg /= 148;
      double cyc = avg / iters;
      if (rep) printf("%-40s box %5d B: %7.1f cyc/box %6.1f B/clk/SM %5.2f cyc/pixel %s\n", c.name, box, cyc, box / cyc, cyc / c.pix, e ? cudaGetErrorString(e) : "");
    }
  }
}
