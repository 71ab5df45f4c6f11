// TMA latency/throughput probe: D-deep ring, one issuing thread per CTA, 148 CTAs.
//   mode 0: tiled 4D box (64 B x 128 rows) ; mode 1: im2col (64 ch x 128 px)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE_%=;\nbra "
      "WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(b)),
      "r"(ph)
      : "memory");
}
__global__ void k(const __grid_constant__ CUtensorMap map, int mode, int iters, int depth, int box_bytes, int Q, int P,
                  int N, long long* out, int per) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int wq = threadIdx.x / 32, nw = blockDim.x / 32;
  if (threadIdx.x % 32 == 0) {
    uint64_t* bar0 = bar + wq * depth;
    if (per < 0) {}
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map) : "memory");
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      int s = it % depth, use = it / depth;
      if (use > 0) wait(&bar0[s], (use - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar0[s])), "r"(box_bytes * per));
      for (int pp = 0; pp < per; pp++) {
      int n = (blockIdx.x + it) & (N - 1), x = it & 31, y = (it >> 5) & 7;
      uint32_t dst = smem_u32(base + (wq * depth + s) * 8192 * per + pp * 8192);
      if (mode == 1)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
            "l"((uint64_t)&map), "r"(smem_u32(&bar0[s])), "r"(0), "r"(y), "r"(x), "r"(n), "h"((uint16_t)1),
            "h"((uint16_t)1)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
            "[%2];" ::"r"(dst),
            "l"((uint64_t)&map), "r"(smem_u32(&bar0[s])), "r"(0), "r"(0), "r"(x), "r"(n)
            : "memory");
      }
    }
    for (int it = iters; it < iters + depth; it++) {
      int s = it % depth, use = it / depth;
      if (use > 0) wait(&bar0[s], (use - 1) & 1);
    }
    if (wq == 0) out[blockIdx.x] = clock64() - t0;
  }
}
int main(int argc, char** argv) {
  int mode = atoi(argv[1]), depth = atoi(argv[2]);
  int N = argc > 3 ? atoi(argv[3]) : 128;
  int nw = argc > 4 ? atoi(argv[4]) : 1;
  int per = argc > 5 ? atoi(argv[5]) : 1;
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeIm2col_v12000)fn;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enct = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int H = 56, W = 56, C = 64;
  uint8_t* g;
  cudaMalloc(&g, (size_t)N * (H + 4) * (W + 4) * C + 4096);
  cudaMemset(g, 1, (size_t)N * H * W * C);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  CUtensorMap m;
  cuuint64_t dim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t str[3] = {(cuuint64_t)C, (cuuint64_t)C * W, (cuuint64_t)C * W * H};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r;
  if (mode == 2) {  // overlapping: 16-byte folded pixels, 64-byte rows starting at every pixel
    int lower[2] = {0, 0}, upper[2] = {0, -3};
    cuuint64_t dim2[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t str2[3] = {16, 16 * (W + 3), 16 * (W + 3) * H};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, g, dim2, str2, lower, upper, 64, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    mode = 1;
  } else if (mode == 3) {  // same geometry but 64-byte pixel stride (no overlap)
    int lower[2] = {0, 0}, upper[2] = {0, -3};
    cuuint64_t dim2[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t str2[3] = {64, 64 * (W + 3), 64 * (W + 3) * H};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, g, dim2, str2, lower, upper, 64, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    mode = 1;
  } else if (mode == 1) {
    int lower[2] = {-1, -1}, upper[2] = {-1, -1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, g, dim, str, lower, upper, 64, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint32_t box[4] = {64, 56, 2, 1};  // 112 rows of 64 B
    r = enct(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, g, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r) {
    printf("encode %d\n", r);
    return 1;
  }
  int box = mode == 0 ? 64 * 112 : 8192;
  int iters = 1000;
  for (int rep = 0; rep < 2; rep++) {
    k<<<148, 32 * nw, 200 * 1024>>>(m, mode, iters, depth, box, W, H, N, d, per);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; i++) avg += h[i];
    avg /= 148;
    double cyc = avg / iters;
    if (rep)
      printf("per %d warps %d mode %d depth %2d N %3d: %7.1f cyc/box/warp  %6.1f B/clk/SM  latency~%.0f cyc %s\n", per, nw, mode, depth, N, cyc,
             box * per / cyc * nw, cyc * depth, e ? cudaGetErrorString(e) : "");
  }
}
