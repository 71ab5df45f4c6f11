// tcgen05.mma kind::i8 issue rate while other warps poll an mbarrier (derived from mma_layout.cu);
// originally: issue rate vs the A/B shared-memory layouts (one CTA per SM, M = 128):
// SW128 K-major; no-swizzle with overlapping rows (the band mode's A: row m at 16 m, LBO 16,
// SBO 128); no-swizzle interleaved (8 x 16 B core matrices, K-adjacent: LBO 128, SBO 256).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mma_layout mma_layout.cu && ./mma_layout
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ uint64_t mk(int mode, uint32_t a) {
  return mode == 0 ? desc(a, 16, 1024, 2) : mode == 1 ? desc(a, 16, 128, 0) : desc(a, 128, 256, 0);
}

__global__ void k(int iters, int N, long long* out, int amode, int bmode, int vary, int hint) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, done;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 120 * 1024; i += blockDim.x) base[i] = (uint8_t)(i * 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = slot;
  uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    uint32_t a = smem_u32(base);
    uint32_t b = smem_u32(base) + 48 * 1024;
    uint64_t ads[8], bds[8];
    for (int q = 0; q < 8; q++) {
      // band A: consecutive k-steps 32 B apart inside the same rows; otherwise 4 KB slices
      const uint32_t ao = vary ? (amode == 1 ? q * 2048 + (q & 1) * 32 : q * 4096) : 0, bo = vary ? (q & 3) * 8192 : 0;
      ads[q] = mk(amode, a + ao);
      bds[q] = mk(bmode, b + bo);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int q = 0; q < 8; q++)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                     "l"(ads[q]), "l"(bds[q]), "r"(idesc), "r"(it + q));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done)) : "memory");
  } else if (threadIdx.x >= 32) {
    // the other warps poll an mbarrier that completes when the MMAs are done (like idle
    // epilogue / producer warps): hint 1 = try_wait with a suspend-time hint, 0 = without,
    // 2 = test_wait spin, 3 = try_wait + nanosleep backoff
    const uint32_t a = smem_u32(&done);
    if (hint == 1)
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0, %1;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(a), "r"(0x989680u) : "memory");
    else if (hint == 0)
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(a) : "memory");
    else if (hint == 2)
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(a) : "memory");
    else {
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\nselp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(a) : "memory");
        if (!ok) __nanosleep(200);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main(int argc, char** argv) {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  // N = 128, band A / SW128 B, varying operands; 0 .. 12 extra polling warps, four poll styles
  for (int hint = 0; hint < 4; hint++)
    for (int warps : {1, 5, 9, 13}) {
      const int iters = 4000;
      cudaMemset(d, 0, 1024 * 8);
      k<<<148, 32 * warps, 128 * 1024>>>(iters, 128, d, 1, 0, 1, hint);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; i++) avg += h[i];
      avg /= 148;
      printf("poll style %d, %2d polling warps: %6.1f cycles/MMA %s\n", hint, warps - 1, avg / iters,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
}
