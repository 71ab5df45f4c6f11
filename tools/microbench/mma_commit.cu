// tcgen05.mma kind::i8 rate (M = 128, N = 128, one CTA per SM, unrolled issue with precomputed
// descriptors) when a tcgen05.commit to an mbarrier follows every C MMAs, and when the issuing
// warp additionally waits for the commit of C MMAs earlier (W = 1: the kernels' ring pattern
// of two in flight; W = 2: for a 128-thread epilogue group that waits each commit and then
// releases the accumulator, the kernels' tfull/tempty handshake) -- does the commit or its wait drain the tensor pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mma_commit mma_commit.cu && ./mma_commit
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (uint64_t)((lbo >> 4) & 0x3FFF) << 16 | (uint64_t)((sbo >> 4) & 0x3FFF) << 32 |
         (uint64_t)1 << 46 | (uint64_t)layout << 61;
}

template <int C>
__global__ void k(int iters, long long* out, int wait_prev) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2], tempty[2];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 100 * 1024; i += blockDim.x) base[i] = (uint8_t)(i * 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(smem_u32(&tempty[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(smem_u32(&tempty[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(base), b = smem_u32(base) + 48 * 1024;
    uint64_t ads[C], bds[C];
#pragma unroll
    for (int q = 0; q < C; q++) {
      ads[q] = desc(a + (q >> 1) * 2048 + (q & 1) * 32, 16, 1024, 2);
      bds[q] = desc(b + (q >> 1) * 4096 + (q & 1) * 32, 16, 1024, 2);
    }
    long long t0 = clock64();
    int n = 0;
    for (int it = 0; it < iters; it += C, n++) {
      if (wait_prev == 2 && n >= 2) {  // the epilogue group released the accumulator two back
        const uint32_t ph = ((n - 2) >> 1) & 1;
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(
                         smem_u32(&tempty[n & 1])),
                     "r"(ph), "r"(0x989680u)
                     : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;");
      } else if (wait_prev == 1 && n >= 2) {  // the commit of the group two back
        const uint32_t ph = ((n - 2) >> 1) & 1;
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(
                         smem_u32(&bar[n & 1])),
                     "r"(ph), "r"(0x989680u)
                     : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
#pragma unroll
      for (int q = 0; q < C; q++)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(
                         tm + (n & 1) * 128),
                     "l"(ads[q]), "l"(bds[q]), "r"(idesc), "r"(q));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[n & 1])));
    }
    const int last = n - 1;
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(
                     smem_u32(&bar[last & 1])),
                 "r"((last >> 1) & 1));
    out[blockIdx.x] = clock64() - t0;
  } else if (wait_prev == 2 && threadIdx.x >= 32) {
    // epilogue group (warps 1-3 + the rest of warp 0 would be irregular: use warps 1..4 -> 96 + 32)
  }
  if (wait_prev == 2 && threadIdx.x >= 32 && threadIdx.x < 160) {
    const int groups = iters / C;
    for (int n = 0; n < groups; n++) {
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(
                       smem_u32(&bar[n & 1])),
                   "r"((n >> 1) & 1), "r"(0x989680u)
                   : "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[n & 1])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int C>
void run(int wait_prev, long long* d) {
  cudaFuncSetAttribute(k<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  const int iters = C * 400;
  k<C><<<148, 160, 110 * 1024>>>(iters, d, wait_prev);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; i++) avg += h[i];
  avg /= 148;
  printf("commit every %2d MMAs, wait two back %d: %6.1f cycles/MMA %s\n", C, wait_prev, avg / iters,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  for (int w : {0, 1, 2}) {
    run<2>(w, d);
    run<4>(w, d);
    run<8>(w, d);
    run<10>(w, d);
    run<16>(w, d);
  }
}
