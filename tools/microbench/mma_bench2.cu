// tcgen05.mma kind::i8 issue rate: dependent vs independent accumulators, A in smem vs TMEM.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

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

__global__ void k(int iters, int N, int naccs, int a_tmem, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) base[i] = (uint8_t)(i * 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
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
    uint32_t b = smem_u32(base) + 64 * 1024;
    uint64_t bd = desc(b, 16, 1024, 2);
    uint64_t ad = desc(a, 16, 1024, 2);
    long long t0 = clock64();
    const uint32_t at = tm + 448;
    uint32_t d0 = tm, d1 = tm + (naccs > 1 ? N : 0), d2 = tm + (naccs > 2 ? 2 * N : 0), d3 = tm + (naccs > 2 ? 3 * N : (naccs > 1 ? N : 0));
#define MMA_SS(D, ACC) asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(D), "l"(ad), "l"(bd), "r"(idesc), "r"(ACC))
#define MMA_TS(D, ACC) asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(D), "r"(at), "l"(bd), "r"(idesc), "r"(ACC))
    if (a_tmem) {
      for (int it = 0; it < iters; it += 4) { MMA_TS(d0, it); MMA_TS(d1, it); MMA_TS(d2, it); MMA_TS(d3, it); }
    } else {
      for (int it = 0; it < iters; it += 4) { MMA_SS(d0, it); MMA_SS(d1, it); MMA_SS(d2, it); MMA_SS(d3, it); }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int a_tmem : {0, 1})
    for (int N : {64, 128, 256})
      for (int naccs : {1, 2, 4}) {
        if (N * naccs > 448) continue;
        int iters = 4000;
        k<<<148, 128, 100 * 1024>>>(iters, N, naccs, a_tmem, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; i++) avg += h[i];
        avg /= 148;
        printf("A_%s N=%3d accs=%d: %6.1f cycles/MMA  (%5.0f MAC/cyc)  %s\n", a_tmem ? "tmem" : "smem", N, naccs,
               avg / iters, 128.0 * N * 32 / (avg / iters), e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
}
