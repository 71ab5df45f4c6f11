// tcgen05.mma kind::i8 issue rate, one CTA (cta_group::1, M = 128) vs a CTA pair
// (cta_group::2, M = 256: each SM's 128 rows from its own smem, the leader issues).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mma_pair mma_pair.cu && ./mma_pair
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

template <int PAIR>
__global__ void k(int iters, int N, long long* out, int sw64, int vary) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 120 * 1024; i += blockDim.x) base[i] = (uint8_t)(i * 7);
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = slot;
  const uint32_t M = PAIR ? 256 : 128;
  uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24);
  if (threadIdx.x == 0 && rank == 0) {
    uint32_t a = smem_u32(base);
    uint32_t b = smem_u32(base) + 40 * 1024;
    uint64_t bd = sw64 ? desc(b, 16, 512, 4) : desc(b, 16, 1024, 2);
    uint64_t ad = sw64 ? desc(a, 16, 512, 4) : desc(a, 16, 1024, 2);
    // eight descriptor pairs (the same one, or different 4 KB A / 8 KB B slices), issued as an
    // unrolled run of eight so the issuing thread spends no instructions between MMAs
    uint64_t ads[8], bds[8];
    for (int q = 0; q < 8; q++) {
      const uint32_t ao = vary ? q * 4096 : 0, bo = vary ? (q & 3) * 8192 : 0;
      ads[q] = sw64 ? desc(a + ao, 16, 512, 4) : desc(a + ao, 16, 1024, 2);
      bds[q] = sw64 ? desc(b + bo, 16, 512, 4) : desc(b + bo, 16, 1024, 2);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int q = 0; q < 8; q++) {
        if (PAIR)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                       "l"(ads[q]), "l"(bds[q]), "r"(idesc), "r"(it + q));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                       "l"(ads[q]), "l"(bds[q]), "r"(idesc), "r"(it + q));
      }
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                       smem_u32(&bar)), "h"((uint16_t)3));
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (PAIR && threadIdx.x == 0 && rank == 1)
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaMemset(d, 0, 1024 * 8);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  for (int pair : {0, 1})
    for (int N : {64, 128, 256})
    for (int sw64 : {0, 1})
    for (int vary : {0, 1}) {
      if (pair && (sw64 || vary)) continue;
      const int iters = 4000;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = 128 * 1024;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = pair ? 2 : 1;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaMemset(d, 0, 1024 * 8);
      cudaError_t e = pair ? cudaLaunchKernelEx(&cfg, k<1>, iters, N, d, sw64, vary)
                           : cudaLaunchKernelEx(&cfg, k<0>, iters, N, d, sw64, vary);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      int n = 0;
      for (int i = 0; i < 148; i++)
        if (h[i]) {
          avg += h[i];
          n++;
        }
      avg /= n > 0 ? n : 1;
      const double macs = (pair ? 256.0 : 128.0) * N * 32;
      printf("%s M=%d N=%3d %s %s: %6.1f cycles/MMA, %5.0f MAC/cyc per SM  %s\n", pair ? "pair" : "single", pair ? 256 : 128, N,
             sw64 ? "SW64 " : "SW128", vary ? "varying operands" : "same operands   ",
             avg / iters, macs / (avg / iters) / (pair ? 2 : 1), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
}
