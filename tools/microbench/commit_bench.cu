// How long does one thread take per tcgen05.commit (no MMAs in flight), and per
// mbarrier.arrive, in a loop?  148 CTAs, one issuing thread each.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int mode, int iters, long long* out) {
  __shared__ __align__(8) uint64_t bar[16];
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(1 << 20));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      uint64_t* b = &bar[it & 15];
      if (mode == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
      else if (mode == 1)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
      else if (mode == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
      } else {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(0) : "memory");
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(32));
}
int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int mode = 0; mode < 4; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      int iters = 4096;
      k<<<148, 64>>>(mode, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; i++) avg += h[i];
      avg /= 148;
      if (rep) printf("mode %d (%s): %.1f cycles per op %s\n", mode,
                      mode == 0 ? "tcgen05.commit" : mode == 1 ? "mbarrier.arrive" : mode == 2 ? "fence+commit" : "arrive.expect_tx",
                      avg / iters, e ? cudaGetErrorString(e) : "");
    }
  }
}
