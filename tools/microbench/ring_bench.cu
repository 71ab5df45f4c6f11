// Producer/consumer mbarrier ring: producer (warp 0) waits empty[s] then arrives full[s];
// consumer (warp 1) waits full[s] then releases empty[s] by tcgen05.commit (mode 0) or a
// plain mbarrier.arrive (mode 1).  Cycles per ring step, 148 CTAs.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph, int hint) {
  if (hint == 2)
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE_%=;\nbra "
        "WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
  else if (hint == 3)
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE_%=;\nbra "
        "WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
  else if (hint)
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@P1 bra DONE_%=;\nbra "
        "WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(b)),
        "r"(ph), "r"(0x989680u)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE_%=;\nbra "
        "WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
}
__global__ void k(int mode, int stages, int iters, int hint, long long* out) {
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; it++) {
      wait(&empty[s], ph ^ 1, hint);
      if (mode == 2)
        asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      if (++s == stages) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; it++) {
      wait(&full[s], ph, hint);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (mode == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[s]))
                     : "memory");
      else if (mode == 2)
        asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      if (++s == stages) {
        s = 0;
        ph ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(32));
  }
}
int main(int argc, char** argv) {
  int mode = atoi(argv[1]), stages = atoi(argv[2]), hint = argc > 3 ? atoi(argv[3]) : 1;
  long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int rep = 0; rep < 2; rep++) {
    int iters = 4096;
    k<<<148, 64>>>(mode, stages, iters, hint, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; i++) avg += h[i];
    avg /= 148;
    if (rep)
      printf("release by %s, %2d stages, hint %d: %.1f cycles per step %s\n", mode == 0 ? "tcgen05.commit" : mode == 1 ? "arrive" : "arrive.relaxed", stages,
             hint, avg / iters, e ? cudaGetErrorString(e) : "");
  }
}
