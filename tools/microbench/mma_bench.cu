// Microbenchmark: tcgen05.mma kind::i8 issue throughput for several smem layouts / N.
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

__global__ void k(int iters, int N, int lbo_a, int sbo_a, int layout, int shift, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) base[i] = (uint8_t)i;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
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
    uint32_t a = smem_u32(base) + shift;
    uint32_t b = smem_u32(base) + 64 * 1024;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      uint64_t ad = desc(a + (it & 7) * 16 * (layout == 0 ? 1 : 0), lbo_a, sbo_a, layout);
      uint64_t bd = desc(b, (uint32_t)N * 16, 128, 0);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(it));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  struct Cfg { const char* name; int N, lbo, sbo, layout, shift; } cfgs[] = {
      {"noswz lbo=4096 N=64", 64, 4096, 128, 0, 0},
      {"noswz lbo=128  N=64", 64, 128, 256, 0, 0},
      {"noswz lbo=4096 N=128", 128, 4096, 128, 0, 0},
      {"noswz lbo=4096 N=256", 256, 4096, 128, 0, 0},
      {"sw128 N=64", 64, 16, 1024, 2, 0},
      {"sw128 N=256", 256, 16, 1024, 2, 0},
      {"sw64 N=64 (rows 64B)", 64, 16, 512, 4, 0},
      {"sw64 N=64 shift 64B", 64, 16, 512, 4, 64},
  };
  for (auto& c : cfgs) {
    int iters = 2000;
    for (int grid : {1, 148}) {
      k<<<grid, 128, 100 * 1024>>>(iters, c.N, c.lbo, c.sbo, c.layout, c.shift, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < grid; i++) avg += h[i];
      avg /= grid;
      printf("%-26s grid %3d: %7.1f cycles/MMA  (ideal %d)  %s\n", c.name, grid, avg / iters, 128 * c.N / 256,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
}
