// Does tcgen05.ld of one accumulator stall while tcgen05.mma writes another?  Warp 0 (one
// thread) issues `nmma` MMAs (M = 128, N = 64, K = 32, i8) into TMEM columns 0..63 and
// commits; warps 4..7 (one per TMEM lane quarter) time `nld` x16 loads + waits of columns
// 256..271 while those MMAs run, vs alone (nmma = 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o ldtm_mma ldtm_mma.cu && ./ldtm_mma
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

__global__ void k(int nmma, int nld, int N, long long* out, long long* mma_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int go;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) base[i] = (uint8_t)(i * 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    go = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0 && nmma > 0) {
    uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t ad = desc(smem_u32(base), 16, 1024, 2), bd = desc(smem_u32(base) + 64 * 1024, 16, 1024, 2);
    go = 1;
    const long long m0 = clock64();
    for (int it = 0; it < nmma; it++)
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(it));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(&bar)));
    mma_out[blockIdx.x] = clock64() - m0;
  }
  if (warp >= 4 && nld > 0) {
    if (nmma > 0)
      while (go == 0) {
      }
    const uint32_t ta = tm + (((warp & 3) * 32) << 16) + 256;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < nld; i++) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
          "tcgen05.wait::ld.sync.aligned;"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
            "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(ta + (i & 7) * 16));
      acc += v[0] ^ v[15];
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 4 + (warp & 3)] = (t1 - t0) + (acc == 12345 ? 1 : 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  long long *d, *dm;
  cudaMalloc(&d, 4096 * 8);
  cudaMalloc(&dm, 4096 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {64, 256})
    for (int nmma : {0, 2000}) {
      const int nld = 200;
      k<<<148, 256, 100 * 1024>>>(nmma, nld, N, d, dm);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148 * 4];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148 * 4; i++) avg += h[i];
      avg /= 148 * 4;
      printf("N=%3d MMAs running=%s: x16 tcgen05.ld + wait %.1f cycles  %s\n", N, nmma ? "yes" : "no ", avg / nld,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  // the other direction: MMA issue rate alone vs while four warps drain TMEM continuously
  for (int N : {64, 128, 256})
    for (int nld : {0, 100000}) {
      const int nmma = 4000;
      k<<<148, 256, 100 * 1024>>>(nmma, nld, N, d, dm);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, dm, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; i++) avg += h[i];
      avg /= 148;
      printf("N=%3d TMEM loads running=%s: %.1f cycles per MMA  %s\n", N, nld ? "yes" : "no ", avg / nmma,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
}
