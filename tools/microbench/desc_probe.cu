// Probe of the tcgen05 K-major SWIZZLE_NONE shared-memory descriptor (i8, M = 128, N = 32,
// K = 32): A is a 16 KB smem region whose byte at offset o holds (o >> 4) & 0x7F (the 16-byte
// unit index) or o & 15 (the byte within the unit); B is the 128B-swizzled identity (row n has
// its 1 at byte n), so D[m][n] = the A byte the MMA reads for row m, k = n.  Prints, per
// descriptor variant, the 16-byte unit and byte offset read for rows 0..17 at k = 0, 8, 16, 24.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o desc_probe desc_probe.cu && ./desc_probe
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ std::uint32_t su32(const void* p) { return static_cast<std::uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(int* out, std::uint32_t lo_lbo, std::uint32_t hi_sbo, int mode, int start) {
  extern __shared__ __align__(1024) std::uint8_t sm[];
  std::uint8_t* A = sm;                 // 16 KB
  std::uint8_t* B = sm + 16384;         // 128 rows x 128 B identity (SW128)
  __shared__ std::uint64_t bar;
  __shared__ std::uint32_t tslot;
  for (int o = threadIdx.x; o < 16384; o += blockDim.x) A[o] = mode ? (o & 15) : ((o >> 4) & 0x7F);
  for (int u = threadIdx.x; u < 1024; u += blockDim.x) {
    const int n = u >> 3, unit = (u & 7) ^ (n & 7);
    std::uint32_t w[4] = {0, 0, 0, 0};
    if (unit == (n >> 4)) w[(n & 15) >> 2] = 1u << (8 * (n & 3));
    reinterpret_cast<uint4*>(B)[u] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const std::uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const std::uint32_t a_lo = ((su32(A) + start) >> 4) | (lo_lbo << 16), a_hi = hi_sbo | (1u << 14);
    const std::uint32_t b_lo = (su32(B) >> 4) | (1u << 16), b_hi = (1024u >> 4) | (1u << 14) | (2u << 29);
    // kind::i8, S32 accumulate, A/B unsigned, K-major, N = 32, M = 128
    const std::uint32_t idesc = (2u << 4) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    asm volatile(
        "{\n\t.reg .b64 da, db;\n\tmov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, 0;\n\t}" ::"r"(tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  std::uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tmem + ((warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int q = 0; q < 32; q++) out[(warp * 32 + lane) * 32 + q] = static_cast<int>(v[q]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  int* d;
  cudaMalloc(&d, 128 * 32 * 4);
  static int h[2][128 * 32];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const std::uint32_t variants[][3] = {{1, 8, 0}, {8, 1, 0}, {1, 16, 0}, {16, 1, 0}, {1, 8, 48}, {1, 8, 176},
                                       {1, 8, 16}, {1, 8, 128}, {1, 8, 352}};
  for (auto& vr : variants) {
    for (int mode = 0; mode < 2; mode++) {
      probe<<<1, 128, 48 * 1024>>>(d, vr[0], vr[1], mode, static_cast<int>(vr[2]));
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { std::printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h[mode], d, sizeof(h[mode]), cudaMemcpyDeviceToHost);
    }
    std::printf("LBO(lo)=%u B, SBO(hi)=%u B, start +%u: row m -> A offset (unit*16+byte) at k = 0, 8, 16, 24\n", vr[0] * 16,
                vr[1] * 16, vr[2]);
    for (int m = 0; m < 18; m++) {
      std::printf("  m=%2d:", m);
      for (int k = 0; k < 32; k += 8) std::printf(" %5d", h[0][m * 32 + k] * 16 + h[1][m * 32 + k]);
      std::printf("\n");
    }
  }
  return 0;
}
