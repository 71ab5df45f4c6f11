// Probe: does cuTensorMapEncodeIm2col accept an overlapping W stride (16 B < 64 B pixel)?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap m, uint8_t* out, int w, int h, int n, int oh) {
  __shared__ __align__(1024) uint8_t buf[128 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    uint32_t b = __cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(128 * 64) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"((uint32_t)__cvta_generic_to_shared(buf)),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(b), "r"(0), "r"(w), "r"(h), "r"(n), "h"((uint16_t)0), "h"((uint16_t)oh)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(b)
        : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int N = 2, Uf = 10, Vf = 12, P = 7, Q = 9;  // folded 16-byte pixels; output P x Q
  std::vector<uint8_t> h(N * Uf * Vf * 16);
  for (size_t i = 0; i < h.size(); i++) h[i] = (uint8_t)(((uint32_t)i * 2654435761u) >> 13);
  uint8_t *d, *o;
  cudaMalloc(&d, h.size() + 4096);
  cudaMalloc(&o, 128 * 64);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
  CUtensorMap m;
  cuuint64_t dim[4] = {64, (cuuint64_t)Q, (cuuint64_t)Uf, (cuuint64_t)N};
  cuuint64_t str[3] = {16, Vf * 16, (cuuint64_t)Uf * Vf * 16};
  int lower[2] = {0, 0}, upper[2] = {0, -(Uf - P)};  // {W, H}?
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d, dim, str, lower, upper, 64, 128, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode im2col overlapping: %d\n", (int)r);
  if (r) return 1;
  // load starting at pixel (n=0, x=1, y=2) with tap row oh=2
  int x0 = 1, y0 = 2, oh = 2;
  k<<<1, 128>>>(m, o, y0, x0, 0, oh);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint8_t> got(128 * 64);
  cudaMemcpy(got.data(), o, got.size(), cudaMemcpyDeviceToHost);
  // expected: pixel p walks (y, x, n) over the P x Q output box
  int bad = 0, npix = 0;
  int x = x0, y = y0, n = 0;
  for (int p = 0; p < 128 && n < N; p++, npix++) {
    for (int c = 0; c < 64; c++) {
      size_t src = ((size_t)(n * Uf + x + oh) * Vf + y) * 16 + c;
      if (got[p * 64 + c] != h[src] && bad++ < 5) printf("p=%d (n%d x%d y%d) c=%d got %d want %d\n", p, n, x, y, c, got[p * 64 + c], h[src]);
    }
    if (++y == Q) { y = 0; if (++x == P) { x = 0; n++; } }
  }
  printf("checked %d pixels, bad=%d\n", npix, bad);
  for (int p = 0; p < 20; p++) { long f=-1; for (size_t s2=0; s2+64<=h.size(); s2++) { bool ok=true; for(int c=0;c<64&&ok;c++) ok = got[p*64+c]==h[s2+c]; if(ok){f=s2;break;} }
    printf("p=%d first=%d,%d src=%ld (pix %ld rem %ld)\n", p, got[p*64], got[p*64+1], f, f/16, f%16); }
  return 0;
}
