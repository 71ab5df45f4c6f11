// fp32 matmul leaves in the fp32 numeric mode (config 1 "fp32 matmul contraction",
// C[i,j] = +(A[i,k] * B[k,j])), bitwise equal to the CPU F32 policy of the port oracle.
//
// The reference's per-point semantics in float: for every output, in lexicographic k order,
// C = C + (A * B) with the product and the sum each rounded to fp32 (no FMA contraction;
// this file is compiled with -fmad=false and uses __fmul_rn/__fadd_rn explicitly).  A
// register-tiled SIMT kernel keeps exactly that order per output: each thread owns a 4x4
// block of C, starts from C's current value, and folds k = 0..K-1 in order.  Tiles are
// staged through shared memory (64 x 16 of A and 16 x 64 of B per step); the k loop never
// runs past K, so no padded +0 terms can flip the sign of a -0 accumulator.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../kernels.hpp"

namespace sb {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

struct F32Args {
  const float* a;
  const float* b;
  float* c;
  long long M, N, K;
  long long a_m, a_k, b_k, b_n, c_m, c_n;  // element strides
  int fresh;                                // C known zero-filled: start from +0
};

__global__ void __launch_bounds__(256) gemm_f32_exact_kernel(const F32Args p) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const long long m0 = static_cast<long long>(blockIdx.y) * TM, n0 = static_cast<long long>(blockIdx.x) * TN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const long long m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      acc[i][j] = (!p.fresh && m < p.M && n < p.N) ? p.c[m * p.c_m + n * p.c_n] : 0.0f;
    }
  for (long long k0 = 0; k0 < p.K; k0 += TK) {
    // stage A[m0 .. +64, k0 .. +16] and B[k0 .. +16, n0 .. +64] (4 elements per thread each)
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int e = threadIdx.x + 256 * r;
      const int am = e / TK, ak = e % TK;
      const long long gm = m0 + am, gk = k0 + ak;
      As[ak][am] = (gm < p.M && gk < p.K) ? p.a[gm * p.a_m + gk * p.a_k] : 0.0f;
      const int bk = e / TN, bn = e % TN;
      const long long gk2 = k0 + bk, gn = n0 + bn;
      Bs[bk][bn] = (gk2 < p.K && gn < p.N) ? p.b[gk2 * p.b_k + gn * p.b_n] : 0.0f;
    }
    __syncthreads();
    const int kn = static_cast<int>(p.K - k0 < TK ? p.K - k0 : TK);
    for (int kk = 0; kk < kn; kk++) {
      const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a4[4] = {av.x, av.y, av.z, av.w};
      const float b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a4[i], b4[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const long long m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < p.M && n < p.N) p.c[m * p.c_m + n * p.c_n] = acc[i][j];
    }
}

}  // namespace

cudaError_t launch_gemm_f32(const GemmPlan& g, const void* a, const void* b, void* c, cudaStream_t s) {
  F32Args p;
  p.a = static_cast<const float*>(a) + g.a0;
  p.b = static_cast<const float*>(b) + g.b0;
  p.c = static_cast<float*>(c) + g.c0;
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.a_m = g.lda;
  p.a_k = 1;
  if (g.b_kmajor) {
    p.b_k = 1;
    p.b_n = g.ldb;
  } else {
    p.b_k = g.ldb;
    p.b_n = 1;
  }
  p.c_m = g.ldc;
  p.c_n = 1;
  p.fresh = g.fresh ? 1 : 0;
  dim3 grid(static_cast<unsigned>((g.N + TN - 1) / TN), static_cast<unsigned>((g.M + TM - 1) / TM));
  gemm_f32_exact_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace sb
