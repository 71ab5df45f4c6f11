// Windowed max/min (pooling) leaf: O[n, x, y, c] = agg(O, I[n, sx*x + i, sy*y + j, c]) over the
// taps (i, j) the interval constraints admit (interp.cpp:426-428 skip predicates; the
// max-pool generator support.cpp:126-155 plus padding).  HBM-bound: one thread owns one
// 16-byte channel vector of one output pixel and folds the taps with SIMD max/min
// (__vmaxs4 / __vmaxs2 / max) in registers; overlapping windows are served from L1/L2.
// max/min are order-free, so the result equals the reference's lexicographic fold.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../kernels.hpp"

namespace sb {
namespace {

struct PoolArgs {
  long long N, H, W, CV;  // CV = channel vectors per pixel
  int R, S, sx, sy;
  long long a_n, a_x, a_y, a0;  // bytes
  long long o_n, o_x, o_y, o0;  // bytes
  int u_lo, u_hi, v_lo, v_hi;
};

template <int KIND, bool MAX>
__device__ __forceinline__ std::uint32_t fold(std::uint32_t a, std::uint32_t b) {
  if (KIND == kI8) return MAX ? __vmaxs4(a, b) : __vmins4(a, b);
  if (KIND == kI16) return MAX ? __vmaxs2(a, b) : __vmins2(a, b);
  const int x = static_cast<int>(a), y = static_cast<int>(b);
  return static_cast<std::uint32_t>(MAX ? (x < y ? y : x) : (y < x ? y : x));
}

template <int KIND, bool MAX>
__global__ void __launch_bounds__(256) pool_kernel(const std::uint8_t* __restrict__ in, std::uint8_t* __restrict__ out,
                                                   const PoolArgs p) {
  const long long total = p.N * p.H * p.W * p.CV;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long cv = g % p.CV;
    long long pix = g / p.CV;
    const int y = static_cast<int>(pix % p.W);
    pix /= p.W;
    const int x = static_cast<int>(pix % p.H);
    const long long n = pix / p.H;
    uint4* o = reinterpret_cast<uint4*>(out + p.o0 + p.o_n * n + p.o_x * x + p.o_y * y + cv * 16);
    uint4 acc = *o;
    const std::uint8_t* ib = in + p.a0 + p.a_n * n + cv * 16;
    const int u0 = p.sx * x, v0 = p.sy * y;
    for (int i = 0; i < p.R; i++) {
      const int u = u0 + i;
      if (u < p.u_lo || u > p.u_hi) continue;
      for (int j = 0; j < p.S; j++) {
        const int v = v0 + j;
        if (v < p.v_lo || v > p.v_hi) continue;
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(ib + p.a_x * u + p.a_y * v));
        acc.x = fold<KIND, MAX>(acc.x, t.x);
        acc.y = fold<KIND, MAX>(acc.y, t.y);
        acc.z = fold<KIND, MAX>(acc.z, t.z);
        acc.w = fold<KIND, MAX>(acc.w, t.w);
      }
    }
    *o = acc;
  }
}

int esize(int kind) { return kind == kI8 ? 1 : kind == kI16 ? 2 : 4; }

}  // namespace

const char* pool_unsupported(const PoolPlan& pp) {
  const int lanes = 16 / esize(pp.kind);
  if (pp.C % lanes) return "channels not a multiple of one 16-byte vector";
  if (pp.a_n % lanes || pp.a_x % lanes || pp.a_y % lanes || pp.a0 % lanes || pp.o_n % lanes || pp.o_x % lanes ||
      pp.o_y % lanes || pp.o0 % lanes)
    return "pixel strides not 16-byte multiples";
  if (pp.R > 64 || pp.S > 64) return "window too large";
  if (pp.u_hi >= (1ll << 30) || pp.v_hi >= (1ll << 30) || pp.u_lo <= -(1ll << 30) || pp.v_lo <= -(1ll << 30))
    return "window bounds out of range";
  return nullptr;
}

cudaError_t launch_pool(const PoolPlan& pp, const void* in, void* out, cudaStream_t s) {
  const int es = esize(pp.kind);
  PoolArgs a;
  a.N = pp.N;
  a.H = pp.H;
  a.W = pp.W;
  a.CV = pp.C * es / 16;
  a.R = static_cast<int>(pp.R);
  a.S = static_cast<int>(pp.S);
  a.sx = static_cast<int>(pp.sx);
  a.sy = static_cast<int>(pp.sy);
  a.a_n = pp.a_n * es;
  a.a_x = pp.a_x * es;
  a.a_y = pp.a_y * es;
  a.a0 = pp.a0 * es;
  a.o_n = pp.o_n * es;
  a.o_x = pp.o_x * es;
  a.o_y = pp.o_y * es;
  a.o0 = pp.o0 * es;
  a.u_lo = static_cast<int>(pp.u_lo);
  a.u_hi = static_cast<int>(pp.u_hi);
  a.v_lo = static_cast<int>(pp.v_lo);
  a.v_hi = static_cast<int>(pp.v_hi);
  const long long total = a.N * a.H * a.W * a.CV;
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 148 * 16)));
  const auto* i = static_cast<const std::uint8_t*>(in);
  auto* o = static_cast<std::uint8_t*>(out);
  const bool mx = pp.agg == static_cast<int>(Agg::Max);
  switch (pp.kind) {
    case kI8: mx ? pool_kernel<kI8, true><<<grid, 256, 0, s>>>(i, o, a) : pool_kernel<kI8, false><<<grid, 256, 0, s>>>(i, o, a); break;
    case kI16: mx ? pool_kernel<kI16, true><<<grid, 256, 0, s>>>(i, o, a) : pool_kernel<kI16, false><<<grid, 256, 0, s>>>(i, o, a); break;
    default: mx ? pool_kernel<kI32, true><<<grid, 256, 0, s>>>(i, o, a) : pool_kernel<kI32, false><<<grid, 256, 0, s>>>(i, o, a); break;
  }
  return cudaGetLastError();
}

}  // namespace sb
