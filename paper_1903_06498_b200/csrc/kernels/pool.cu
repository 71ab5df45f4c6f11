// Windowed max/min (pooling) leaf: O[n, x, y, c] = agg(O, I[n, sx*x + i, sy*y + j, c]) over the
// taps (i, j) the interval constraints admit (interp.cpp:426-428 skip predicates; the
// max-pool generator support.cpp:126-155 plus padding).  HBM-bound: one thread owns one
// 16-byte channel vector of one output pixel and folds the taps with SIMD max/min
// (__vmaxs4 / __vmaxs2 / max) in registers; overlapping windows are served from L1/L2.
// max/min are order-free, so the result equals the reference's lexicographic fold.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "../kernels.hpp"

namespace sb {
namespace {

struct PoolArgs {
  long long N, H, W, CV;  // CV = channel vectors per pixel
  int R, S, sx, sy;
  long long a_n, a_x, a_y, a0;  // bytes
  long long o_n, o_x, o_y, o0;  // bytes
  int u_lo, u_hi, v_lo, v_hi;
  int fresh;           // start from init (the elided fill) instead of reading the output
  std::uint32_t init;  // fill value replicated over the 4-byte lane word
};

template <int KIND, bool MAX>
__device__ __forceinline__ std::uint32_t fold(std::uint32_t a, std::uint32_t b) {
  if (KIND == kI8) return MAX ? __vmaxs4(a, b) : __vmins4(a, b);
  if (KIND == kI16) return MAX ? __vmaxs2(a, b) : __vmins2(a, b);
  const int x = static_cast<int>(a), y = static_cast<int>(b);
  return static_cast<std::uint32_t>(MAX ? (x < y ? y : x) : (y < x ? y : x));
}

// i8 lanes as two sign-extended s16x2 halves (even bytes | odd bytes): packed max/min of bytes
// has no instruction, max.s16x2 does -- two prmt + two max per 4-byte word instead of the
// ~13-instruction byte emulation
__device__ __forceinline__ std::uint32_t sx_even(std::uint32_t w) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0xA280;" : "=r"(r) : "r"(w));
  return r;
}
__device__ __forceinline__ std::uint32_t sx_odd(std::uint32_t w) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0xB391;" : "=r"(r) : "r"(w));
  return r;
}
template <bool MAX>
__device__ __forceinline__ std::uint32_t mm16x2(std::uint32_t a, std::uint32_t b) {
  std::uint32_t r;
  if (MAX) asm("max.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  else asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

template <int KIND, bool MAX, typename IDX>
__global__ void __launch_bounds__(256) pool_kernel(const std::uint8_t* __restrict__ in, std::uint8_t* __restrict__ out,
                                                   const PoolArgs p) {
  // IDX = int when the index space fits (32-bit division is several times cheaper)
  const IDX total = static_cast<IDX>(p.N * p.H * p.W * p.CV);
  const IDX CV = static_cast<IDX>(p.CV), W = static_cast<IDX>(p.W), H = static_cast<IDX>(p.H);
  for (IDX g = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<IDX>(gridDim.x) * blockDim.x) {
    const IDX pix0 = g / CV, cv = g - pix0 * CV;
    const IDX pix1 = pix0 / W;
    const int y = static_cast<int>(pix0 - pix1 * W);
    const IDX n = pix1 / H;
    const int x = static_cast<int>(pix1 - n * H);
    uint4* o = reinterpret_cast<uint4*>(out + p.o0 + p.o_n * n + p.o_x * x + p.o_y * y + cv * 16);
    uint4 acc = p.fresh ? make_uint4(p.init, p.init, p.init, p.init) : *o;
    std::uint32_t ev[4], od[4];  // i8: the accumulator as s16x2 halves
    if (KIND == kI8) {
      const std::uint32_t a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int q = 0; q < 4; q++) {
        ev[q] = sx_even(a4[q]);
        od[q] = sx_odd(a4[q]);
      }
    }
    const std::uint8_t* ib = in + p.a0 + p.a_n * n + cv * 16;
    const int u0 = p.sx * x, v0 = p.sy * y;
    auto fold_tap = [&](const uint4 t) {
      if (KIND == kI8) {
        const std::uint32_t t4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          ev[q] = mm16x2<MAX>(ev[q], sx_even(t4[q]));
          od[q] = mm16x2<MAX>(od[q], sx_odd(t4[q]));
        }
      } else {
        acc.x = fold<KIND, MAX>(acc.x, t.x);
        acc.y = fold<KIND, MAX>(acc.y, t.y);
        acc.z = fold<KIND, MAX>(acc.z, t.z);
        acc.w = fold<KIND, MAX>(acc.w, t.w);
      }
    };
    if (p.R == 3 && p.S == 3) {
      // the common 3x3 window: all nine loads in flight before the folds (memory-level parallelism)
      uint4 t[9];
      bool ok[9];
#pragma unroll
      for (int k = 0; k < 9; k++) {
        const int u = u0 + k / 3, v = v0 + k % 3;
        ok[k] = u >= p.u_lo && u <= p.u_hi && v >= p.v_lo && v <= p.v_hi;
        t[k] = ok[k] ? __ldg(reinterpret_cast<const uint4*>(ib + p.a_x * u + p.a_y * v)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < 9; k++)
        if (ok[k]) fold_tap(t[k]);
    } else {
      for (int i = 0; i < p.R; i++) {
        const int u = u0 + i;
        if (u < p.u_lo || u > p.u_hi) continue;
        for (int j = 0; j < p.S; j++) {
          const int v = v0 + j;
          if (v < p.v_lo || v > p.v_hi) continue;
          fold_tap(__ldg(reinterpret_cast<const uint4*>(ib + p.a_x * u + p.a_y * v)));
        }
      }
    }
    if (KIND == kI8) {
      std::uint32_t r[4];
#pragma unroll
      for (int q = 0; q < 4; q++) r[q] = __byte_perm(ev[q], od[q], 0x6240);
      acc = make_uint4(r[0], r[1], r[2], r[3]);
    }
    *o = acc;
  }
}

// 3x3 / stride-2 windows (the ResNet stem pool): one thread folds a horizontal PAIR of output
// pixels (y0, y0 + 1) of one channel vector; their windows share the middle column, so 15
// vector loads (all in flight) serve 2 outputs instead of 18 -- a sixth less L1/L2 traffic.
template <int KIND, bool MAX, typename IDX>
__global__ void __launch_bounds__(256) pool_pair_kernel(const std::uint8_t* __restrict__ in, std::uint8_t* __restrict__ out,
                                                        const PoolArgs p) {
  const IDX CV = static_cast<IDX>(p.CV), W2 = static_cast<IDX>((p.W + 1) / 2), H = static_cast<IDX>(p.H);
  const IDX total = static_cast<IDX>(p.N) * H * W2 * CV;
  for (IDX g = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<IDX>(gridDim.x) * blockDim.x) {
    const IDX q0 = g / CV, cv = g - q0 * CV;
    const IDX q1 = q0 / W2;
    const int y0 = 2 * static_cast<int>(q0 - q1 * W2);
    const IDX n = q1 / H;
    const int x = static_cast<int>(q1 - n * H);
    const bool two = y0 + 1 < p.W;
    uint4* o0 = reinterpret_cast<uint4*>(out + p.o0 + p.o_n * n + p.o_x * x + p.o_y * y0 + cv * 16);
    uint4* o1 = reinterpret_cast<uint4*>(reinterpret_cast<std::uint8_t*>(o0) + p.o_y);
    uint4 acc[2] = {p.fresh ? make_uint4(p.init, p.init, p.init, p.init) : *o0,
                    p.fresh || !two ? make_uint4(p.init, p.init, p.init, p.init) : *o1};
    std::uint32_t ev[2][4], od[2][4];
    if (KIND == kI8) {
#pragma unroll
      for (int a = 0; a < 2; a++) {
        const std::uint32_t a4[4] = {acc[a].x, acc[a].y, acc[a].z, acc[a].w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          ev[a][q] = sx_even(a4[q]);
          od[a][q] = sx_odd(a4[q]);
        }
      }
    }
    auto fold_tap = [&](int a, const uint4 t) {
      if (KIND == kI8) {
        const std::uint32_t t4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          ev[a][q] = mm16x2<MAX>(ev[a][q], sx_even(t4[q]));
          od[a][q] = mm16x2<MAX>(od[a][q], sx_odd(t4[q]));
        }
      } else {
        acc[a].x = fold<KIND, MAX>(acc[a].x, t.x);
        acc[a].y = fold<KIND, MAX>(acc[a].y, t.y);
        acc[a].z = fold<KIND, MAX>(acc[a].z, t.z);
        acc[a].w = fold<KIND, MAX>(acc[a].w, t.w);
      }
    };
    const std::uint8_t* ib = in + p.a0 + p.a_n * n + cv * 16;
    const int u0 = 2 * x, v0 = 2 * y0;
    uint4 t[15];
    bool ok[15];
#pragma unroll
    for (int k = 0; k < 15; k++) {
      const int u = u0 + k / 5, v = v0 + k % 5;
      ok[k] = u >= p.u_lo && u <= p.u_hi && v >= p.v_lo && v <= p.v_hi && (k % 5 < 3 || two);
      t[k] = ok[k] ? __ldg(reinterpret_cast<const uint4*>(ib + p.a_x * u + p.a_y * v)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 15; k++) {
      if (!ok[k]) continue;
      if (k % 5 <= 2) fold_tap(0, t[k]);
      if (k % 5 >= 2) fold_tap(1, t[k]);
    }
#pragma unroll
    for (int a = 0; a < 2; a++) {
      if (KIND == kI8) {
        std::uint32_t r[4];
#pragma unroll
        for (int q = 0; q < 4; q++) r[q] = __byte_perm(ev[a][q], od[a][q], 0x6240);
        acc[a] = make_uint4(r[0], r[1], r[2], r[3]);
      }
    }
    *o0 = acc[0];
    if (two) *o1 = acc[1];
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
  a.fresh = pp.fresh ? 1 : 0;
  {
    const std::uint32_t v = static_cast<std::uint32_t>(pp.fill_value);
    a.init = es == 1 ? (v & 0xFFu) * 0x01010101u : es == 2 ? (v & 0xFFFFu) * 0x00010001u : v;
  }
  const long long total = a.N * a.H * a.W * a.CV;
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 148 * 16)));
  const auto* i = static_cast<const std::uint8_t*>(in);
  auto* o = static_cast<std::uint8_t*>(out);
  const bool mx = pp.agg == static_cast<int>(Agg::Max);
  const bool small = total < (1ll << 31) - 148ll * 16 * 256;
  if (pp.R == 3 && pp.S == 3 && pp.sx == 2 && pp.sy == 2 && !std::getenv("SB_POOL_SINGLE")) {
    const long long pairs = a.N * a.H * ((a.W + 1) / 2) * a.CV;
    const int pgrid = static_cast<int>(std::max<long long>(1, std::min<long long>((pairs + 255) / 256, 148 * 16)));
    const auto* i = static_cast<const std::uint8_t*>(in);
    auto* o = static_cast<std::uint8_t*>(out);
    const bool mx = pp.agg == static_cast<int>(Agg::Max);
#define SB_POOL2(K, M)                                                                      \
  (small ? pool_pair_kernel<K, M, int><<<pgrid, 256, 0, s>>>(i, o, a)                      \
         : pool_pair_kernel<K, M, long long><<<pgrid, 256, 0, s>>>(i, o, a))
    switch (pp.kind) {
      case kI8: mx ? SB_POOL2(kI8, true) : SB_POOL2(kI8, false); break;
      case kI16: mx ? SB_POOL2(kI16, true) : SB_POOL2(kI16, false); break;
      default: mx ? SB_POOL2(kI32, true) : SB_POOL2(kI32, false); break;
    }
#undef SB_POOL2
    return cudaGetLastError();
  }
#define SB_POOL(K, M)                                                                      \
  (small ? pool_kernel<K, M, int><<<grid, 256, 0, s>>>(i, o, a)                           \
         : pool_kernel<K, M, long long><<<grid, 256, 0, s>>>(i, o, a))
  switch (pp.kind) {
    case kI8: mx ? SB_POOL(kI8, true) : SB_POOL(kI8, false); break;
    case kI16: mx ? SB_POOL(kI16, true) : SB_POOL(kI16, false); break;
    default: mx ? SB_POOL(kI32, true) : SB_POOL(kI32, false); break;
  }
#undef SB_POOL
  return cudaGetLastError();
}

}  // namespace sb
