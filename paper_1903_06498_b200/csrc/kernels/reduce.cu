// Streaming reduce/copy kernel for the commonest memory-bound Stripe leaf:
//     $v = load(I); O = store($v)     with O:{assign,add,max,min,mul}
// (max-pool windows, global sums, copies, transposes of a contiguous dim), no
// constraints.  Owner computes (one thread = V consecutive outputs of the contiguous
// output dim, V = 16 bytes of input), the serial dims are walked in declaration order
// through a precomputed offset table in shared memory, accumulation stays in registers
// with the exact store-time wrap of the reference (ir.cpp:79-97), and the output is
// written once with vector stores.  When the output is a fresh prepare_outputs
// identity that this launch covers exactly once, the initial read is skipped.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <limits>

#include "../kernels.hpp"

namespace sb {
namespace {

template <typename T>
struct Vec16;  // 16-byte vector of T
template <>
struct Vec16<std::int8_t> {
  static constexpr int N = 16;
};
template <>
struct Vec16<std::int16_t> {
  static constexpr int N = 8;
};
template <>
struct Vec16<std::int32_t> {
  static constexpr int N = 4;
};

template <int AGG, typename TO>
__device__ __forceinline__ std::int64_t agg(std::int64_t cur, std::int64_t in) {
  // incoming is already a TI value; wrap to the output dtype first (ir.cpp:81)
  std::int64_t v = static_cast<TO>(in);
  if constexpr (AGG == 0) return v;
  if constexpr (AGG == 1) return static_cast<TO>(static_cast<std::uint64_t>(cur) + static_cast<std::uint64_t>(v));
  if constexpr (AGG == 2) return cur > v ? cur : v;
  if constexpr (AGG == 3) return cur < v ? cur : v;
  return static_cast<TO>(static_cast<std::uint64_t>(cur) * static_cast<std::uint64_t>(v));
}

template <typename TI>
__device__ __forceinline__ void load16(const TI* p, TI (&v)[Vec16<TI>::N]) {
  int4 w = __ldg(reinterpret_cast<const int4*>(p));
  const TI* s = reinterpret_cast<const TI*>(&w);
#pragma unroll
  for (int l = 0; l < Vec16<TI>::N; l++) v[l] = s[l];
}

template <int AGG, typename TI, typename TO>
__global__ void __launch_bounds__(256) reduce_kernel(const ReduceArgs a) {
  constexpr int V = Vec16<TI>::N;
  extern __shared__ std::int64_t roff[];  // input offset of every serial point, lex order
  for (int r = threadIdx.x; r < a.rcount; r += blockDim.x) {
    std::int64_t rest = r, off = 0;
    for (int i = a.nr - 1; i >= 0; i--) {
      off += (rest % a.rrange[i]) * a.rstep[i];
      rest /= a.rrange[i];
    }
    roff[r] = off;
  }
  __syncthreads();
  const TI* in = static_cast<const TI*>(a.in);
  TO* out = static_cast<TO*>(a.out);
  const std::int64_t nvec = a.prange[0] / V;
  const std::int64_t total = a.pcount / V;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t lin = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; lin < total;
       lin += stride) {
    std::int64_t rest = lin;
    std::int64_t c0 = (rest % nvec) * V;
    rest /= nvec;
    std::int64_t ib = a.in_c + c0, ob = a.out_c + c0;
    for (int i = 1; i < a.np; i++) {
      std::int64_t c = rest % a.prange[i];
      rest /= a.prange[i];
      ib += c * a.pin[i];
      ob += c * a.pout[i];
    }
    std::int64_t acc[V];
    if (a.fresh) {
#pragma unroll
      for (int l = 0; l < V; l++) acc[l] = a.identity;
    } else {
#pragma unroll
      for (int l = 0; l < V; l++) acc[l] = out[ob + l];
    }
    int r = 0;
    // four independent loads in flight per iteration
    for (; r + 3 < a.rcount; r += 4) {
      int4 w[4];
#pragma unroll
      for (int u = 0; u < 4; u++) w[u] = __ldg(reinterpret_cast<const int4*>(in + ib + roff[r + u]));
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const TI* x = reinterpret_cast<const TI*>(&w[u]);
#pragma unroll
        for (int l = 0; l < V; l++) acc[l] = agg<AGG, TO>(acc[l], x[l]);
      }
    }
    for (; r + 1 < a.rcount; r += 2) {
      TI x[V], y[V];
      load16<TI>(in + ib + roff[r], x);
      load16<TI>(in + ib + roff[r + 1], y);
#pragma unroll
      for (int l = 0; l < V; l++) acc[l] = agg<AGG, TO>(agg<AGG, TO>(acc[l], x[l]), y[l]);
    }
    if (r < a.rcount) {
      TI x[V];
      load16<TI>(in + ib + roff[r], x);
#pragma unroll
      for (int l = 0; l < V; l++) acc[l] = agg<AGG, TO>(acc[l], x[l]);
    }
    // V outputs = V * sizeof(TO) bytes, written as 16-byte stores
    constexpr int per16 = 16 / sizeof(TO);
#pragma unroll
    for (int q = 0; q < V / per16; q++) {
      int4 w;
      TO* s = reinterpret_cast<TO*>(&w);
#pragma unroll
      for (int l = 0; l < per16; l++) s[l] = static_cast<TO>(acc[q * per16 + l]);
      *reinterpret_cast<int4*>(out + ob + q * per16) = w;
    }
  }
}

// Short reductions (rcount <= 8: max-pool windows, small sums) over index spaces that fit
// 32 bits: 32-bit index math (64-bit div/mod costs several times the instructions the
// loads themselves take at 16 bytes per thread) and all rcount vector loads in flight before
// the fold.  The offsets come straight from the serial dims (no shared-memory table).
constexpr int kShortR = 8;

template <int AGG, typename TI, typename TO>
__global__ void __launch_bounds__(256) reduce_short_kernel(const ReduceArgs a) {
  constexpr int V = Vec16<TI>::N;
  int roff[kShortR];
#pragma unroll
  for (int r = 0; r < kShortR; r++) {
    int rest = r, off = 0;
    for (int i = a.nr - 1; i >= 0; i--) {
      off += (rest % static_cast<int>(a.rrange[i])) * static_cast<int>(a.rstep[i]);
      rest /= static_cast<int>(a.rrange[i]);
    }
    roff[r] = off;
  }
  const TI* in = static_cast<const TI*>(a.in);
  TO* out = static_cast<TO*>(a.out);
  const int nvec = static_cast<int>(a.prange[0] / V);
  const int total = static_cast<int>(a.pcount / V);
  for (int lin = blockIdx.x * blockDim.x + threadIdx.x; lin < total; lin += gridDim.x * blockDim.x) {
    int rest = lin / nvec;
    const int c0 = (lin - rest * nvec) * V;
    int ib = static_cast<int>(a.in_c) + c0, ob = static_cast<int>(a.out_c) + c0;
    for (int i = 1; i < a.np; i++) {
      const int pr = static_cast<int>(a.prange[i]);
      const int q = rest / pr;
      const int c = rest - q * pr;
      rest = q;
      ib += c * static_cast<int>(a.pin[i]);
      ob += c * static_cast<int>(a.pout[i]);
    }
    int4 w[kShortR];  // raw 16-byte vectors, all loads in flight before the fold
#pragma unroll
    for (int r = 0; r < kShortR; r++)
      if (r < a.rcount) w[r] = __ldg(reinterpret_cast<const int4*>(in + ib + roff[r]));
    std::int64_t acc[V];
#pragma unroll
    for (int l = 0; l < V; l++) acc[l] = a.fresh ? a.identity : static_cast<std::int64_t>(out[ob + l]);
#pragma unroll
    for (int r = 0; r < kShortR; r++)
      if (r < a.rcount) {
        const TI* x = reinterpret_cast<const TI*>(&w[r]);
#pragma unroll
        for (int l = 0; l < V; l++) acc[l] = agg<AGG, TO>(acc[l], x[l]);
      }
    constexpr int per16 = 16 / sizeof(TO);
#pragma unroll
    for (int q = 0; q < V / per16; q++) {
      int4 w;
      TO* st = reinterpret_cast<TO*>(&w);
#pragma unroll
      for (int l = 0; l < per16; l++) st[l] = static_cast<TO>(acc[q * per16 + l]);
      *reinterpret_cast<int4*>(out + ob + q * per16) = w;
    }
  }
}

// whether every index reduce_short_kernel forms fits a positive int
bool short_ok(const ReduceArgs& a, int V) {
  if (a.rcount < 1 || a.rcount > kShortR || std::getenv("SB_REDUCE_LONG")) return false;
  const std::int64_t lim = (1ll << 31) - 1;
  std::int64_t in_hi = a.in_c + a.prange[0], out_hi = a.out_c + a.prange[0], r_hi = 0;
  if (a.in_c < 0 || a.out_c < 0 || a.pcount / V > lim) return false;
  for (int i = 1; i < a.np; i++) {
    if (a.pin[i] < 0 || a.pout[i] < 0) return false;
    in_hi += (a.prange[i] - 1) * a.pin[i];
    out_hi += (a.prange[i] - 1) * a.pout[i];
  }
  for (int i = 0; i < a.nr; i++) {
    if (a.rstep[i] < 0) return false;
    r_hi += (a.rrange[i] - 1) * a.rstep[i];
  }
  return in_hi + r_hi + V < lim && out_hi + V < lim;
}

// Few outputs, long reductions (the ResNet global sum: 16K vectors x 49 rows): a block is 32
// output vectors x kSplit row phases; each thread folds rows r = phase (mod kSplit) into
// an identity-started accumulator, then the kSplit partials are folded in shared memory.
// add (wrapping), max, min and mul fold in any order to the same wrapped result, so this
// equals the reference's lexicographic sequence of wrapping stores.
constexpr int kSplit = 8;

template <int AGG, typename TO>
__device__ __forceinline__ std::int64_t agg_identity() {
  if constexpr (AGG == 1) return 0;
  if constexpr (AGG == 2) return static_cast<std::int64_t>(std::numeric_limits<TO>::min());
  if constexpr (AGG == 3) return static_cast<std::int64_t>(std::numeric_limits<TO>::max());
  return 1;
}

template <int AGG, typename TI, typename TO>
__global__ void __launch_bounds__(256) reduce_split_kernel(const ReduceArgs a) {
  constexpr int V = Vec16<TI>::N;
  extern __shared__ std::int64_t roff[];  // [rcount] offsets, then [256][V] partials
  for (int r = threadIdx.x; r < a.rcount; r += blockDim.x) {
    std::int64_t rest = r, off = 0;
    for (int i = a.nr - 1; i >= 0; i--) {
      off += (rest % a.rrange[i]) * a.rstep[i];
      rest /= a.rrange[i];
    }
    roff[r] = off;
  }
  std::int64_t* part = roff + ((a.rcount + 1) & ~1);
  __syncthreads();
  const TI* in = static_cast<const TI*>(a.in);
  TO* out = static_cast<TO*>(a.out);
  const std::int64_t nvec = a.prange[0] / V;
  const std::int64_t total = a.pcount / V;
  const int vi = threadIdx.x & 31, phase = threadIdx.x >> 5;
  for (std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * 32; base < total;
       base += static_cast<std::int64_t>(gridDim.x) * 32) {
    const std::int64_t lin = base + vi;
    const bool live = lin < total;
    std::int64_t ib = 0, ob = 0;
    if (live) {
      std::int64_t rest = lin;
      const std::int64_t c0 = (rest % nvec) * V;
      rest /= nvec;
      ib = a.in_c + c0;
      ob = a.out_c + c0;
      for (int i = 1; i < a.np; i++) {
        const std::int64_t c = rest % a.prange[i];
        rest /= a.prange[i];
        ib += c * a.pin[i];
        ob += c * a.pout[i];
      }
    }
    std::int64_t acc[V];
#pragma unroll
    for (int l = 0; l < V; l++) acc[l] = agg_identity<AGG, TO>();
    if (live) {
      // four rows of this phase per step, their loads in flight before the folds
      int r = phase;
      for (; r + 3 * kSplit < a.rcount; r += 4 * kSplit) {
        int4 w[4];
#pragma unroll
        for (int u = 0; u < 4; u++) w[u] = __ldg(reinterpret_cast<const int4*>(in + ib + roff[r + u * kSplit]));
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const TI* x = reinterpret_cast<const TI*>(&w[u]);
#pragma unroll
          for (int l = 0; l < V; l++) acc[l] = agg<AGG, TO>(acc[l], x[l]);
        }
      }
      for (; r < a.rcount; r += kSplit) {
        TI x[V];
        load16<TI>(in + ib + roff[r], x);
#pragma unroll
        for (int l = 0; l < V; l++) acc[l] = agg<AGG, TO>(acc[l], x[l]);
      }
    }
#pragma unroll
    for (int l = 0; l < V; l++) part[threadIdx.x * V + l] = acc[l];
    __syncthreads();
    if (phase == 0 && live) {
#pragma unroll
      for (int l = 0; l < V; l++) acc[l] = a.fresh ? a.identity : static_cast<std::int64_t>(out[ob + l]);
      for (int q = 0; q < kSplit; q++)
#pragma unroll
        for (int l = 0; l < V; l++) acc[l] = agg<AGG, TO>(acc[l], part[(q * 32 + vi) * V + l]);
      constexpr int per16 = 16 / sizeof(TO);
#pragma unroll
      for (int q = 0; q < V / per16; q++) {
        int4 w;
        TO* st = reinterpret_cast<TO*>(&w);
#pragma unroll
        for (int l = 0; l < per16; l++) st[l] = static_cast<TO>(acc[q * per16 + l]);
        *reinterpret_cast<int4*>(out + ob + q * per16) = w;
      }
    }
    __syncthreads();
  }
}

template <int AGG, typename TI>
cudaError_t dispatch_out(const ReduceArgs& a, int grid, std::size_t smem, cudaStream_t s) {
  const int V = Vec16<TI>::N;
  const std::int64_t vecs = a.pcount / V;
  // split the rows when the outputs alone cannot fill the GPU (assign stays sequential)
  if (AGG != 0 && a.rcount >= 2 * kSplit && a.rcount <= 1024 && vecs < 148ll * 256 * 2) {
    const int sgrid = static_cast<int>(std::min<std::int64_t>((vecs + 31) / 32, 148 * 8));
    const std::size_t ssmem = ((a.rcount + 1) & ~1) * sizeof(std::int64_t) + 256 * V * sizeof(std::int64_t);
    switch (a.out_kind) {
      case kI8: reduce_split_kernel<AGG, TI, std::int8_t><<<sgrid, 256, ssmem, s>>>(a); break;
      case kI16: reduce_split_kernel<AGG, TI, std::int16_t><<<sgrid, 256, ssmem, s>>>(a); break;
      default: reduce_split_kernel<AGG, TI, std::int32_t><<<sgrid, 256, ssmem, s>>>(a); break;
    }
    return cudaGetLastError();
  }
  if (short_ok(a, V)) {
    switch (a.out_kind) {
      case kI8: reduce_short_kernel<AGG, TI, std::int8_t><<<grid, 256, 0, s>>>(a); break;
      case kI16: reduce_short_kernel<AGG, TI, std::int16_t><<<grid, 256, 0, s>>>(a); break;
      default: reduce_short_kernel<AGG, TI, std::int32_t><<<grid, 256, 0, s>>>(a); break;
    }
    return cudaGetLastError();
  }
  switch (a.out_kind) {
    case kI8: reduce_kernel<AGG, TI, std::int8_t><<<grid, 256, smem, s>>>(a); break;
    case kI16: reduce_kernel<AGG, TI, std::int16_t><<<grid, 256, smem, s>>>(a); break;
    default: reduce_kernel<AGG, TI, std::int32_t><<<grid, 256, smem, s>>>(a); break;
  }
  return cudaGetLastError();
}

template <int AGG>
cudaError_t dispatch_in(const ReduceArgs& a, int grid, std::size_t smem, cudaStream_t s) {
  switch (a.in_kind) {
    case kI8: return dispatch_out<AGG, std::int8_t>(a, grid, smem, s);
    case kI16: return dispatch_out<AGG, std::int16_t>(a, grid, smem, s);
    default: return dispatch_out<AGG, std::int32_t>(a, grid, smem, s);
  }
}

}  // namespace

int reduce_vec_lanes(int in_kind) { return in_kind == kI8 ? 16 : in_kind == kI16 ? 8 : 4; }

cudaError_t launch_reduce(const ReduceArgs& a, cudaStream_t s) {
  const int V = reduce_vec_lanes(a.in_kind);
  std::int64_t threads = a.pcount / V;
  std::int64_t g = (threads + 255) / 256;
  // blocks per SM: 16 for the table-driven kernels; the short-window kernel (all loads of a
  // window in flight per thread) streams better with 8 (C4a 106 -> 103 us, tools/ab_steps.py)
  const int per_sm = std::getenv("SB_REDUCE_GRID") ? std::atoi(std::getenv("SB_REDUCE_GRID"))
                     : (a.rcount >= 1 && a.rcount <= kShortR) ? 8 : 16;
  const std::int64_t cap = 148ll * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  std::size_t smem = static_cast<std::size_t>(a.rcount) * sizeof(std::int64_t);
  switch (a.agg) {
    case 0: return dispatch_in<0>(a, static_cast<int>(g), smem, s);
    case 1: return dispatch_in<1>(a, static_cast<int>(g), smem, s);
    case 2: return dispatch_in<2>(a, static_cast<int>(g), smem, s);
    case 3: return dispatch_in<3>(a, static_cast<int>(g), smem, s);
    default: return dispatch_in<4>(a, static_cast<int>(g), smem, s);
  }
}

}  // namespace sb
