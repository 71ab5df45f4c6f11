// Constraint-satisfying point count of one block: the reference's
// count_valid_points (tile.cpp:338-370) enumerates every point on one CPU thread (~60-130
// ns/point: minutes at config scale, which is what makes its autotile search infeasible).
// Here one thread owns one "row" of the innermost index: every constraint is affine in that
// index, so its valid values form an interval computed in closed form, and the row's count
// is the length of the intersection.  Rows are reduced with a warp shuffle + one atomic per
// warp.  Exact: the same set of points as the reference's odometer.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../kernels.hpp"

namespace sb {
namespace {

constexpr int kMaxCountDims = 24, kMaxCountCons = 32;

struct CountArgs {
  int nd, nc;
  long long range[kMaxCountDims];
  long long c[kMaxCountCons];
  long long k[kMaxCountCons][kMaxCountDims];
  long long rows;  // product of all ranges but the last
};

__device__ __forceinline__ long long floor_div(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}

__global__ void __launch_bounds__(256) count_points_kernel(const CountArgs* __restrict__ A,
                                                           unsigned long long* out) {
  const CountArgs& a = *A;
  const int last = a.nd - 1;
  const long long r_last = a.range[last];
  unsigned long long mine = 0;
  for (long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; row < a.rows;
       row += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long coord[kMaxCountDims];
    long long rest = row;
    for (int d = last - 1; d >= 0; d--) {
      coord[d] = rest % a.range[d];
      rest /= a.range[d];
    }
    long long lo = 0, hi = r_last - 1;
    for (int c = 0; c < a.nc && lo <= hi; c++) {
      long long v = a.c[c];
      for (int d = 0; d < last; d++) v += a.k[c][d] * coord[d];
      const long long kl = a.k[c][last];
      if (kl == 0) {
        if (v < 0) hi = lo - 1;
      } else if (kl > 0) {
        lo = max(lo, -floor_div(v, kl));  // v + kl*t >= 0  <=>  t >= ceil(-v/kl)
      } else {
        hi = min(hi, floor_div(v, -kl));  // v + kl*t >= 0  <=>  t <= floor(v/-kl)
      }
    }
    if (hi >= lo) mine += static_cast<unsigned long long>(hi - lo + 1);
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(out, mine);
}

}  // namespace

cudaError_t launch_count_points(int nd, const long long* ranges, int nc, const long long* cons_c,
                                const long long* cons_k, void* scratch, unsigned long long* h_out, cudaStream_t s) {
  if (nd < 1 || nd > kMaxCountDims || nc > kMaxCountCons) return cudaErrorInvalidValue;
  CountArgs a{};
  a.nd = nd;
  a.nc = nc;
  a.rows = 1;
  for (int d = 0; d < nd; d++) {
    a.range[d] = ranges[d];
    if (d < nd - 1) a.rows *= ranges[d];
  }
  for (int c = 0; c < nc; c++) {
    a.c[c] = cons_c[c];
    for (int d = 0; d < nd; d++) a.k[c][d] = cons_k[c * nd + d];
  }
  auto* d_args = static_cast<CountArgs*>(scratch);
  auto* d_out = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + sizeof(CountArgs));
  cudaError_t e = cudaMemcpyAsync(d_args, &a, sizeof(a), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(d_out, 0, sizeof(*d_out), s)) != cudaSuccess) return e;
  const long long blocks = std::min<long long>((a.rows + 255) / 256, 148 * 16);
  count_points_kernel<<<static_cast<int>(std::max<long long>(blocks, 1)), 256, 0, s>>>(d_args, d_out);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(h_out, d_out, sizeof(*d_out), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

std::size_t count_points_scratch_bytes() { return sizeof(CountArgs) + 16; }

}  // namespace sb
