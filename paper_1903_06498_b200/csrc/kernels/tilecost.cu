// Distinct cache lines per tile, for every line residue at once (the
// inner loop of the reference's tile_cost, tile.cpp:413-453, and so of its autotile search,
// tile.cpp:475-535).
//
// The reference enumerates a refinement's tile elements F (tile_elements_of, tile.cpp:239-336)
// and, per distinct tile base residue r = base mod L, inserts floor((r + f) / L) for every f
// into a std::set.  Here one CTA owns one (candidate, refinement) item:
//   1. F is generated as a sum of "axes" (a constant plus one value from each axis list; the
//      host builds the lists, duplicates are harmless because only the line SET matters).  A
//      unit-step last axis is a run: each prefix then marks one interval instead of n points.
//   2. For every fine line q = floor(f / L) present, keep min and max of m = f mod L (shared
//      memory, or a global scratch slab when the span is too wide).
//   3. Line q is touched at residue r iff min_m(q) < L - r (r + m stays in line q) or
//      max_m(q - 1) >= L - r (r + m spills from q - 1 into q): residues [0, a) U [b, L) with
//      a = L - min_m(q), b = L - max_m(q - 1).  A difference array over r gives all L counts
//      in one pass over q, so no residue needs its own enumeration.
// Exact: the count per residue equals the size of the reference's set.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../kernels.hpp"

namespace sb {
namespace {

constexpr int kThreads = 512;
constexpr int kSmemQ = 12288;  // q slots held in shared memory (2 x 48 KB)

__device__ __forceinline__ long long fdiv(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}

__global__ void __launch_bounds__(kThreads) tile_lines_kernel(const TileLineItem* __restrict__ items,
                                                              const long long* __restrict__ values,
                                                              unsigned* __restrict__ scratch,
                                                              long long* __restrict__ counts, int first, int L) {
  extern __shared__ unsigned sm[];
  const TileLineItem it = items[first + blockIdx.x];
  unsigned* mn = it.scratch_off < 0 ? sm : scratch + it.scratch_off;
  unsigned* mx = mn + it.nq;
  int* diff = reinterpret_cast<int*>(sm + 2 * kSmemQ);
  const unsigned UL = static_cast<unsigned>(L);
  for (int q = threadIdx.x; q < it.nq; q += blockDim.x) {
    mn[q] = UL;  // absent: a = 0
    mx[q] = 0;   // absent (or max 0): b = L
  }
  for (int r = threadIdx.x; r <= L; r += blockDim.x) diff[r] = 0;
  __syncthreads();

  const long long* vals = values + it.val_off;
  const int np = it.run ? it.naxes - 1 : it.naxes;  // axes decoded per prefix
  for (long long p = threadIdx.x; p < it.prefixes; p += blockDim.x) {
    long long f = it.cst, rest = p;
    int off = 0;
    for (int a = 0; a < np; a++) {
      const int n = it.len[a];
      f += vals[off + static_cast<int>(rest % n)];
      rest /= n;
      off += n;
    }
    if (!it.run) {
      const long long qa = fdiv(f, L);
      const int q = static_cast<int>(qa - it.qbase);
      const unsigned m = static_cast<unsigned>(f - qa * L);
      atomicMin(&mn[q], m);
      atomicMax(&mx[q], m);
    } else {
      const long long lo = f + vals[off], hi = lo + it.len[np] - 1;
      const long long q0 = fdiv(lo, L), q1 = fdiv(hi, L);
      const unsigned m0 = static_cast<unsigned>(lo - q0 * L), m1 = static_cast<unsigned>(hi - q1 * L);
      for (long long qa = q0; qa <= q1; qa++) {
        const int q = static_cast<int>(qa - it.qbase);
        atomicMin(&mn[q], qa == q0 ? m0 : 0u);
        atomicMax(&mx[q], qa == q1 ? m1 : UL - 1);
      }
    }
  }
  __syncthreads();

  // lines q' = 0 .. nq (q' = nq only takes spill from q' - 1)
  for (int q = threadIdx.x; q <= it.nq; q += blockDim.x) {
    const int a = q < it.nq ? L - static_cast<int>(mn[q]) : 0;
    const int b = q > 0 ? L - static_cast<int>(mx[q - 1]) : L;
    if (a >= b) {
      atomicAdd(&diff[0], 1);
      atomicAdd(&diff[L], -1);
    } else {
      if (a > 0) {
        atomicAdd(&diff[0], 1);
        atomicAdd(&diff[a], -1);
      }
      if (b < L) {
        atomicAdd(&diff[b], 1);
        atomicAdd(&diff[L], -1);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    long long* out = counts + static_cast<long long>(first + blockIdx.x) * L;
    for (int r = 0; r < L; r++) {
      run += diff[r];
      out[r] = run;
    }
  }
}

}  // namespace

int tile_lines_smem_q() { return kSmemQ; }

cudaError_t launch_tile_lines(const std::vector<TileLineItem>& items, const std::vector<long long>& values,
                              long long scratch_words, int L, std::vector<long long>* counts, cudaStream_t s) {
  counts->assign(items.size() * static_cast<std::size_t>(L), 0);
  if (items.empty()) return cudaSuccess;
  const std::size_t smem = (2 * kSmemQ + L + 1) * sizeof(unsigned);
  static bool attr = false;
  cudaError_t e;
  if (!attr) {
    if ((e = cudaFuncSetAttribute(tile_lines_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)) !=
        cudaSuccess)
      return e;
    attr = true;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  TileLineItem* d_items = nullptr;
  long long *d_vals = nullptr, *d_counts = nullptr;
  unsigned* d_scratch = nullptr;
  auto cleanup = [&] {
    cudaFreeAsync(d_items, s);
    cudaFreeAsync(d_vals, s);
    cudaFreeAsync(d_counts, s);
    if (d_scratch) cudaFreeAsync(d_scratch, s);
  };
  if ((e = cudaMallocAsync(&d_items, items.size() * sizeof(TileLineItem), s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&d_vals, std::max<std::size_t>(values.size(), 1) * sizeof(long long), s)) != cudaSuccess ||
      (e = cudaMallocAsync(&d_counts, counts->size() * sizeof(long long), s)) != cudaSuccess ||
      (scratch_words > 0 &&
       (e = cudaMallocAsync(&d_scratch, static_cast<std::size_t>(scratch_words) * sizeof(unsigned), s)) != cudaSuccess)) {
    cleanup();
    return e;
  }
  if ((e = cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(TileLineItem), cudaMemcpyHostToDevice, s)) !=
          cudaSuccess ||
      (!values.empty() && (e = cudaMemcpyAsync(d_vals, values.data(), values.size() * sizeof(long long),
                                               cudaMemcpyHostToDevice, s)) != cudaSuccess)) {
    cleanup();
    return e;
  }
  const int n = static_cast<int>(items.size());
  for (int first = 0; first < n; first += 65535) {
    const int cnt = std::min(65535, n - first);
    tile_lines_kernel<<<cnt, kThreads, smem, s>>>(d_items, d_vals, d_scratch, d_counts, first, L);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      cleanup();
      return e;
    }
  }
  e = cudaMemcpyAsync(counts->data(), d_counts, counts->size() * sizeof(long long), cudaMemcpyDeviceToHost, s);
  cleanup();
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

}  // namespace sb
