// tcgen05 GEMM for Stripe matmul-shaped contraction blocks (K3):
//     $a = load(A); $b = load(B); $p = mul($a, $b); C = store($p)   C:add
// with i8 operands: C[m, n] (+)= sum_k A[m, k] * B[k, n]  (gen_matmul, support.cpp:50-77;
// matmul64.stripe).  A is K-major (k contiguous), B either N-major (n contiguous, the
// reference generator's layout) or K-major.
//
// B200 mapping: persistent CTAs over 128x128 output tiles; warp 0 = TMA producer
// (128-byte-swizzled boxes: A 128 m x 128 k, B 128 k x 128 n or 128 n x 128 k), 4-stage
// mbarrier ring; warp 1 = one thread issuing tcgen05.mma.cta_group::1.kind::i8 (M=128,
// N=128, K=32 per instruction); warps 2-5 = epilogue: tcgen05.ld -> registers ->
// 128B-swizzled smem -> TMA tensor store (out-of-range rows/cols clipped), or a direct
// read-modify-write when the output accumulates into existing contents.  TMA zero-fill
// of the K tail contributes exact zeros.  Exactness: s32 accumulation with
// K * 128 * 128 < 2^31 (checked by the planner) equals the reference's int64 sum.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../kernels.hpp"

namespace sb {
namespace {

constexpr int kThreads = 192;
constexpr int kStages = 4;  // ring depth of 128-wide tiles (3 for 256-wide tiles: same smem)
constexpr int BM = 128, BN = 128, BK = 128;
constexpr std::uint32_t kStageA = BM * BK;  // bytes (i8); a B stage is BK * bn

struct GemmKParams {
  int M, N, K;
  int tiles_m, tiles_n, kblocks;
  int b_kmajor;
  int fresh, tma_out, out_kind;
  void* c;
  long long ldc;  // elements
  std::uint32_t idesc;
  int pdl, b_early;
  int tf32;  // kind::tf32 (fp32 accumulators, f32 output)
  int bk_el;  // k-block width in elements (128 bytes)
  int pdl_wait;
  // split-K over a CTA pair (cluster of 2, opt-in): rank r runs k-blocks [r * kb_per, (r + 1) * kb_per);
  // rank 1 parks its partial tile in its own staging buffer, rank 0 adds it over DSMEM in the
  // epilogue and stores the sum (no zero fill, no atomics, no second pass)
  int ksplit, kb_per;
  // tile width 128 or 256 (N = 256 MMAs: 85 instead of 64 MACs per staged byte, for problems
  // with at least two 128 x 256 tiles per SM), ring depth
  int bn, stages;
};

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(std::uint32_t dst, const CUtensorMap* map, std::uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_i8(std::uint32_t d, std::uint32_t a_lo, std::uint32_t a_hi, std::uint32_t b_lo,
                                        std::uint32_t b_hi, std::uint32_t idesc, std::uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %2};\n\t"
      "mov.b64 db, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, p;\n\t}" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_tf32(std::uint32_t d, std::uint32_t a_lo, std::uint32_t a_hi, std::uint32_t b_lo,
                                          std::uint32_t b_hi, std::uint32_t idesc, std::uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %2};\n\t"
      "mov.b64 db, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t}" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, std::uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16_async(std::uint32_t taddr, std::uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ std::uint32_t cluster_rank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ std::uint32_t cluster_id() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ std::uint32_t cluster_count() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of this CTA's shared variable `a` in cluster CTA `rank`
__device__ __forceinline__ std::uint32_t peer_addr(std::uint32_t a, std::uint32_t rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_peer(std::uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONEC_%=;\n\t"
      "bra WAITC_%=;\n\t"
      "DONEC_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ bool elect_one_sync() {
  std::uint32_t is;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(is));
  return is != 0;
}

// SWIZZLE_128B descriptors (version 1, layout 2 in bits 61-63).
// K-major: rows of 128 B, 8-row atoms (SBO = 1024 B), LBO unused (16 B).
// MN-major: 128-element MN rows per k, 8-k-row atoms (SBO = 1024 B), LBO = next 128-element MN block.
constexpr std::uint32_t kHiSW128 = (1024u >> 4) | (1u << 14) | (2u << 29);

__global__ void __launch_bounds__(kThreads, 1)
    gemm_i8_tc_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                      const __grid_constant__ CUtensorMap cmap, const GemmKParams p) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* base =
      reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
  const int bn = p.bn, nst = p.stages;
  const std::uint32_t stage_b = static_cast<std::uint32_t>(BK * bn);
  std::uint8_t* sa = base;                              // stages x 16 KB
  std::uint8_t* sbm = sa + nst * kStageA;               // stages x (16 | 32) KB
  std::uint8_t* stg = sbm + nst * stage_b;              // 64 KB output staging (4 x 16 KB column quarters)
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(stg + BM * 128 * 4);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + kStages;
  std::uint64_t* tfull = bars + 2 * kStages;
  std::uint64_t* tempty = bars + 2 * kStages + 2;
  std::uint64_t* peer_full = bars + 2 * kStages + 4;   // rank 0: rank 1's partial tile is staged
  std::uint64_t* peer_empty = bars + 2 * kStages + 5;  // rank 1: rank 0 has read it
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * kStages + 6);
  const std::uint32_t tmem_cols = static_cast<std::uint32_t>(2 * bn);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles = p.tiles_m * p.tiles_n;
  const bool split = p.ksplit > 1;
  const std::uint32_t rank = split ? cluster_rank() : 0;
  const int t_first = split ? static_cast<int>(cluster_id()) : static_cast<int>(blockIdx.x);
  const int t_step = split ? static_cast<int>(cluster_count()) : static_cast<int>(gridDim.x);
  const int kb_lo = split ? static_cast<int>(rank) * p.kb_per : 0;
  const int kb_hi = split ? min(p.kblocks, kb_lo + p.kb_per) : p.kblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    mbar_init(peer_full, 128);
    mbar_init(peer_empty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (split) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  const std::uint32_t tmem_base = *tmem_slot;
  // dependents are released after this grid's wait (see conv_tc.cu)
  if (p.pdl && !p.pdl_wait && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      if (p.pdl_wait) asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
      int stage = 0;
      std::uint32_t phase = 0;
      for (int t = t_first; t < tiles; t += t_step) {
        const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * bn;
        for (int kb = kb_lo; kb < kb_hi; kb++) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kStageA + stage_b);
          tma_load_2d(smem_u32(sa + stage * kStageA), &amap, &full[stage], kb * p.bk_el, m0);
          if (p.b_kmajor) {
            tma_load_2d(smem_u32(sbm + stage * stage_b), &bmap, &full[stage], kb * p.bk_el, n0);
          } else {  // 128-element MN blocks of BK k-rows each (LBO = 16 KB in the descriptor)
            for (int j = 0; j < bn / 128; j++)
              tma_load_2d(smem_u32(sbm + stage * stage_b + j * 16384), &bmap, &full[stage], n0 + j * 128, kb * p.bk_el);
          }
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0, iter = 0;
      std::uint32_t phase = 0;
      for (int t = t_first; t < tiles; t += t_step, iter++) {
        const int acc = iter & 1;
        mbar_wait(&tempty[acc], ((iter >> 1) & 1) ^ 1);
        tc_fence_after();
        const std::uint32_t d = tmem_base + static_cast<std::uint32_t>(acc * bn);
        for (int kb = kb_lo; kb < kb_hi; kb++) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const std::uint32_t a0 = (smem_u32(sa + stage * kStageA) >> 4) | (1u << 16);
          const std::uint32_t bsm = smem_u32(sbm + stage * stage_b);
#pragma unroll
          for (int ks = 0; ks < BK / 32; ks++) {
            // A: +32 bytes along the 128-byte K row; B: K-major +32 bytes, N-major +32 rows (4 KB)
            std::uint32_t b_lo = p.b_kmajor ? (((bsm + ks * 32) >> 4) | (1u << 16))
                                            : (((bsm + ks * 32 * 128) >> 4) | ((static_cast<std::uint32_t>(BK * 128) >> 4) << 16));
            const std::uint32_t accum = (kb != kb_lo || ks != 0) ? 1u : 0u;
            if (p.tf32) umma_tf32(d, a0 + ks * 2, kHiSW128, b_lo, kHiSW128, p.idesc, accum);
            else umma_i8(d, a0 + ks * 2, kHiSW128, b_lo, kHiSW128, p.idesc, accum);
          }
          umma_commit(&empty[stage]);
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const bool leader = threadIdx.x == 64;
    int iter = 0;
    for (int t = t_first; t < tiles; t += t_step, iter++) {
      const int acc = iter & 1;
      const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * bn;
      if (split && rank == 1) {
        // park the partial tile in the own staging buffer (same swizzled layout rank 0 uses)
        if (iter > 0) mbar_wait_cluster(peer_empty, (iter - 1) & 1);
        mbar_wait(&tfull[acc], (iter >> 1) & 1);
        tc_fence_after();
        for (int h = 0; h < BN / 32; h++) {
          std::uint32_t v[32];
          tmem_ld32(tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) +
                        static_cast<std::uint32_t>(acc * bn + h * 32),
                    v);
          const std::uint32_t rbase = smem_u32(stg + h * 16384 + row * 128);
#pragma unroll
          for (int q = 0; q < 8; q++)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((q ^ (row & 7)) << 4)),
                         "r"(v[4 * q]), "r"(v[4 * q + 1]), "r"(v[4 * q + 2]), "r"(v[4 * q + 3]));
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        mbar_arrive_peer(peer_addr(smem_u32(peer_full), 0));
        continue;
      }
      if (p.tma_out) {
        if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      mbar_wait(&tfull[acc], (iter >> 1) & 1);
      tc_fence_after();
      for (int h = 0; h < bn / 32; h++) {
        std::uint32_t v[32];
        tmem_ld32(tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) + static_cast<std::uint32_t>(acc * bn + h * 32),
                  v);
        if (p.tma_out && h > 0 && (h & 3) == 0) {
          // 256-wide tiles: the first 128 columns go out before the staging is reused
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (leader) {
            for (int q = 0; q < 4; q++)
              asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                               reinterpret_cast<std::uint64_t>(&cmap)),
                           "r"(smem_u32(stg + q * 16384)), "r"(n0 + (h - 4 + q) * 32), "r"(m0)
                           : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        if (p.tma_out) {
          std::uint32_t rbase = smem_u32(stg + (h & 3) * 16384 + row * 128);
          if (split) {  // + rank 1's partial, read over DSMEM at the same swizzled address
            if (h == 0) mbar_wait_cluster(peer_full, iter & 1);
            const std::uint32_t pbase = peer_addr(rbase, 1);
#pragma unroll
            for (int q = 0; q < 8; q++) {
              std::uint32_t w0, w1, w2, w3;
              asm volatile("ld.shared::cluster.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                           : "r"(pbase + ((q ^ (row & 7)) << 4)));
              v[4 * q] += w0;
              v[4 * q + 1] += w1;
              v[4 * q + 2] += w2;
              v[4 * q + 3] += w3;
            }
            if (h == BN / 32 - 1) mbar_arrive_peer(peer_addr(smem_u32(peer_empty), 1));
          }
#pragma unroll
          for (int q = 0; q < 8; q++)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((q ^ (row & 7)) << 4)),
                         "r"(v[4 * q]), "r"(v[4 * q + 1]), "r"(v[4 * q + 2]), "r"(v[4 * q + 3]));
        } else if (m0 + row < p.M) {
          for (int q = 0; q < 32; q++) {
            int n = n0 + h * 32 + q;
            if (n >= p.N) break;
            long long idx = static_cast<long long>(m0 + row) * p.ldc + n;
            if (p.tf32) {
              float* o = static_cast<float*>(p.c) + idx;
              *o = p.fresh ? __uint_as_float(v[q]) : *o + __uint_as_float(v[q]);
            } else if (p.out_kind == kI32) {
              std::int32_t* o = static_cast<std::int32_t*>(p.c) + idx;
              *o = static_cast<std::int32_t>(p.fresh ? v[q] : static_cast<std::uint32_t>(*o) + v[q]);
            } else if (p.out_kind == kI16) {
              std::int16_t* o = static_cast<std::int16_t*>(p.c) + idx;
              *o = static_cast<std::int16_t>(p.fresh ? v[q] : static_cast<std::uint32_t>(*o) + v[q]);
            } else {
              std::int8_t* o = static_cast<std::int8_t*>(p.c) + idx;
              *o = static_cast<std::int8_t>(p.fresh ? v[q] : static_cast<std::uint32_t>(*o) + v[q]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (p.tma_out) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (leader) {
          const int hq0 = bn / 32 - 4;  // the last 128 columns are still staged
          for (int q = 0; q < 4; q++)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                             reinterpret_cast<std::uint64_t>(&cmap)),
                         "r"(smem_u32(stg + q * 16384)), "r"(n0 + (hq0 + q) * 32), "r"(m0)
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (p.tma_out && leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    // rank 1 stays resident until rank 0 has read its last partial tile
    if (split && rank == 1 && iter > 0) mbar_wait_cluster(peer_empty, (iter - 1) & 1);
  }
  __syncwarp();  // reconverge the single-lane role warps before the CTA barrier
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

std::size_t smem_bytes(int bn, int stages) { return 1024 + stages * (kStageA + BK * bn) + BM * 128 * 4 + 256; }
constexpr std::size_t kSmemMax = 1024 + 3 * (BM * BK + BK * 256) + BM * 128 * 4 + 256;

struct Prepared {
  GemmPlan gp;
  const void *a, *b;
  void* c;
  GemmKParams kp;
  CUtensorMap amap, bmap, cmap;
};

bool same(const GemmPlan& x, const GemmPlan& y) {
  return std::memcmp(&x.M, &y.M, sizeof(long long) * 9) == 0 && x.b_kmajor == y.b_kmajor && x.fresh == y.fresh &&
         x.c_dtype == y.c_dtype && x.unsigned_ab == y.unsigned_ab && x.tf32x3 == y.tf32x3;
}

std::mutex g_mu;
std::vector<Prepared>* g_prep = nullptr;

cudaError_t prepare(const GemmPlan& g, const GemmArgs& args, Prepared* out, int num_sms) {
  out->gp = g;
  out->a = args.a;
  out->b = args.b;
  out->c = args.c;
  auto encode = get_encode();
  if (!encode) return cudaErrorNotSupported;
  GemmKParams& kp = out->kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.M = static_cast<int>(g.M);
  kp.N = static_cast<int>(g.N);
  kp.K = static_cast<int>(g.K);
  const int es_ab = g.tf32x3 ? 4 : 1;  // operand element bytes; a k-block is always 128 bytes
  const int bk_el = BK / es_ab;
  kp.tf32 = g.tf32x3 ? 1 : 0;
  kp.bk_el = bk_el;
  kp.tiles_m = static_cast<int>((g.M + BM - 1) / BM);
  // 256-wide tiles when every SM still gets at least two of them (SB_GEMM_BN=128|256 forces)
  const long long wide_tiles = static_cast<long long>(kp.tiles_m) * ((g.N + 255) / 256);
  kp.bn = !g.tf32x3 && g.N >= 256 && wide_tiles >= 2ll * num_sms ? 256 : 128;
  if (const char* f = std::getenv("SB_GEMM_BN")) kp.bn = !g.tf32x3 && std::atoi(f) == 256 ? 256 : 128;
  kp.stages = kp.bn == 256 ? 3 : kStages;
  kp.tiles_n = static_cast<int>((g.N + kp.bn - 1) / kp.bn);
  kp.kblocks = static_cast<int>((g.K + bk_el - 1) / bk_el);
  kp.b_kmajor = g.b_kmajor ? 1 : 0;
  kp.fresh = g.fresh ? 1 : 0;
  kp.out_kind = g.c_dtype == DType::I8 ? kI8 : g.c_dtype == DType::I16 ? kI16 : kI32;  // F32: 32-bit
  kp.ldc = g.ldc;
  kp.c = static_cast<char*>(args.c) + g.c0 * (kp.out_kind == kI8 ? 1 : kp.out_kind == kI16 ? 2 : 4);
  kp.tma_out = kp.fresh && kp.out_kind == kI32 && g.ldc % 4 == 0 &&
               reinterpret_cast<std::uintptr_t>(kp.c) % 16 == 0;
  // idesc: S32 accumulate, signed A/B, A K-major, B K- or MN-major, N = 128, M = 128
  const std::uint32_t sgn = g.unsigned_ab ? 0u : 1u;  // atype/btype: 0 = U8, 1 = S8
  kp.idesc = (2u << 4) | (sgn << 7) | (sgn << 10) | ((kp.b_kmajor ? 0u : 1u) << 16) |
             ((static_cast<std::uint32_t>(kp.bn) >> 3) << 17) | ((128u >> 4) << 24);
  if (g.tf32x3)  // D = F32 (1), A = B = TF32 (2), both K-major
    kp.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  const CUtensorMapDataType ttype = g.tf32x3 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  cuuint32_t es[2] = {1, 1};
  const std::int8_t* a = static_cast<const std::int8_t*>(args.a) + g.a0 * es_ab;
  const std::int8_t* b = static_cast<const std::int8_t*>(args.b) + g.b0 * es_ab;
  if (reinterpret_cast<std::uintptr_t>(a) % 16 || reinterpret_cast<std::uintptr_t>(b) % 16) return cudaErrorMisalignedAddress;
  cuuint64_t adim[2] = {static_cast<cuuint64_t>(g.K), static_cast<cuuint64_t>(g.M)};
  cuuint64_t astr[1] = {static_cast<cuuint64_t>(g.lda * es_ab)};
  cuuint32_t abox[2] = {static_cast<cuuint32_t>(bk_el), BM};
  if (encode(&out->amap, ttype, 2, const_cast<std::int8_t*>(a), adim, astr, abox, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  cuuint64_t bdim[2], bstr[1] = {static_cast<cuuint64_t>(g.ldb * es_ab)};
  cuuint32_t bbox[2];
  if (g.b_kmajor) {
    bdim[0] = static_cast<cuuint64_t>(g.K);
    bdim[1] = static_cast<cuuint64_t>(g.N);
    bbox[0] = static_cast<cuuint32_t>(bk_el);
    bbox[1] = static_cast<cuuint32_t>(kp.bn);
  } else {  // 128-element MN boxes (one 128-byte swizzle span); 256-wide tiles load two
    bdim[0] = static_cast<cuuint64_t>(g.N);
    bdim[1] = static_cast<cuuint64_t>(g.K);
    bbox[0] = 128;
    bbox[1] = BK;
  }
  if (encode(&out->bmap, ttype, 2, const_cast<std::int8_t*>(b), bdim, bstr, bbox, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  std::memset(&out->cmap, 0, sizeof(out->cmap));
  if (kp.tma_out) {
    cuuint64_t cdim[2] = {static_cast<cuuint64_t>(g.N), static_cast<cuuint64_t>(g.M)};
    cuuint64_t cstr[1] = {static_cast<cuuint64_t>(g.ldc * 4)};
    cuuint32_t cbox[2] = {32, BM};
    if (encode(&out->cmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, kp.c, cdim, cstr, cbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(std::max(kSmemMax, smem_bytes(128, kStages))));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return cudaSuccess;
}

}  // namespace

const char* gemm_tc_unsupported(const GemmPlan& g) {
  if (g.limbs_a) {
    if (g.K % 16 || (!g.b_kmajor && g.N % 16)) return "limb planes need 16-byte rows";
    for (int s = 0; s <= limb_smax(g); s++)
      if (const char* e = gemm_tc_unsupported(limb_sum_plan(g, s))) return e;
    return nullptr;
  }
  const long long amax = g.unsigned_ab ? 255 * 255 : 128 * 128;
  if (g.K * amax >= (1ll << 31)) return "reduction too long for exact s32 accumulation";
  if (g.lda % 16 || g.ldb % 16 || g.a0 % 16 || g.b0 % 16) return "operand rows not 16-byte aligned";
  if (g.M < 1 || g.N < 1 || g.K < 1) return "empty";
  if (g.lda < g.K || (g.b_kmajor ? g.ldb < g.K : g.ldb < g.N)) return "overlapping operand rows";
  return nullptr;
}

// ---- byte-limb mode ------------------------------------------------------------------------

// Offsets (bytes) of sum s's concatenated A / B operands inside the plane buffers.
long long limb_a_off(const GemmPlan& g, int s) {
  long long o = 0;
  for (int t = 0; t < s; t++) o += static_cast<long long>(limb_pairs(g, t)) * g.M * g.K;
  return o;
}
long long limb_b_off(const GemmPlan& g, int s) {
  long long o = 0;
  for (int t = 0; t < s; t++) o += static_cast<long long>(limb_pairs(g, t)) * g.K * g.N;
  return o;
}

namespace {

__device__ __forceinline__ std::uint32_t elem_bits(const void* p, int kind, long long i) {
  if (kind == kI8) return static_cast<std::uint32_t>(static_cast<const std::int8_t*>(p)[i]);
  if (kind == kI16) return static_cast<std::uint32_t>(static_cast<const std::int16_t*>(p)[i]);
  return static_cast<std::uint32_t>(static_cast<const std::int32_t*>(p)[i]);
}

struct SplitArgs {
  const void* src;
  std::uint8_t* dst;
  int kind, limbs, smax, lb_other;  // lb_other: limbs of the other operand
  long long rows, cols, ld, off;    // source matrix rows x cols (cols contiguous), element strides
  long long pair_stride;            // bytes between pair segments inside one concatenated row/col
  long long dst_ld;                 // bytes per destination row
  int is_a, kcat_cols;              // A: pairs concatenate along cols (k); B: along rows or cols
  long long sum_off[4];             // byte offset of each sum's operand
  int pairs[4];
};

// Every source element's limb i goes to each sum s whose pair list contains it.  One thread
// per 4 consecutive columns: limb i of the 4 elements is one 32-bit word, stored once per
// (s, pair) segment it belongs to (cols % 4 == 0, 16-byte aligned plane rows).
__global__ void limb_split_kernel(SplitArgs a) {
  const long long cq = a.cols / 4;
  const long long total = a.rows * cq;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = g / cq, c = (g - r * cq) * 4;
    std::uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; e++) v[e] = elem_bits(a.src, a.kind, a.off + r * a.ld + c + e);
    std::uint32_t limb[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const unsigned sel = static_cast<unsigned>(i | ((4 + i) << 4));  // [x.byte i, y.byte i]
      limb[i] = __byte_perm(__byte_perm(v[0], v[1], sel), __byte_perm(v[2], v[3], sel), 0x5410);
    }
    for (int s = 0; s <= a.smax; s++) {
      int p = 0;
      for (int i = 0; i <= s; i++) {
        const int j = s - i;
        if (i >= (a.is_a ? a.limbs : a.lb_other) || j >= (a.is_a ? a.lb_other : a.limbs)) continue;
        const int mine = a.is_a ? i : j;
        long long idx;
        if (a.kcat_cols) idx = r * (a.pairs[s] * a.cols) + p * a.cols + c;  // [rows][pairs * cols]
        else idx = (p * a.rows + r) * a.cols + c;                          // [pairs * rows][cols]
        *reinterpret_cast<std::uint32_t*>(a.dst + a.sum_off[s] + idx) = limb[mine];
        p++;
      }
    }
  }
}

__global__ void limb_combine_kernel(const std::int32_t* __restrict__ sums, void* c, int smax, long long M, long long N,
                                    long long ldc, int out_kind, int fresh) {
  const long long total = M * N;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    std::uint32_t v = 0;
    for (int s = 0; s <= smax; s++) v += static_cast<std::uint32_t>(sums[s * total + g]) << (8 * s);
    const long long m = g / N, n = g - m * N, o = m * ldc + n;
    if (out_kind == kI32) {
      auto* p = static_cast<std::int32_t*>(c) + o;
      *p = static_cast<std::int32_t>(fresh ? v : static_cast<std::uint32_t>(*p) + v);
    } else if (out_kind == kI16) {
      auto* p = static_cast<std::int16_t*>(c) + o;
      *p = static_cast<std::int16_t>(fresh ? v : static_cast<std::uint32_t>(*p) + v);
    } else {
      auto* p = static_cast<std::int8_t*>(c) + o;
      *p = static_cast<std::int8_t>(fresh ? v : static_cast<std::uint32_t>(*p) + v);
    }
  }
}

}  // namespace

GemmPlan limb_sum_plan(const GemmPlan& g, int s) {
  GemmPlan u = g;
  u.limbs_a = u.limbs_b = 0;
  u.unsigned_ab = true;
  const int p = limb_pairs(g, s);
  u.K = p * g.K;
  u.lda = u.K;
  u.a0 = 0;
  u.ldb = g.b_kmajor ? u.K : g.N;
  u.b0 = 0;
  u.ldc = g.N;
  u.c0 = 0;
  u.c_dtype = DType::I32;
  u.fresh = true;
  return u;
}

cudaError_t launch_limb_split(const GemmPlan& g, const void* a, const void* b, void* pa, void* pb, cudaStream_t s) {
  const int smax = limb_smax(g);
  SplitArgs A{};
  A.src = a;
  A.dst = static_cast<std::uint8_t*>(pa);
  A.kind = g.a_kind;
  A.limbs = g.limbs_a;
  A.lb_other = g.limbs_b;
  A.smax = smax;
  A.rows = g.M;
  A.cols = g.K;
  A.ld = g.lda;
  A.off = g.a0;
  A.is_a = 1;
  A.kcat_cols = 1;
  for (int t = 0; t <= smax; t++) {
    A.sum_off[t] = limb_a_off(g, t);
    A.pairs[t] = limb_pairs(g, t);
  }
  SplitArgs B = A;
  B.src = b;
  B.dst = static_cast<std::uint8_t*>(pb);
  B.kind = g.b_kind;
  B.limbs = g.limbs_b;
  B.lb_other = g.limbs_a;
  B.is_a = 0;
  if (g.b_kmajor) {  // B[n][k]: pairs concatenate along k (columns)
    B.rows = g.N;
    B.cols = g.K;
    B.kcat_cols = 1;
  } else {  // B[k][n]: pairs stack along k (rows)
    B.rows = g.K;
    B.cols = g.N;
    B.kcat_cols = 0;
  }
  B.ld = g.ldb;
  B.off = g.b0;
  for (int t = 0; t <= smax; t++) B.sum_off[t] = limb_b_off(g, t);
  const int grid = 148 * 8;
  limb_split_kernel<<<grid, 256, 0, s>>>(A);
  limb_split_kernel<<<grid, 256, 0, s>>>(B);
  return cudaGetLastError();
}

cudaError_t launch_limb_combine(const GemmPlan& g, const void* sums, void* c, cudaStream_t s) {
  const int ob = g.c_dtype == DType::I8 ? 1 : g.c_dtype == DType::I16 ? 2 : 4;
  const int ok = g.c_dtype == DType::I8 ? kI8 : g.c_dtype == DType::I16 ? kI16 : kI32;
  limb_combine_kernel<<<148 * 8, 256, 0, s>>>(static_cast<const std::int32_t*>(sums),
                                              static_cast<char*>(c) + g.c0 * ob, limb_smax(g), g.M, g.N, g.ldc, ok,
                                              g.fresh ? 1 : 0);
  return cudaGetLastError();
}

long long limb_plane_bytes_a(const GemmPlan& g) { return limb_a_off(g, limb_smax(g) + 1); }

// ---- fused byte-limb GEMM ------------------------------------------------------------------
// All output-byte sums in ONE kernel: per 128 x 128 output tile, TMEM holds S_0 .. S_smax
// (128 columns each, 512 in all) and every 64-byte k-block of the la A planes and lb B planes
// (u8, K-major [limb][rows][Kp], SW64) feeds the pairs (i, s - i) of every sum s.  The
// epilogue combines C = sum_s S_s << 8s (mod 2^32) straight from TMEM into the output: no
// sums buffer and no combine pass.  Split-K (ksplit > 1) runs k-chunks on separate CTAs that
// add their partial C with red.global.add (wrap-around add: exact mod 2^32; the output was
// zeroed first when it is fresh).

namespace {

constexpr int kLimbThreads = 256;  // warp 0: A loads, warp 1: MMA, warp 2: B loads, 4..7: epilogue
constexpr int kLimbStages = 3;
constexpr std::uint32_t kLimbPlane = 128 * 64;  // one plane's 128 rows x 64 bytes

struct LimbKParams {
  int M, N, Kp, la, lb, smax;
  int tiles_m, tiles_n, ksplit, kb_per;  // k-blocks of 64 bytes per split chunk
  int out_kind, fresh, atomic;
  int tma_c;  // i32 output tile through swizzled staging: TMA store (fresh, one chunk) or TMA add
  void* c;
  long long ldc;
  std::uint32_t idesc;
  long long* trace;  // SB_LIMB_TRACE: per-CTA clock64 stamps [start, first stage, MMAs done, epilogue done]
};

__device__ __forceinline__ long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<long long>(t);
}

__device__ __forceinline__ void tma_load_3d(std::uint32_t dst, const CUtensorMap* map, std::uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__global__ void __launch_bounds__(kLimbThreads, 1)
    gemm_limb_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                     const __grid_constant__ CUtensorMap cmap, const LimbKParams p) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* base =
      reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
  const std::uint32_t stage_bytes = (p.la + p.lb) * kLimbPlane;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(base + kLimbStages * stage_bytes);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + kLimbStages;
  std::uint64_t* tfull = bars + 2 * kLimbStages;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * kLimbStages + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x / p.ksplit, chunk = blockIdx.x % p.ksplit;
  const int m0 = (tile / p.tiles_n) * 128, n0 = (tile % p.tiles_n) * 128;
  const int kb0 = chunk * p.kb_per, kb1 = min(kb0 + p.kb_per, p.Kp / 64);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kLimbStages; s++) {
      mbar_init(&full[s], 2);  // A and B producers each arrive with their bytes
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem_base = *tmem_slot;
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 8] = gtime();
  if (warp == 0 || warp == 2) {
    if (lane == 0) {
      const bool is_a = warp == 0;
      const int np = is_a ? p.la : p.lb, r0 = is_a ? m0 : n0;
      int stage = 0;
      std::uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; kb++) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], np * kLimbPlane);
        const std::uint32_t dst = smem_u32(base + stage * stage_bytes) + (is_a ? 0u : p.la * kLimbPlane);
        // every limb plane in one box (limb is the outer box dimension: planes 8 KB apart)
        tma_load_3d(dst, is_a ? &amap : &bmap, &full[stage], kb * 64, r0, 0);
        if (++stage == kLimbStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    const bool issuer = elect_one_sync();
    int stage = 0;
    std::uint32_t phase = 0;
    // SW64 K-major descriptors: SBO = 8 rows x 64 bytes, layout 4
    const std::uint32_t hi = (512u >> 4) | (1u << 14) | (4u << 29);
    for (int kb = kb0; kb < kb1; kb++) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (p.trace && issuer && kb == kb0) p.trace[blockIdx.x * 8 + 1] = gtime();
      if (issuer) {
        const std::uint32_t sb = smem_u32(base + stage * stage_bytes);
        for (int ks = 0; ks < 2; ks++)
          for (int s = 0; s <= p.smax; s++)
            for (int i = 0; i <= s; i++) {
              const int j = s - i;
              if (i >= p.la || j >= p.lb) continue;
              const std::uint32_t a = ((sb + i * kLimbPlane) >> 4) + ks * 2, b = ((sb + (p.la + j) * kLimbPlane) >> 4) + ks * 2;
              // the first product of sum s in this CTA overwrites its accumulator
              const bool first = kb == kb0 && ks == 0 && i == max(0, s - p.lb + 1);
              umma_i8(tmem_base + s * 128, a | (1u << 16), hi, b | (1u << 16), hi, p.idesc, first ? 0u : 1u);
            }
        umma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == kLimbStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (issuer) umma_commit(tfull);
    if (p.trace && issuer) p.trace[blockIdx.x * 8 + 2] = gtime();
    __syncwarp();
  } else if (warp >= 4) {
    // epilogue: row m0 + 32 q + lane, 16 columns at a time: C = sum_s S_s << 8s
    const int quarter = warp & 3, row = m0 + quarter * 32 + lane;
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (p.trace && threadIdx.x == 128) p.trace[blockIdx.x * 8 + 3] = gtime();
    const std::uint32_t lanes = static_cast<std::uint32_t>(quarter * 32) << 16;
    for (int c16 = 0; c16 < 8; c16++) {
      std::uint32_t v[4][16];
#pragma unroll
      for (int s = 0; s < 4; s++)
        if (s <= p.smax) tmem_ld16_async(tmem_base + lanes + s * 128 + c16 * 16, v[s]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      std::uint32_t o[16];
#pragma unroll
      for (int q = 0; q < 16; q++) {
        std::uint32_t x = 0;
#pragma unroll
        for (int s = 0; s < 4; s++)
          if (s <= p.smax) x += v[s][q] << (8 * s);
        o[q] = x;
      }
      if (p.tma_c) {
        // staging (the drained stage ring): 4 boxes of 32 columns x 128 rows, 128B swizzle
        const int r = quarter * 32 + lane;
        const std::uint32_t rb = smem_u32(base) + (c16 >> 1) * 16384 + r * 128;
#pragma unroll
        for (int q = 0; q < 4; q++)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rb + ((((c16 & 1) * 4 + q) ^ (r & 7)) << 4)),
                       "r"(o[4 * q]), "r"(o[4 * q + 1]), "r"(o[4 * q + 2]), "r"(o[4 * q + 3]));
        continue;
      }
      const int n = n0 + c16 * 16;
      if (row >= p.M || n >= p.N) continue;
      const long long base_idx = static_cast<long long>(row) * p.ldc + n;
      const int cnt = min(16, p.N - n);
      if (p.out_kind == kI32 && p.atomic) {
        std::uint32_t* d = static_cast<std::uint32_t*>(p.c) + base_idx;
        for (int q = 0; q < cnt; q++) asm volatile("red.global.add.u32 [%0], %1;" ::"l"(d + q), "r"(o[q]) : "memory");
      } else if (p.out_kind == kI32 && p.fresh && cnt == 16 && (base_idx & 3) == 0) {
        uint4* d = reinterpret_cast<uint4*>(static_cast<std::uint32_t*>(p.c) + base_idx);
#pragma unroll
        for (int q = 0; q < 4; q++) d[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      } else {
        for (int q = 0; q < cnt; q++) {
          if (p.out_kind == kI32) {
            std::uint32_t* d = static_cast<std::uint32_t*>(p.c) + base_idx + q;
            *d = p.fresh ? o[q] : *d + o[q];
          } else if (p.out_kind == kI16) {
            std::int16_t* d = static_cast<std::int16_t*>(p.c) + base_idx + q;
            *d = static_cast<std::int16_t>(p.fresh ? o[q] : static_cast<std::uint32_t>(*d) + o[q]);
          } else {
            std::int8_t* d = static_cast<std::int8_t*>(p.c) + base_idx + q;
            *d = static_cast<std::int8_t>(p.fresh ? o[q] : static_cast<std::uint32_t>(*d) + o[q]);
          }
        }
      }
    }
    if (p.tma_c) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 128) {
        for (int h = 0; h < 4; h++) {
          if (n0 + h * 32 >= p.N) break;
          if (p.atomic)
            asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                             reinterpret_cast<std::uint64_t>(&cmap)),
                         "r"(smem_u32(base) + h * 16384), "r"(n0 + h * 32), "r"(m0)
                         : "memory");
          else
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                             reinterpret_cast<std::uint64_t>(&cmap)),
                         "r"(smem_u32(base) + h * 16384), "r"(n0 + h * 32), "r"(m0)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    }
    if (p.trace && threadIdx.x == 128) p.trace[blockIdx.x * 8 + 5] = gtime();
  }
  __syncwarp();  // the producer warps' other lanes wait for lane 0 (bar.sync is per warp)
  tc_fence_before();
  __syncthreads();
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 8 + 4] = gtime();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// Unsigned byte planes [limb][rows][Kp] (K-major, zero past K) of a row-major source whose
// k index is contiguous (A, or B stored [n][k]): one thread per 4 consecutive k.
__global__ void limb_planes_kernel(const void* __restrict__ src, int kind, long long rows, long long K, long long Kp,
                                   long long ld, long long off, int limbs, std::uint8_t* __restrict__ dst) {
  const long long kq = Kp / 4, total = rows * kq;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = g / kq, k = (g - r * kq) * 4;
    std::uint32_t v[4];
    const long long e0 = off + r * ld + k;
    if (kind == kI32 && k + 4 <= K && (e0 & 3) == 0) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(static_cast<const std::int32_t*>(src) + e0));
      v[0] = q.x;
      v[1] = q.y;
      v[2] = q.z;
      v[3] = q.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; e++) v[e] = k + e < K ? elem_bits(src, kind, e0 + e) : 0u;
    }
    for (int i = 0; i < limbs; i++) {
      const unsigned sel = static_cast<unsigned>(i | ((4 + i) << 4));
      *reinterpret_cast<std::uint32_t*>(dst + (i * rows + r) * Kp + k) =
          __byte_perm(__byte_perm(v[0], v[1], sel), __byte_perm(v[2], v[3], sel), 0x5410);
    }
  }
}

// Same for B stored [k][n] (n contiguous): 32 x 32 element tiles through shared memory so
// both the reads (along n) and the plane writes (along k) are coalesced.
__global__ void limb_planes_t_kernel(const void* __restrict__ src, int kind, long long N, long long K, long long Kp,
                                     long long ldk, long long off, int limbs, std::uint8_t* __restrict__ dst) {
  __shared__ std::uint32_t tile[32][33];
  const long long tn = (N + 31) / 32, tk = (Kp + 31) / 32;
  for (long long t = blockIdx.x; t < tn * tk; t += gridDim.x) {
    const long long n0 = (t % tn) * 32, k0 = (t / tn) * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const long long k = k0 + r, n = n0 + threadIdx.x;
      tile[r][threadIdx.x] = (k < K && n < N) ? elem_bits(src, kind, off + k * ldk + n) : 0u;
    }
    __syncthreads();
    // write phase: thread (x, y) -> n = n0 + 4 y + x / 8 (8 passes of 32 rows... 4 per pass),
    // k = k0 + 4 (x % 8): one 32-bit word of 4 consecutive k per limb
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int q = tid; q < 32 * 8; q += blockDim.x * blockDim.y) {
      const int rr = q / 8, kk = (q % 8) * 4;
      const long long n = n0 + rr, k = k0 + kk;
      if (n < N && k < Kp) {
        const std::uint32_t x0 = tile[kk][rr], x1 = tile[kk + 1][rr], x2 = tile[kk + 2][rr], x3 = tile[kk + 3][rr];
        for (int i = 0; i < limbs; i++) {
          const unsigned sel = static_cast<unsigned>(i | ((4 + i) << 4));
          *reinterpret_cast<std::uint32_t*>(dst + (i * N + n) * Kp + k) =
              __byte_perm(__byte_perm(x0, x1, sel), __byte_perm(x2, x3, sel), 0x5410);
        }
      }
    }
    __syncthreads();
  }
}

struct LimbPrepared {
  GemmPlan gp;
  const void *pa, *pb;
  void* c;
  LimbKParams kp;
  CUtensorMap amap, bmap, cmap;
};
std::mutex g_limb_mu;
std::vector<LimbPrepared>* g_limb_prep = nullptr;

}  // namespace

long long limb_fused_kp(const GemmPlan& g) { return (g.K + 63) / 64 * 64; }

cudaError_t launch_limb_fused(const GemmPlan& g, const void* a, const void* b, void* pa, void* pb, void* c,
                              cudaStream_t s, int num_sms) {
  const long long Kp = limb_fused_kp(g);
  auto* A = static_cast<std::uint8_t*>(pa);
  auto* B = static_cast<std::uint8_t*>(pb);
  limb_planes_kernel<<<148 * 8, 256, 0, s>>>(a, g.a_kind, g.M, g.K, Kp, g.lda, g.a0, g.limbs_a, A);
  if (g.b_kmajor)
    limb_planes_kernel<<<148 * 8, 256, 0, s>>>(b, g.b_kind, g.N, g.K, Kp, g.ldb, g.b0, g.limbs_b, B);
  else
    limb_planes_t_kernel<<<148 * 8, dim3(32, 8), 0, s>>>(b, g.b_kind, g.N, g.K, Kp, g.ldb, g.b0, g.limbs_b, B);
  const int ob = g.c_dtype == DType::I8 ? 1 : g.c_dtype == DType::I16 ? 2 : 4;
  void* cc = static_cast<char*>(c) + g.c0 * ob;
  LimbPrepared prep;
  {
    LimbPrepared* pr = nullptr;
    std::lock_guard<std::mutex> lock(g_limb_mu);
    if (!g_limb_prep) g_limb_prep = new std::vector<LimbPrepared>();
    for (auto& e : *g_limb_prep)
      if (e.pa == pa && e.pb == pb && e.c == cc && same(e.gp, g)) pr = &e;
    if (!pr) {
      if (g_limb_prep->size() >= 64) g_limb_prep->clear();
      LimbPrepared f;
      f.gp = g;
      f.pa = pa;
      f.pb = pb;
      f.c = cc;
      LimbKParams& kp = f.kp;
      std::memset(&kp, 0, sizeof(kp));
      kp.M = static_cast<int>(g.M);
      kp.N = static_cast<int>(g.N);
      kp.Kp = static_cast<int>(Kp);
      kp.la = g.limbs_a;
      kp.lb = g.limbs_b;
      kp.smax = limb_smax(g);
      kp.tiles_m = static_cast<int>((g.M + 127) / 128);
      kp.tiles_n = static_cast<int>((g.N + 127) / 128);
      const int kbs = static_cast<int>(Kp / 64), tiles = kp.tiles_m * kp.tiles_n;
      // split-K (i32 outputs: red.global.add) while tiles alone leave SMs idle
      kp.ksplit = 1;
      if (g.c_dtype == DType::I32 && !std::getenv("SB_LIMB_NOSPLIT"))
        while (kp.ksplit < 8 && tiles * kp.ksplit * 2 <= num_sms && kbs / (kp.ksplit * 2) >= 4) kp.ksplit *= 2;
      kp.kb_per = (kbs + kp.ksplit - 1) / kp.ksplit;
      kp.out_kind = ob == 1 ? kI8 : ob == 2 ? kI16 : kI32;
      kp.fresh = g.fresh ? 1 : 0;
      kp.atomic = kp.ksplit > 1 || !g.fresh ? 1 : 0;  // partial or accumulating tiles add into C
      kp.tma_c = kp.out_kind == kI32 && g.ldc % 4 == 0 && reinterpret_cast<std::uintptr_t>(cc) % 16 == 0 ? 1 : 0;
      if (!kp.tma_c) kp.ksplit = 1, kp.atomic = 0;
      kp.c = cc;
      kp.ldc = g.ldc;
      // u8 x u8 -> s32, both K-major, N = 128, M = 128
      kp.idesc = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      auto encode = get_encode();
      if (!encode) return cudaErrorNotSupported;
      cuuint32_t es[3] = {1, 1, 1};
      cuuint64_t adim[3] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(g.M), static_cast<cuuint64_t>(g.limbs_a)};
      cuuint64_t astr[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Kp * g.M)};
      cuuint32_t box[3] = {64, 128, static_cast<cuuint32_t>(g.limbs_a)};
      if (encode(&f.amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, pa, adim, astr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
        return cudaErrorInvalidValue;
      cuuint64_t bdim[3] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(g.N), static_cast<cuuint64_t>(g.limbs_b)};
      cuuint64_t bstr[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Kp * g.N)};
      box[2] = static_cast<cuuint32_t>(g.limbs_b);
      if (encode(&f.bmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, pb, bdim, bstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
        return cudaErrorInvalidValue;
      std::memset(&f.cmap, 0, sizeof(f.cmap));
      if (kp.tma_c) {
        cuuint64_t cdim[2] = {static_cast<cuuint64_t>(g.N), static_cast<cuuint64_t>(g.M)};
        cuuint64_t cstr[1] = {static_cast<cuuint64_t>(g.ldc * 4)};
        cuuint32_t cbox[2] = {32, 128};
        if (encode(&f.cmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, cc, cdim, cstr, cbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
          return cudaErrorInvalidValue;
      }
      static bool attr = false;
      if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gemm_limb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
      }
      g_limb_prep->push_back(f);
      pr = &g_limb_prep->back();
    }
    prep = *pr;
  }
  const LimbKParams& kp = prep.kp;
  if (kp.atomic && kp.fresh && kp.ksplit > 1) {
    // partial sums add into the output: start it from the identity
    for (long long m = 0; m < g.M; m++) {
      if (g.ldc == g.N) {
        cudaError_t e = cudaMemsetAsync(cc, 0, static_cast<std::size_t>(g.M * g.N) * 4, s);
        if (e != cudaSuccess) return e;
        break;
      }
      cudaError_t e = cudaMemsetAsync(static_cast<std::uint32_t*>(cc) + m * g.ldc, 0, static_cast<std::size_t>(g.N) * 4, s);
      if (e != cudaSuccess) return e;
    }
  }
  const std::size_t smem = 1024 + kLimbStages * (kp.la + kp.lb) * kLimbPlane + 256;
  const int grid = kp.tiles_m * kp.tiles_n * kp.ksplit;
  static const bool tracing = std::getenv("SB_LIMB_TRACE") != nullptr;
  if (!tracing) {
    gemm_limb_kernel<<<grid, kLimbThreads, smem, s>>>(prep.amap, prep.bmap, prep.cmap, kp);
    return cudaGetLastError();
  }
  LimbKParams kt = kp;
  static long long* tr = nullptr;
  if (!tr) cudaMalloc(&tr, 1024 * 8 * 8);
  cudaMemsetAsync(tr, 0, 1024 * 8 * 8, s);
  kt.trace = tr;
  gemm_limb_kernel<<<grid, kLimbThreads, smem, s>>>(prep.amap, prep.bmap, prep.cmap, kt);
  std::vector<long long> h(static_cast<std::size_t>(grid) * 8);
  cudaStreamSynchronize(s);
  cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
  long long t0 = h[0];
  for (int b = 0; b < grid; b++) t0 = std::min(t0, h[b * 8]);
  for (int b = 0; b < grid; b += grid / 8)
    std::fprintf(stderr, "limb CTA %3d (ns): start %6lld first-stage %6lld mma-done %6lld epi-start %6lld epi-done %6lld end %6lld\n", b,
                 h[b * 8] - t0, h[b * 8 + 1] - t0, h[b * 8 + 2] - t0, h[b * 8 + 3] - t0, h[b * 8 + 5] - t0, h[b * 8 + 4] - t0);
  return cudaGetLastError();
}

// ---- 3xTF32 mode -----------------------------------------------------------------------
// a = hi(a) + lo(a) with hi = tf32(a), lo = tf32(a - hi); A*B ~= hi*hi + hi*lo + lo*hi as
// ONE kind::tf32 GEMM over k concatenated three times: A' = [a_hi | a_hi | a_lo] (M x 3K),
// B'^T = [b_hi | b_lo | b_hi] (N x 3K, K-major).  fp32 accumulation in TMEM.

namespace {

__device__ __forceinline__ float tf32_rn(float x) {
  std::uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void tf32_split_a_kernel(const float* __restrict__ a, float* pa, long long M, long long K, long long lda) {
  const long long ta = M * K;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < ta;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long m = g / K, k = g - m * K;
    const float x = a[m * lda + k];
    const float hi = tf32_rn(x), lo = tf32_rn(x - hi);
    float* row = pa + m * 3 * K;
    row[k] = hi;
    row[K + k] = hi;
    row[2 * K + k] = lo;
  }
}

// B'^T[n][seg * K + k] from B[k][n] (N-major) through a 32 x 32 smem tile: coalesced reads
// along n and coalesced writes along k.  K-major sources (b_k == 1) need no transpose.
__global__ void tf32_split_b_kernel(const float* __restrict__ b, float* pb, long long N, long long K, long long b_k,
                                    long long b_n) {
  __shared__ float tile[32][33];
  const long long tiles_n = (N + 31) / 32, tiles_k = (K + 31) / 32;
  for (long long t = blockIdx.x; t < tiles_n * tiles_k; t += gridDim.x) {
    const long long n0 = (t % tiles_n) * 32, k0 = (t / tiles_n) * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const long long k = k0 + r, n = n0 + threadIdx.x;
      tile[r][threadIdx.x] = (k < K && n < N) ? b[k * b_k + n * b_n] : 0.0f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const long long n = n0 + r, k = k0 + threadIdx.x;
      if (n < N && k < K) {
        const float x = tile[threadIdx.x][r];
        const float hi = tf32_rn(x), lo = tf32_rn(x - hi);
        float* row = pb + n * 3 * K;
        row[k] = hi;
        row[K + k] = lo;
        row[2 * K + k] = hi;
      }
    }
    __syncthreads();
  }
}

}  // namespace

// Product t (0: hi*hi, 1: hi*lo, 2: lo*hi) as its own GEMM over segment t of the planes,
// written to sums[t]; the three run side by side and tf32_combine adds them.
GemmPlan tf32_sum_plan(const GemmPlan& g, int t) {
  GemmPlan u = g;
  u.tf32x3 = true;
  u.f32 = false;
  u.lda = 3 * g.K;
  u.a0 = t * g.K;
  u.b_kmajor = true;
  u.ldb = 3 * g.K;
  u.b0 = t * g.K;
  u.ldc = g.N;
  u.c0 = 0;
  u.fresh = true;
  u.c_dtype = DType::I32;  // 32-bit output path (fp32 bits)
  return u;
}

namespace {
__global__ void tf32_combine_kernel(const float* __restrict__ sums, float* c, long long M, long long N, long long ldc,
                                    int fresh) {
  const long long total = M * N;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long m = g / N, n = g - m * N;
    const float v = sums[g] + (sums[total + g] + sums[2 * total + g]);
    float* o = c + m * ldc + n;
    *o = fresh ? v : *o + v;
  }
}
}  // namespace

cudaError_t launch_tf32_combine(const GemmPlan& g, const void* sums, void* c, cudaStream_t s) {
  tf32_combine_kernel<<<148 * 8, 256, 0, s>>>(static_cast<const float*>(sums), static_cast<float*>(c) + g.c0, g.M,
                                              g.N, g.ldc, g.fresh ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_tf32_split(const GemmPlan& g, const void* a, const void* b, void* pa, void* pb, cudaStream_t s) {
  const float* af = static_cast<const float*>(a) + g.a0;
  const float* bf = static_cast<const float*>(b) + g.b0;
  const long long b_k = g.b_kmajor ? 1 : g.ldb, b_n = g.b_kmajor ? g.ldb : 1;
  tf32_split_a_kernel<<<148 * 8, 256, 0, s>>>(af, static_cast<float*>(pa), g.M, g.K, g.lda);
  tf32_split_b_kernel<<<148 * 8, dim3(32, 8), 0, s>>>(bf, static_cast<float*>(pb), g.N, g.K, b_k, b_n);
  return cudaGetLastError();
}
long long limb_plane_bytes_b(const GemmPlan& g) { return limb_b_off(g, limb_smax(g) + 1); }

cudaError_t launch_gemm_tc(const GemmPlan& g, const GemmArgs& args, cudaStream_t s, int num_sms) {
  Prepared prep;  // copied under the lock: another thread's push_back may move the cache
  {
    Prepared* pr = nullptr;
    std::lock_guard<std::mutex> lock(g_mu);
    if (!g_prep) g_prep = new std::vector<Prepared>();
    for (auto& e : *g_prep)
      if (e.a == args.a && e.b == args.b && e.c == args.c && same(e.gp, g)) pr = &e;
    if (!pr) {
      if (g_prep->size() >= 256) g_prep->clear();
      Prepared fresh;
      cudaError_t err = prepare(g, args, &fresh, num_sms);
      if (err != cudaSuccess) return err;
      g_prep->push_back(fresh);
      pr = &g_prep->back();
    }
    prep = *pr;
  }
  GemmKParams kp = prep.kp;
  kp.pdl = args.pdl_mode != kPdlOff ? 1 : 0;
  kp.pdl_wait = args.pdl_mode == kPdlWait ? 1 : 0;
  int tiles = kp.tiles_m * kp.tiles_n;
  // split-K over CTA pairs while the tiles alone leave at least half the SMs idle: opt-in
  // (SB_GEMM_SPLIT=1), measured slower at config 1 (1024^3: 11.2 vs 7.8 us per pipelined step,
  // 17.5 vs 13.4 us per launch; the pair's DSMEM hand-off serialises both epilogues)
  kp.ksplit = 1;
  if (kp.tma_out && !kp.tf32 && kp.bn == 128 && kp.kblocks >= 2 && 2 * tiles <= num_sms && std::getenv("SB_GEMM_SPLIT")) {
    kp.ksplit = 2;
    kp.kb_per = (kp.kblocks + 1) / 2;
  }
  cudaLaunchConfig_t cfg = {};
  const int ctas = kp.ksplit * tiles;
  cfg.gridDim = dim3(static_cast<unsigned>(kp.ksplit > 1 ? ctas : (tiles < num_sms ? tiles : num_sms)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes(kp.bn, kp.stages);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (kp.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (kp.ksplit > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, gemm_i8_tc_kernel, prep.amap, prep.bmap, prep.cmap, kp);
}

}  // namespace sb
