// tcgen05 implicit-GEMM convolution for Stripe contraction blocks (K3 in SURVEY §2.1).
//
// Matches leaf bodies  $a = load(I); $b = load(F); $p = mul($a, $b); O = store($p)
// with O:add, I/F i8 and halo constraints (the reference's conv shape,
// tests/support.cpp:79-124; fig6a / conv_relu fixtures).  Per output pixel
// block the GEMM is  O[m, k] += sum_{i,j,c} I[m shifted by (i,j), c] * F[i,j,k,c].
//
// B200 mapping
//   * one persistent CTA per SM; warp 0 = TMA producer, warp 1 = MMA issuer
//     (single elected thread, tcgen05.mma.cta_group::1.kind::i8), warps 2-5 =
//     epilogue (tcgen05.ld TMEM -> registers -> global);
//   * M tile = 128 output pixels = TX output rows x P (pitch, >= W + S - 1);
//     ONE 4-D TMA box per 16-channel plane brings the haloed input strip
//     (TX + R - 1 rows x P columns) into shared memory.  TMA zero-fills
//     coordinates outside the constraint window, which is exactly the
//     reference's skip-predicate semantics for these constraints;
//   * the strip is stored [plane][row][col][16 B] so the A operand of every tap
//     (i, j) is the same no-swizzle K-major UMMA layout shifted by
//     (i * P + j) * 16 bytes: 9 taps reuse one strip (no im2col traffic);
//   * the whole filter stays resident in shared memory (loaded once per CTA);
//   * s32 accumulators live in TMEM, double-buffered so the epilogue of tile t
//     overlaps the MMAs of tile t + 1.
// Exactness: i8 x i8 products are exact and the planner only routes here when
// |sum| < 2^31 (K_total * 128 * 128 < 2^31), so the s32 accumulation equals the
// reference's int64 sum wrapped at store (ir.cpp:79-97) bit for bit.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstring>

#include "../kernels.hpp"

namespace sb {
namespace {

constexpr int kThreads = 192;  // 6 warps
constexpr int kStages = 4;
constexpr int kTileM = 128;

struct ConvKParams {
  std::int64_t N, H, W, C, K, R, S;
  int P, TX, CH;            // pitch, rows per tile, channels per chunk
  int tiles_x, tiles;       // x tiles per image, total tiles
  std::int64_t b_i, b_j, b_k, b_c, b0;
  std::int64_t c_n, c_x, c_y, c0;
  std::int64_t ox, oy, u_lo, v_lo;  // strip origin = (x0 + ox - u_lo, oy - v_lo)
  int out_kind;             // kI8/kI16/kI32
  int fresh;                // overwrite (prepare_outputs identity is fused) vs accumulate
  int vec_out;              // i32 output, 16-byte aligned rows -> int4 stores
  int filt_vec;             // filter channels contiguous and 16-byte aligned -> uint4 loads
  int tma_out;              // fresh i32 output written through swizzled staging + TMA stores
  int nstg;                 // staging buffers (1 or 2)
  std::uint32_t staging_bytes;
  std::uint32_t strip_bytes, plane_bytes, filt_bytes;
  std::uint32_t tmem_cols;
  std::uint32_t idesc;
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

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// K-major, no-swizzle UMMA shared-memory descriptor (sm100 version 1).
__device__ __forceinline__ std::uint64_t umma_desc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<std::uint64_t>(1) << 46;  // version = 1 (Blackwell)
  return d;                                  // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ void umma_i8(std::uint32_t tmem_d, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                        std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
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

__global__ void __launch_bounds__(kThreads, 1)
    conv_i8_tc_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap omap,
                      const std::int8_t* __restrict__ filt, void* __restrict__ out, const ConvKParams p) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  // carve: [output staging (1024-aligned, 128B swizzle)][stages strips][filter][barriers]
  std::uint8_t* staging = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
  std::uint8_t* strips = staging + p.staging_bytes;
  std::uint8_t* fsm = strips + kStages * p.strip_bytes + 1024;  // +slack: junk rows read past a strip
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(fsm + ((p.filt_bytes + 127) / 128) * 128);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + kStages;
  std::uint64_t* tfull = bars + 2 * kStages;
  std::uint64_t* tempty = bars + 2 * kStages + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * kStages + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  // Filter -> shared memory in the UMMA K-major layout:
  // byte (tap, plane, k, c%16) at ((tap * C/16 + plane) * K + k) * 16 + c%16.
  if (p.filt_vec) {
    // 16-byte rows of contiguous input channels: one cp.async per (tap, plane, k); k fastest so
    // consecutive threads fill consecutive 16-byte smem slots (conflict-free).
    const std::uint32_t planes = static_cast<std::uint32_t>(p.C / 16), K = static_cast<std::uint32_t>(p.K);
    const std::uint32_t S = static_cast<std::uint32_t>(p.S);
    const std::uint32_t total = static_cast<std::uint32_t>(p.R * p.S) * K * planes;
    for (std::uint32_t e = threadIdx.x; e < total; e += kThreads) {
      std::uint32_t k = e % K;
      std::uint32_t rest = e / K;
      std::uint32_t pl = rest % planes;
      std::uint32_t tap = rest / planes;
      std::uint32_t i = tap / S, j = tap % S;
      const std::int8_t* src = filt + (p.b_i * i + p.b_j * j + p.b_k * k + 16 * pl + p.b0);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(fsm + e * 16)), "l"(src) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    const int planes = static_cast<int>(p.C / 16);
    const std::int64_t total = p.R * p.S * p.K * p.C;
    for (std::int64_t e = threadIdx.x; e < total; e += kThreads) {
      std::int64_t c = e % p.C;
      std::int64_t rest = e / p.C;
      std::int64_t k = rest % p.K;
      rest /= p.K;
      std::int64_t j = rest % p.S;
      std::int64_t i = rest / p.S;
      std::int64_t tap = i * p.S + j;
      std::int64_t src = p.b_i * i + p.b_j * j + p.b_k * k + p.b_c * c + p.b0;
      fsm[((tap * planes + c / 16) * p.K + k) * 16 + (c % 16)] = static_cast<std::uint8_t>(filt[src]);
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // make generic-proxy filter writes visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem_base = *tmem_slot;

  const int chunks = static_cast<int>(p.C / p.CH);
  const int ksteps = p.CH / 32;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      std::uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        int n = t / p.tiles_x;
        int x0 = (t % p.tiles_x) * p.TX;
        for (int cc = 0; cc < chunks; cc++) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], p.strip_bytes);
          std::uint8_t* dst = strips + stage * p.strip_bytes;
          int u0 = static_cast<int>(x0 + p.ox - p.u_lo);
          int v0 = static_cast<int>(p.oy - p.v_lo);
          for (int pl = 0; pl < p.CH / 16; pl++)
            tma_load_4d(dst + pl * p.plane_bytes, &amap, &full[stage], cc * p.CH + pl * 16, v0, u0, n);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (one thread) ----------------
      int stage = 0;
      std::uint32_t phase = 0;
      int iter = 0;
      const std::uint32_t fsm_addr = smem_u32(fsm);
      const std::uint32_t b_plane = static_cast<std::uint32_t>(p.K) * 16;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, iter++) {
        int acc = iter & 1;
        std::uint32_t aphase = (iter >> 1) & 1;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        std::uint32_t dcol = tmem_base + static_cast<std::uint32_t>(acc * p.K);
        for (int cc = 0; cc < chunks; cc++) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          std::uint32_t sbase = smem_u32(strips + stage * p.strip_bytes);
          for (int i = 0; i < p.R; i++) {
            for (int j = 0; j < p.S; j++) {
              int tap = i * static_cast<int>(p.S) + j;
              for (int s = 0; s < ksteps; s++) {
                std::uint32_t a_addr = sbase + 2 * s * p.plane_bytes + static_cast<std::uint32_t>(i * p.P + j) * 16;
                std::uint32_t b_addr =
                    fsm_addr + (static_cast<std::uint32_t>(tap) * (p.C / 16) + cc * (p.CH / 16) + 2 * s) * b_plane;
                std::uint64_t ad = umma_desc(a_addr, p.plane_bytes, 128);
                std::uint64_t bd = umma_desc(b_addr, b_plane, 128);
                umma_i8(dcol, ad, bd, p.idesc, (cc | tap | s) != 0);
              }
            }
          }
          umma_commit(&empty[stage]);  // smem slot free once these MMAs retire
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 ----------------
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const int row = quarter * 32 + lane;
    const int xl = row / p.P;
    const int y = row % p.P;
    int iter = 0;
    if (p.tma_out) {
      // Fresh i32 output: TMEM -> registers -> 128B-swizzled smem staging (conflict-free,
      // row = TMEM lane) -> TMA tensor stores of full lines; rows outside the image are
      // clipped by the tensor map bounds.
      const bool leader = threadIdx.x == 64;
      const int halves = static_cast<int>(p.K / 32);
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, iter++) {
        int acc = iter & 1;
        std::uint32_t aphase = (iter >> 1) & 1;
        int sb = p.nstg == 2 ? (iter & 1) : 0;
        if (leader) {
          if (p.nstg == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // staging buffer sb is free again
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        std::uint8_t* stg = staging + static_cast<std::uint32_t>(sb * halves) * 16384u;
        for (int h = 0; h < halves; h++) {
          std::uint32_t v[32];
          tmem_ld32(tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) +
                        static_cast<std::uint32_t>(acc * p.K + h * 32),
                    v);
          std::uint32_t rbase = smem_u32(stg + h * 16384 + row * 128);
#pragma unroll
          for (int q = 0; q < 8; q++)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((q ^ (row & 7)) << 4)),
                         "r"(v[4 * q]), "r"(v[4 * q + 1]), "r"(v[4 * q + 2]), "r"(v[4 * q + 3])
                         : "memory");
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);  // accumulator drained: MMA may reuse it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (leader) {
          int n = t / p.tiles_x;
          int x0 = (t % p.tiles_x) * p.TX;
          for (int h = 0; h < halves; h++)
            asm volatile(
                "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                    reinterpret_cast<std::uint64_t>(&omap)),
                "r"(smem_u32(stg + h * 16384)), "r"(h * 32), "r"(0), "r"(x0), "r"(n)
                : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, iter++) {
      int acc = iter & 1;
      std::uint32_t aphase = (iter >> 1) & 1;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      int n = t / p.tiles_x;
      int x = (t % p.tiles_x) * p.TX + xl;
      bool valid = y < p.W && x < p.H && xl < p.TX;
      std::int64_t obase = p.c_n * n + p.c_x * x + p.c_y * y + p.c0;
      for (int k0 = 0; k0 < p.K; k0 += 32) {
        std::uint32_t v[32];
        tmem_ld32(tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) +
                      static_cast<std::uint32_t>(acc * p.K + k0),
                  v);
        if (!valid) continue;
        if (p.out_kind == kI32) {
          std::int32_t* o = static_cast<std::int32_t*>(out) + obase + k0;
          if (p.vec_out) {
            int4* o4 = reinterpret_cast<int4*>(o);
#pragma unroll
            for (int q = 0; q < 8; q++) {
              int4 w = make_int4(static_cast<int>(v[4 * q]), static_cast<int>(v[4 * q + 1]),
                                 static_cast<int>(v[4 * q + 2]), static_cast<int>(v[4 * q + 3]));
              if (!p.fresh) {
                int4 old = o4[q];
                w.x += old.x;
                w.y += old.y;
                w.z += old.z;
                w.w += old.w;
              }
              o4[q] = w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 32; q++) {
              std::int32_t w = static_cast<std::int32_t>(v[q]);
              o[q] = p.fresh ? w : static_cast<std::int32_t>(static_cast<std::uint32_t>(o[q]) + v[q]);
            }
          }
        } else if (p.out_kind == kI16) {
          std::int16_t* o = static_cast<std::int16_t*>(out) + obase + k0;
#pragma unroll
          for (int q = 0; q < 32; q++)
            o[q] = static_cast<std::int16_t>(p.fresh ? v[q] : static_cast<std::uint32_t>(o[q]) + v[q]);
        } else {
          std::int8_t* o = static_cast<std::int8_t*>(out) + obase + k0;
#pragma unroll
          for (int q = 0; q < 32; q++)
            o[q] = static_cast<std::int8_t>(p.fresh ? v[q] : static_cast<std::uint32_t>(o[q]) + v[q]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols));
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

int pitch_for(std::int64_t W, std::int64_t S) {
  std::int64_t need = W + S - 1;
  for (int p = 8; p <= 128; p *= 2)
    if (p >= need) return p;
  return -1;
}

std::size_t smem_bytes(const ConvKParams& kp) {
  return 1024 /*align*/ + kp.staging_bytes + kStages * kp.strip_bytes + 1024 + ((kp.filt_bytes + 127) / 128) * 128 +
         256;
}

bool fill_params(const ConvPlan& cp, ConvKParams* kp) {
  std::memset(kp, 0, sizeof(*kp));
  kp->N = cp.N;
  kp->H = cp.H;
  kp->W = cp.W;
  kp->C = cp.C;
  kp->K = cp.K;
  kp->R = cp.R;
  kp->S = cp.S;
  kp->P = pitch_for(cp.W, cp.S);
  if (kp->P < 0) return false;
  kp->TX = kTileM / kp->P;
  kp->CH = cp.C % 64 == 0 ? 64 : 32;
  kp->tiles_x = static_cast<int>((cp.H + kp->TX - 1) / kp->TX);
  kp->tiles = static_cast<int>(cp.N * kp->tiles_x);
  kp->b_i = cp.b_i;
  kp->b_j = cp.b_j;
  kp->b_k = cp.b_k;
  kp->b_c = cp.b_c;
  kp->b0 = cp.b0;
  kp->c_n = cp.c_n;
  kp->c_x = cp.c_x;
  kp->c_y = cp.c_y;
  kp->c0 = cp.c0;
  kp->ox = cp.ox;
  kp->oy = cp.oy;
  kp->u_lo = cp.u_lo;
  kp->v_lo = cp.v_lo;
  kp->out_kind = cp.c_dtype == DType::I8 ? kI8 : cp.c_dtype == DType::I16 ? kI16 : kI32;
  kp->fresh = cp.fresh_output ? 1 : 0;
  kp->vec_out = kp->out_kind == kI32 && cp.c_n % 4 == 0 && cp.c_x % 4 == 0 && cp.c_y % 4 == 0 && cp.c0 % 4 == 0;
  kp->filt_vec = cp.b_c == 1 && cp.b_i % 16 == 0 && cp.b_j % 16 == 0 && cp.b_k % 16 == 0 && cp.b0 % 16 == 0;
  kp->plane_bytes = static_cast<std::uint32_t>((kp->TX + cp.R - 1) * kp->P * 16);
  kp->strip_bytes = kp->plane_bytes * (kp->CH / 16);
  kp->filt_bytes = static_cast<std::uint32_t>(cp.R * cp.S * cp.K * cp.C);
  kp->tma_out = kp->fresh && kp->out_kind == kI32 && cp.c_y % 4 == 0 && cp.c_x % 4 == 0 && cp.c_n % 4 == 0 &&
                cp.c0 % 4 == 0 && cp.K % 32 == 0;
  kp->nstg = 2;
  kp->staging_bytes = kp->tma_out ? static_cast<std::uint32_t>(kp->nstg * (cp.K / 32) * 16384) : 0;
  if (kp->tma_out && smem_bytes(*kp) > 220 * 1024) {
    kp->nstg = 1;
    kp->staging_bytes = static_cast<std::uint32_t>((cp.K / 32) * 16384);
  }
  if (kp->tma_out && smem_bytes(*kp) > 220 * 1024) {
    kp->tma_out = 0;
    kp->staging_bytes = 0;
  }
  std::uint32_t cols = 32;
  while (cols < 2 * cp.K) cols *= 2;
  kp->tmem_cols = cols;
  // instruction descriptor: S32 accum, signed A/B, K-major both, N, M=128
  kp->idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((static_cast<std::uint32_t>(cp.K) >> 3) << 17) |
              ((128u >> 4) << 24);
  return true;
}

}  // namespace

const char* conv_tc_unsupported(const ConvPlan& cp) {
  ConvKParams kp;
  if (!fill_params(cp, &kp)) return "image row too wide for one 128-row tile";
  if (cp.C % 32 != 0) return "channels not a multiple of 32";
  if (cp.K % 32 != 0 || cp.K > 256) return "output channels not a multiple of 32 in [32, 256]";
  if (cp.R * cp.S > 64) return "filter too large";
  if (smem_bytes(kp) > 220 * 1024) return "filter + strips exceed shared memory";
  if (cp.a_y % 16 != 0 || cp.a_x % 16 != 0 || cp.a_n % 16 != 0) return "input strides not 16-byte multiples";
  return nullptr;
}

cudaError_t launch_conv_tc(const ConvPlan& cp, const ConvArgs& args, cudaStream_t s, int num_sms) {
  ConvKParams kp;
  if (!fill_params(cp, &kp) || conv_tc_unsupported(cp)) return cudaErrorNotSupported;
  auto encode = get_encode();
  if (!encode) return cudaErrorNotSupported;
  const std::int8_t* base = static_cast<const std::int8_t*>(args.a) + cp.a0 + cp.a_x * cp.u_lo + cp.a_y * cp.v_lo;
  if (reinterpret_cast<std::uintptr_t>(base) % 16 != 0) return cudaErrorMisalignedAddress;
  CUtensorMap map;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(cp.C), static_cast<cuuint64_t>(cp.v_hi - cp.v_lo + 1),
                        static_cast<cuuint64_t>(cp.u_hi - cp.u_lo + 1), static_cast<cuuint64_t>(cp.N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(cp.a_y), static_cast<cuuint64_t>(cp.a_x),
                           static_cast<cuuint64_t>(cp.a_n)};
  cuuint32_t box[4] = {16u, static_cast<cuuint32_t>(kp.P), static_cast<cuuint32_t>(kp.TX + cp.R - 1), 1u};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<std::int8_t*>(base), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  CUtensorMap omap;
  std::memset(&omap, 0, sizeof(omap));
  if (kp.tma_out) {
    std::int32_t* obase = static_cast<std::int32_t*>(args.c) + cp.c0;
    if (reinterpret_cast<std::uintptr_t>(obase) % 16 != 0) return cudaErrorMisalignedAddress;
    cuuint64_t odims[4] = {static_cast<cuuint64_t>(cp.K), static_cast<cuuint64_t>(cp.W),
                           static_cast<cuuint64_t>(cp.H), static_cast<cuuint64_t>(cp.N)};
    cuuint64_t ostr[3] = {static_cast<cuuint64_t>(cp.c_y * 4), static_cast<cuuint64_t>((cp.c_x ? cp.c_x : cp.c_y * cp.W) * 4),
                          static_cast<cuuint64_t>((cp.c_n ? cp.c_n : cp.c_y * cp.W * cp.H) * 4)};
    cuuint32_t obox[4] = {32u, static_cast<cuuint32_t>(kp.P), static_cast<cuuint32_t>(kp.TX), 1u};
    r = encode(&omap, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, obase, odims, ostr, obox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  std::size_t smem = smem_bytes(kp);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(conv_i8_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int grid = kp.tiles < num_sms ? kp.tiles : num_sms;
  conv_i8_tc_kernel<<<grid, kThreads, smem, s>>>(map, omap, static_cast<const std::int8_t*>(args.b), args.c, kp);
  return cudaGetLastError();
}

}  // namespace sb
