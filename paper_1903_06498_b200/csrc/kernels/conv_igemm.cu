// General tcgen05 implicit-GEMM convolution (K3) for conv leaves the
// resident-filter kernel (conv_tc.cu) does not take: strided convs, 1x1 convs, wide
// filters that do not fit shared memory (3x3x512x512 = 2.4 MB), any output-channel count.
//
//     O[n, x, y, k] (+)= sum_{i, j, c} I[n, sx*x + i + ox, sy*y + j + oy, c] * F[i, j, k, c]
//
// GEMM view: M = output pixels in (n, x, y) order, N = output channels k, reduction =
// (i, j, c).  The A operand is produced by TMA in im2col mode: one
// cp.async.bulk.tensor.4d...im2col load brings 128 consecutive output pixels' input rows
// for one filter tap (im2col offsets) and one 64/128-channel slice, walking (y, x, n) with
// the conv strides and zero-filling the padding halo.  The Stripe constraints that skip
// out-of-window taps (interp.cpp:426-428) become exactly that zero fill: a skipped point
// contributes nothing to an add aggregation, a zero product contributes nothing either.
// The filter B (k rows, c contiguous) streams through the same mbarrier ring.
//
// Warp roles as in gemm_tc.cu: warp 0 TMA producer, warp 1 single-thread
// tcgen05.mma.kind::i8 issuer (M=128, N=128, K=32 per instruction), warps 2-5 epilogue
// (tcgen05.ld -> 128B-swizzled staging -> TMA tensor store, or read-modify-write).
// Double-buffered TMEM accumulators let the epilogue of tile t overlap the MMAs of t+1.
// Exactness: s32 accumulation with R*S*C*128*128 < 2^31 (planner check).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "../kernels.hpp"

// Development aid (make trace): per-tile timestamps of CTA 0 printed after each launch.
#ifdef SB_TILE_TRACE
#define EPI_EXP p.exp
#define EXPB(b) (p.exp & (b))
#include <cstdio>
#define TILE_STAMP(slot, i) \
  do {                                                                            \
    if (p.trace && blockIdx.x == 0 && (i) < 128) p.trace[(slot)*128 + (i)] = clock64(); \
  } while (0)
#define STAGE_STAMP(iter, st, k)                                                                      \
  do {                                                                                                \
    if (p.trace && blockIdx.x == 0 && (iter) < 32 && (st) < 4) p.trace[640 + ((iter)*4 + (st)) * 3 + (k)] = clock64(); \
  } while (0)
#else
// (SB_EXP_CONST: compile-time knock-out bits for experiment builds, see tools/exp_build.sh)
#ifndef SB_EXP_CONST
#define SB_EXP_CONST 0
#endif
#define EPI_EXP SB_EXP_CONST
#define EXPB(b) (SB_EXP_CONST & (b))
#define STAGE_STAMP(iter, st, k) \
  do {                           \
  } while (0)
#define TILE_STAMP(slot, i) \
  do {                      \
  } while (0)
#endif

namespace sb {
namespace {

constexpr int kRawStages = 4;        // band_raw: raw-row stages in flight (cp.async groups)
constexpr int kThreadsGather = 448;  // + 8 warps gathering A tiles (small-channel convs), 2 per row
constexpr int BM = 128, BN = 128;
constexpr int kRingBytes = 192 * 1024;  // A+B stage ring (cap)
constexpr int kStgBytes = BM * BN * 4;    // output staging (i32 worst case)
constexpr int kVecBytes = 2048 * 4;       // per-channel epilogue vector
constexpr int kMaxVecK = 2048;

struct IgKParams {
  int M, N;           // GEMM rows (output pixels) and cols (output channels)
  int P, Q;           // output rows / cols per image (x, y extents)
  int sx, sy;         // conv strides (traversal strides of the im2col map)
  int lower_h, lower_w;
  int S, cblocks, kblocks;
  int tiles_m, tiles_n;
  int bk, stages;     // channels per k-block (64 or 128), ring depth
  int stg_off, res_off, vec_off, bar_off;  // dynamic smem layout (bytes from the 1 KB-aligned base)
  int smem;
  // gather mode (ConvPlan::packed): A rows built by warps 6-9 from the original input
  int gather, tab_off, rsc, g_C, g_S, g_R, g_run;
  int epi_warps;  // 4 or 8 (two warps per TMEM lane quarter, each taking half the columns)
  int epi_split;  // 8 epilogue warps as two independent groups of 4 taking alternate tiles
  int b_res, bres_off;
  int b_early;  // resident filter immutable: loaded before griddepcontrol.wait
  int bn;      // tile width in output channels: 128 or 256 (N = 256 MMAs, 512 TMEM columns)
  int mt;      // 128-row M sub-tiles per tile (1 or 2): one stage feeds mt x the MMAs
  int bn_box;  // filter rows per TMA box / smem tile: 64 when N <= 64, else bn
  int stg4;    // split i8 epilogue with two staging buffers per group (when smem allows)
  // residual added by the tensor core: res tile (pixels x channels, SW128) x identity (128 x 128,
  // resident) accumulated into the tile after its k-blocks; loaded by a fifth producer warp
  int res_mma, ident_off;
  int kpb;  // k-blocks per ring stage (one barrier handshake per stage: ~200 cycles each, measured)  // whole filter resident in smem (one n-tile, small reduction): the ring holds A only
  int pdl_wait;   // griddepcontrol.wait before touching buffers (else independent of in-flight work)
  long long g_an, g_ax, g_ay, g_a0;
  int g_ulo, g_uhi, g_vlo, g_vhi;
  const std::int8_t* g_in;
  int fresh, tma_out, out_kind;
  void* c;
  long long ldc;      // elements between consecutive output pixels
  std::uint32_t idesc, desc_hi;
  int pdl;
  long long* trace;  // SB_TILE_TRACE builds only: per-tile clock64 stamps of CTA 0
  int exp;           // SB_TILE_TRACE builds only: SB_IG_EXP knock-out bits (experiments)
  // fused epilogue: out = wrap(max(acc + vec[k], lo))
  int epi, epi_vec, epi_lo, epi_res, vec_kind;
  int fast_clamp;  // |acc| + 128 < 2^31: clamp decided by an int32 compare against lo - vec[k]
  // i8 TMA-store epilogue in int32 arithmetic: out = wrap8(max(acc + res + vec[k], lo)); exact when
  // there is no clamp (wrapped low bits) or every |vec[k]| <= bias_bound (no int32 overflow)
  int fast8;
  long long bias_bound;
  int thr_always;  // fast8 with a clamp bound outside int32: always the threshold form
  int epi_pipe;    // fast8 epilogue with the next chunk's TMEM load in flight
  // n-stationary: tiles_n > 1 with the grid a multiple of tiles_n, so CTA c only ever sees
  // n-tile c % tiles_n and keeps that slice of the filter resident (b_res); res1: the
  // tensor-core residual single-buffered (the smem the resident slice needs)
  int nstat, res1;
  // band mode (ConvPlan::fold_band): tile t = output rows (img, band*(t % band_rpi) ..) x 128
  // columns; A = one bulk copy of band_bytes from the compact folded rows (band_rowb bytes
  // each, band_img per image) into a ring stage of band_stage bytes, read with overlapping-row
  // descriptors (a_hi); the band's rows stacked along N (vector index k % vec_mod)
  int band, band_rpi, band_bytes, band_stage, vec_mod;
  long long band_rowb, band_img;
  const std::int8_t* band_src;
  std::uint32_t a_hi;
  // band_raw (ConvPlan::band_raw): no folded copy; four producer warps cp.async each band's
  // 2 * kblocks raw input rows (raw_chunks 16-byte chunks of the valid columns, zero-filled
  // outside [r_ulo, r_uhi]) into a ring of kRawStages raw stages (raw_rp bytes per row, the
  // valid bytes from raw_col0, zero padding either side written once), then build the band's
  // folded rows from them: folded pixel (j, V) = raw rows 2j, 2j+1, 6 bytes each from window
  // column 2V, then 4 zero bytes
  int band_raw, raw_rp, raw_col0, raw_chunks, raw_stage, raw_off, raw_fv;
  long long r_an, r_ax, r_a0;
  int r_ulo, r_uhi, r_vlo;
  // strip mode (stride-1 3x3 over 64 channels into a fresh i8 activation): tile t = image
  // t / strip_tx, output rows strip_rows * (t % strip_tx) .. (mt sub-tiles of 2 rows x 64-pixel
  // pitch); A = ONE haloed strip (rows + 2, 64 pixels, 64 channels, SW64 4-D TMA box, zero
  // outside the constraint window) per tile and the 9 taps are descriptor shifts of it
  // ((i * 64 + j) * 64 bytes), so no input byte is fetched 9 times; 4-D clipped TMA store
  int strip, strip_tx, strip_rows, strip_uoff, strip_voff, strip_stage;
  const void* vec;
  long long vec_k;
  long long lo;
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
__device__ __forceinline__ void tma_load_im2col(std::uint32_t dst, const CUtensorMap* map, std::uint64_t* bar, int c,
                                                int w, int h, int n, std::uint16_t ow, std::uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(std::uint32_t dst, const CUtensorMap* map, std::uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
          "r"(dst),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
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
__device__ __forceinline__ bool elect_one() {
  std::uint32_t is;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(is));
  return is != 0;
}
__device__ __forceinline__ void umma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// tcgen05.ld without the wait: the registers are valid only after tmem_wait_ld(v), whose
// "+r" operands keep every use of v behind the wait.
__device__ __forceinline__ void tmem_ld32_async(std::uint32_t taddr, std::uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld(std::uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
                 "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                 "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}

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

// 16-column TMEM loads (32 lanes x 16 columns): the i8 epilogue ping-pongs two of these
__device__ __forceinline__ void tmem_ld16_async(std::uint32_t taddr, std::uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16(std::uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}

// i8 TMA-store epilogue of one tile, software-pipelined: chunk c+1's TMEM load is in flight
// while chunk c is transformed and staged (tcgen05.wait::ld waits for every outstanding load,
// so the next load is issued right after the wait that makes chunk c valid).  Chunks run over
// (sub-tile, 32-column chunk) pairs; out = wrap8(max(acc + res + vec, lo)) or, with THR, the
// exact threshold form acc + res >= t[k] ? acc + res + vec : lo (see IgKParams::fast8).
// vaddr / taddr: this tile's vector / threshold in smem; raddr / saddr: this thread's row of
// the residual / staging buffer (16 KB boxes of 128 rows x 128 bytes, 128B swizzle).
__device__ __forceinline__ std::uint32_t lds32(std::uint32_t a) {
  std::uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(std::uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
// one 16-column half chunk (columns 32 h + 16 hf ..): transform v and stage its 16 bytes
template <bool THR, bool RES>
__device__ __forceinline__ void epi8_half(const std::uint32_t (&v)[16], int sub, int h, int hf, std::uint32_t vaddr,
                                          std::uint32_t taddr, std::uint32_t raddr, std::uint32_t saddr, int hcnt,
                                          int hsh, int sw, std::uint32_t lo32u, std::int32_t lo8, int exp = 0) {
  // 16 KB staging box and swizzled 16-byte unit of this half: 128-byte rows hold 1 << hsh
  // 32-column chunks (hsh = 2; band mode with 64 channels: hsh = 1, one band row per box)
  const std::uint32_t box = (sub * hcnt + (h >> hsh)) * 16384;
  const std::uint32_t unit = (((2 * (h & ((1 << hsh) - 1)) + hf) ^ sw) << 4);
  uint4 r4 = make_uint4(0, 0, 0, 0);
  if (RES) r4 = lds128(raddr + box + unit);
  const std::uint32_t rq[4] = {r4.x, r4.y, r4.z, r4.w};
  std::uint32_t w[4];
#pragma unroll
  for (int q4 = 0; q4 < 4; q4++) {
    const int col = h * 32 + hf * 16 + 4 * q4;
    const uint4 b4 = (exp & 1024) ? make_uint4(col, col, col, col) : lds128(vaddr + col * 4);  // (trace: no vector loads)
    const std::uint32_t bq[4] = {b4.x, b4.y, b4.z, b4.w};
    uint4 t4 = make_uint4(0, 0, 0, 0);
    if (THR) t4 = lds128(taddr + col * 4);
    const std::uint32_t tq[4] = {t4.x, t4.y, t4.z, t4.w};
    std::uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; e++) {
      std::int32_t x = static_cast<std::int32_t>(v[4 * q4 + e]);
      if (RES) {
        std::int32_t r;  // sign-extended residual byte (prmt sign-replicate selector)
        asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(rq[q4]), "r"(0x8880u + 0x1111u * e));
        x += r;
      }
      if (THR) o[e] = x >= static_cast<std::int32_t>(tq[e]) ? static_cast<std::uint32_t>(x) + bq[e] : lo32u;
      else o[e] = static_cast<std::uint32_t>(max(x + static_cast<std::int32_t>(bq[e]), lo8));
    }
    w[q4] = __byte_perm(__byte_perm(o[0], o[1], 0x0040), __byte_perm(o[2], o[3], 0x0040), 0x5410);
  }
  if (exp & 512) {  // (trace: no staging stores; keep the values live)
    if ((w[0] ^ w[1] ^ w[2] ^ w[3]) == 0x12345678u) asm volatile("st.shared.b32 [%0], %1;" ::"r"(saddr), "r"(w[0]));
  } else
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr + box + unit), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]));
}

// i8 TMA-store epilogue of one tile, software-pipelined over two 16-column register buffers:
// half k+1's TMEM load is in flight while half k is transformed and staged (tcgen05.wait::ld
// waits for every outstanding load, so the next load is issued right after the wait that made
// half k valid; two named buffers, no register copies).  Halves run over (sub-tile, 32-column
// chunk, half); out = wrap8(max(acc + res + vec, lo)) or, with THR, the exact threshold form
// acc + res >= t[k] ? acc + res + vec : lo (see IgKParams::fast8).  vaddr / taddr: this tile's
// vector / threshold in smem; raddr / saddr: this thread's row of the residual / staging
// buffer (16 KB boxes of 128 rows x 128 bytes, 128B swizzle).
template <bool THR, bool RES>
__device__ __forceinline__ void epi8_pipelined(std::uint32_t tbase, int bn, int mt, int c_lo, int per,
                                               std::uint32_t vaddr, std::uint32_t taddr, std::uint32_t raddr,
                                               std::uint32_t saddr, int hcnt, int hsh, int sw, std::uint32_t lo32u,
                                               std::int32_t lo8, int exp) {
  const int total = mt * per, c_end = c_lo + per;
  if (total <= 0) return;
  std::uint32_t va[16], vb[16];
  // chunk (sub, h): half 0 in va, half 1 in vb; the next chunk's column advanced incrementally
  if (exp & 256) {  // (trace: no TMEM loads)
    for (int q = 0; q < 16; q++) va[q] = vb[q] = q * 977u;
  } else
  tmem_ld16_async(tbase + c_lo * 32, va);
  int sub = 0, h = c_lo;
  for (int c = 0; c < total; c++) {
    int nsub = sub, nh = h + 1;
    if (nh == c_end) {
      nh = c_lo;
      nsub++;
    }
    const std::uint32_t col = tbase + sub * bn + h * 32;
    if (!(exp & 256)) {
      tmem_wait_ld16(va);
      tmem_ld16_async(col + 16, vb);
    }
    epi8_half<THR, RES>(va, sub, h, 0, vaddr, taddr, raddr, saddr, hcnt, hsh, sw, lo32u, lo8, exp);
    if (!(exp & 256)) {
      tmem_wait_ld16(vb);
      if (c + 1 < total) tmem_ld16_async(tbase + nsub * bn + nh * 32, va);
    }
    epi8_half<THR, RES>(vb, sub, h, 1, vaddr, taddr, raddr, saddr, hcnt, hsh, sw, lo32u, lo8, exp);
    sub = nsub;
    h = nh;
  }
}

__global__ void __launch_bounds__(kThreadsGather, 1)
    conv_igemm_i8_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                         const __grid_constant__ CUtensorMap cmap, const __grid_constant__ CUtensorMap rmap,
                         const IgKParams p) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* base =
      reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t{1023});
  const int TM = BM * p.mt;  // tile rows (output pixels)
  const std::uint32_t stage_a = TM * p.bk, stage_b = p.bn_box * p.bk;
  std::uint8_t* ring = base;                    // stages x (A | B), or stages x A with the filter resident
  const std::uint32_t sstride = p.band    ? static_cast<std::uint32_t>(p.band_stage)
                                 : p.strip ? static_cast<std::uint32_t>(p.strip_stage)
                                           : p.kpb * (stage_a + (p.b_res ? 0u : stage_b));
  std::uint8_t* bres = base + p.bres_off;       // resident filter: kblocks x stage_b
  std::uint8_t* stg = base + p.stg_off;         // output staging: i32 4 x 16 KB quarters | i8 2 x 16 KB
  std::uint8_t* rstg = base + p.res_off;        // residual tiles (i8, 2 x 16 KB)
  std::int32_t* vec_s = reinterpret_cast<std::int32_t*>(base + p.vec_off);  // per-channel vector (<= 2048)
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(base + p.bar_off);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + 16;
  std::uint64_t* tfull = bars + 32;
  std::uint64_t* tempty = bars + 34;
  std::uint64_t* rfull = bars + 36;  // [2]
  std::uint64_t* bfull = bars + 38;  // resident filter landed
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 40);
  std::uint64_t* rempty = bars + 44;  // [2] residual buffer consumed by the MMAs (res_mma)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles = p.tiles_m * p.tiles_n;
  const int stages = p.stages;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; s++) {
      // A and B transactions (B + 256 gathering threads); no B arrival with the filter resident
      mbar_init(&full[s], (p.gather ? 256 : 1) + (p.b_res ? 0 : 1));
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], p.epi_split ? 128 : 32 * p.epi_warps);
    }
    mbar_init(&rfull[0], 1);
    mbar_init(&rfull[1], 1);
    mbar_init(&rempty[0], 1);
    mbar_init(&rempty[1], 1);
    mbar_init(bfull, 1);
    *reinterpret_cast<int*>(bars + 41) = 0;  // some |vec[k]| > bias_bound
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    // all 512 columns (one CTA per SM): the allocation is then column 0, so the MMA issuer
    // addresses accumulators with compile-time-uniform values
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (p.res_mma) {
    // identity B operand 32 x 32, K-major without swizzle: core matrices of 8 rows x 16 bytes,
    // the two along K 128 bytes apart (LBO), the four 8-row groups 256 bytes apart (SBO):
    // byte (n, k) at (n / 8) 256 + (k / 16) 128 + (n % 8) 16 + k % 16, one where n == k
    uint4* id = reinterpret_cast<uint4*>(base + p.ident_off);
    for (int u = threadIdx.x; u < 64; u += blockDim.x) {
      const int grp = u >> 4, kc = (u >> 3) & 1, r = u & 7, n = grp * 8 + r;
      std::uint32_t w[4] = {0, 0, 0, 0};
      if ((n >> 4) == kc) w[(n & 15) >> 2] = 1u << (8 * (n & 3));
      id[u] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem_base = *tmem_slot;
  // Dependents are released only after a griddepcontrol.wait of this grid returned (the
  // predecessor has completed): at most this launch and its successor overlap.
  if (p.pdl && !p.pdl_wait && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // TMA producers.  One thread issues a tensor load only every ~260 cycles whatever the box
  // size (measured, scratch/tma_lat.cu), so im2col mode splits the issue over four warps:
  // A and B loads on separate threads, alternate k-blocks on two chains.  Gather mode has
  // one producer (B only; the A rows are built by the gather warps).
  const int pw0 = 2 + p.epi_warps + (p.gather ? 8 : 0);  // extra producer warps pw0 .. pw0 + 2
  const int pidx = warp == 0 ? 0 : (!p.gather && warp >= pw0) ? warp - pw0 + 1 : -1;
  if (pidx >= 0) {
    {  // converged warp; one elected lane issues (uniform-register operands, see the MMA warp)
      const bool issuer = elect_one();
      const bool do_a = !p.gather && (pidx & 1) == 0 && pidx != 4, do_b = p.gather || (pidx & 1) == 1;
      // an immutable resident filter (a root `in` buffer no plan step writes) is fetched while
      // the predecessor still runs; everything else waits for it
      if (p.pdl_wait && !(p.b_early && do_b && p.b_res)) asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
      const int nchains = p.gather ? 1 : 2, chain = p.gather ? 0 : pidx >> 1;
      const int PQ = p.P * p.Q;
      if (p.band_raw && pidx != 1) {
        // band_raw fold producers: warps pidx 0, 2, 3, 4 (128 threads, named barrier 5)
        const int tt = (pidx == 0 ? 0 : pidx - 1) * 32 + lane;
        std::uint8_t* raw = base + p.raw_off;
        const int rrows = 2 * p.kblocks, rp = p.raw_rp, c16 = p.raw_rp / 16;
        auto tbar = [] { asm volatile("bar.sync 5, 128;" ::: "memory"); };
        // padding bytes of every raw row (outside the copied chunks): zero once
        for (int i = tt; i < kRawStages * rrows * c16; i += 128) {
          const int r = i / c16, b = (i - r * c16) * 16;
          const int rs = r / rrows;
          if (b < p.raw_col0 || b >= p.raw_col0 + p.raw_chunks * 16)
            *reinterpret_cast<uint4*>(raw + rs * p.raw_stage + (r - rs * rrows) * rp + b) = make_uint4(0, 0, 0, 0);
        }
        // copy role: thread tt owns chunk ch0 of rows r0, r0 + rstep, ... (no per-chunk division)
        const int rstep = 128 / p.raw_chunks, r0 = tt / p.raw_chunks, ch0 = tt - r0 * p.raw_chunks;
        auto issue = [&](int k) {  // raw rows of this CTA's k-th tile into raw stage k % kRawStages
          const int t = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
          if (t < tiles && r0 < rstep && !EXPB(65536)) {
            const int img = t / p.band_rpi, U0 = (t - img * p.band_rpi) * p.band;
            const std::uint32_t dst0 = smem_u32(raw + (k % kRawStages) * p.raw_stage) + p.raw_col0 + ch0 * 16;
            const std::int8_t* src0 = p.band_src + p.r_a0 + p.r_an * img + 3ll * p.r_vlo + ch0 * 16;
            for (int r = r0; r < rrows; r += rstep) {
              const int u = 2 * U0 + r;
              const bool ok = u >= p.r_ulo && u <= p.r_uhi;
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst0 + r * rp),
                           "l"(src0 + p.r_ax * (ok ? u : p.r_ulo)), "r"(ok ? 16 : 0)
                           : "memory");
            }
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        };
        for (int k = 0; k < kRawStages - 1; k++) issue(k);
        int stage = 0;
        std::uint32_t phase = 0;
        const int s0 = p.raw_col0 - 3 * p.r_vlo;
        for (int k = 0, t = blockIdx.x; t < tiles; k++, t += gridDim.x) {
          issue(k + kRawStages - 1);
          asm volatile("cp.async.wait_group %0;" ::"n"(kRawStages - 1) : "memory");
          tbar();  // tile k's raw rows have landed (every thread's chunks)
          mbar_wait(&empty[stage], phase ^ 1);
          const std::uint32_t rs = smem_u32(raw + (k % kRawStages) * p.raw_stage);
          const std::uint32_t dst = smem_u32(ring + stage * sstride);
          for (int j = 0; j < p.kblocks && !EXPB(32768); j++)
          for (int V = tt; V < p.raw_fv; V += 128) {
            const std::uint32_t a = rs + 2 * j * rp + s0 + 6 * V, a4 = a & ~3u, sh = (a & 3u) * 8;
            const std::uint32_t x0 = lds32(a4), x1 = lds32(a4 + 4), x2 = lds32(a4 + 8);
            const std::uint32_t y0 = lds32(a4 + rp), y1 = lds32(a4 + rp + 4), y2 = lds32(a4 + rp + 8);
            const std::uint32_t lo0 = __funnelshift_r(x0, x1, sh), hi0 = __funnelshift_r(x1, x2, sh);
            const std::uint32_t lo1 = __funnelshift_r(y0, y1, sh), hi1 = __funnelshift_r(y1, y2, sh);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + j * static_cast<std::uint32_t>(p.band_rowb) + V * 16),
                         "r"(lo0), "r"((hi0 & 0xFFFFu) | (lo1 << 16)), "r"((lo1 >> 16) | (hi1 << 16)), "r"(0u)
                         : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
          tbar();
          if (tt == 0) mbar_arrive(&full[stage]);
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
      } else if (pidx == 4) {
        // residual tiles for the tensor-core add, double-buffered by tile parity
        const int res_buf = TM * p.bn, hcount = (p.bn + 127) / 128;
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, it++) {
          const int b = p.res1 ? 0 : it & 1;
          mbar_wait(&rempty[b], (p.res1 ? it & 1 : (it >> 1) & 1) ^ 1);
          const int m0 = (t / p.tiles_n) * TM, n0 = (t % p.tiles_n) * p.bn;
          const int halves = min(p.bn, p.N - n0 + 127) / 128;
          if (issuer) {
            mbar_expect_tx(&rfull[b], p.mt * BM * 128 * halves);
            for (int sub = 0; sub < p.mt; sub++)
              for (int hh = 0; hh < halves; hh++)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
                    "[%2];" ::"r"(smem_u32(base + p.res_off + b * res_buf + (sub * hcount + hh) * 16384)),
                    "l"(reinterpret_cast<std::uint64_t>(&rmap)), "r"(smem_u32(&rfull[b])), "r"(n0 + hh * 128),
                    "r"(m0 + sub * BM)
                    : "memory");
          }
          __syncwarp();
        }
      } else if (do_b && p.b_res) {
        // the whole filter once (tiles_n == 1), then this producer is done
        if (chain == 0 && issuer) {
          mbar_expect_tx(bfull, p.kblocks * stage_b);
          int cb = 0, r = 0, s = 0;
          for (int kb = 0; kb < p.kblocks; kb++) {
            const std::uint32_t dst = smem_u32(bres + kb * stage_b);
            const int nb0 = p.nstat ? static_cast<int>(blockIdx.x % p.tiles_n) * p.bn : 0;  // this CTA's slice
            if (p.gather) tma_load_4d(dst, &bmap, bfull, kb * p.bk, nb0, 0, 0);
            else tma_load_4d(dst, &bmap, bfull, cb * p.bk, nb0, s, r);
            if (++cb == p.cblocks) {
              cb = 0;
              if (++s == p.S) {
                s = 0;
                r++;
              }
            }
          }
        }
      } else if (p.strip) {
        // one haloed strip per tile (4-D TMA box, SW64)
        if (pidx == 0) {
          int stage = 0;
          std::uint32_t phase = 0;
          for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (issuer) {
              const int img = t / p.strip_tx, x0 = (t - img * p.strip_tx) * p.strip_rows;
              mbar_expect_tx(&full[stage], static_cast<std::uint32_t>(p.strip_stage));
              tma_load_4d(smem_u32(ring + stage * sstride), &amap, &full[stage], 0, p.strip_voff, x0 + p.strip_uoff, img);
            }
            __syncwarp();
            if (++stage == stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      } else if (p.band) {
        // one bulk copy per tile: the band's folded rows (plus the junk rows' tail)
        if (pidx == 0) {
          int stage = 0;
          std::uint32_t phase = 0;
          for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (issuer) {
              const int img = t / p.band_rpi, u = (t - img * p.band_rpi) * p.band;
              const std::int8_t* src = p.band_src + img * p.band_img + u * p.band_rowb;
              if (EXPB(1)) mbar_arrive(&full[stage]);  // (trace builds: no A loads)
              else {
              mbar_expect_tx(&full[stage], static_cast<std::uint32_t>(p.band_bytes));
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      smem_u32(ring + stage * sstride)),
                  "l"(reinterpret_cast<std::uint64_t>(src)), "r"(p.band_bytes), "r"(smem_u32(&full[stage]))
                  : "memory");
              }
            }
            __syncwarp();
            if (++stage == stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      } else {
      int stage = 0, kit = 0;
      std::uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        // n-tiles of one m-tile are adjacent in t: the A strip stays hot in L2
        const int m0 = (t / p.tiles_n) * TM, n0 = (t % p.tiles_n) * p.bn;
        const int img = m0 / PQ, rem = m0 - img * PQ;
        const int ox = rem / p.Q, oy = rem - ox * p.Q;
        const int h0 = p.lower_h + ox * p.sx, w0 = p.lower_w + oy * p.sy;
        int cb = 0, r = 0, s = 0;
        for (int kb0 = 0; kb0 < p.kblocks; kb0 += p.kpb, kit++) {
          const bool mine = kit % nchains == chain;
          if (mine) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (issuer && pidx == 0 && kb0 == 0)
              TILE_STAMP(0, (t - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x));
#ifdef SB_TILE_TRACE
            if (issuer && do_a && (p.exp & 1)) mbar_arrive(&full[stage]);
            else
#endif
            if (issuer && do_a) mbar_expect_tx(&full[stage], p.kpb * stage_a);
            if (issuer && do_b && !p.b_res) mbar_expect_tx(&full[stage], p.kpb * stage_b);
          }
          const std::uint32_t sa = smem_u32(ring + stage * sstride);
          for (int j = 0; j < p.kpb; j++) {
            const int kb = kb0 + j;
            if (issuer && mine && do_a
#ifdef SB_TILE_TRACE
                && !(p.exp & 1)
#endif
            )
              tma_load_im2col(sa + j * stage_a, &amap, &full[stage], cb * p.bk, w0, h0, img,
                              static_cast<std::uint16_t>(s), static_cast<std::uint16_t>(r));
            if (issuer && mine && do_b && !p.b_res) {
              const std::uint32_t sb = sa + p.kpb * stage_a + j * stage_b;
              if (p.gather) tma_load_4d(sb, &bmap, &full[stage], kb * p.bk, n0, 0, 0);
              else tma_load_4d(sb, &bmap, &full[stage], cb * p.bk, n0, s, r);
            }
            if (++cb == p.cblocks) {
              cb = 0;
              if (++s == p.S) {
                s = 0;
                r++;
              }
            }
          }
          __syncwarp();
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the loop (converged, so the descriptors stay in uniform registers);
    // one elected lane issues the MMAs and commits
    const bool issuer = elect_one();
    int stage = 0, iter = 0;
    std::uint32_t phase = 0;
    const int ksteps = p.bk / 32;
    if (p.b_res) {
      mbar_wait(bfull, 0);
      tc_fence_after();
    }
    // shared-memory bases as integers once: the per-stage descriptor arithmetic then stays
    // in uniform registers (no vector-register round trip per MMA)
    const std::uint32_t ring_s = smem_u32(ring), bres_s = smem_u32(bres);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, iter++) {
      const int acc = iter & 1;
      mbar_wait(&tempty[acc], ((iter >> 1) & 1) ^ 1);
      tc_fence_after();
      if (issuer) TILE_STAMP(1, iter);
      const std::uint32_t d = static_cast<std::uint32_t>(acc * p.mt * p.bn);  // TMEM column (allocation at 0)
      // a last n-tile with few valid output channels runs narrower instructions
      const int nrem = p.N - (t % p.tiles_n) * p.bn;
      const std::uint32_t ninst = nrem <= 64 ? 64u : nrem <= 128 ? 128u : static_cast<std::uint32_t>(p.bn);
      const std::uint32_t idesc = (p.idesc & ~(0x3Fu << 17)) | ((ninst >> 3) << 17);
      for (int kb0 = 0; kb0 < p.kblocks; kb0 += p.kpb) {
        if (issuer) STAGE_STAMP(iter, kb0 / p.kpb, 0);
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (issuer) STAGE_STAMP(iter, kb0 / p.kpb, 1);
        const std::uint32_t sa = ring_s + stage * sstride;
        const std::uint32_t a0 = (sa >> 4) | (1u << 16);
        const std::uint32_t b0 = ((p.b_res ? bres_s + kb0 * stage_b : sa + p.kpb * stage_a) >> 4) | (1u << 16);
        const std::uint32_t as = stage_a >> 4, bs = stage_b >> 4, hi = p.desc_hi;
        const bool first = kb0 == 0;
#ifdef SB_TILE_TRACE
        if (issuer && p.band && blockIdx.x == 0 && iter == 0 && p.trace && (p.exp & 16)) {
          // debug: the first band stage as the MMA sees it (2 KB) and its descriptor fields
          const long long* src = reinterpret_cast<const long long*>(ring + stage * sstride);
          for (int i = 0; i < 256; i++) p.trace[1280 + i] = src[i];
          p.trace[1536] = sa;
          p.trace[1537] = static_cast<long long>(stage);
        }
#endif
        if (EXPB(2)) {  // (trace builds: no MMAs)
        } else if (issuer) {
          // rolled issue: only the innermost k-steps unrolled, descriptors advanced by adds, so
          // few 64-bit descriptor pairs are live in uniform registers at once (fully unrolled
          // runs of 16-18 MMAs spilled uniform registers through vector ones: stage-1 3x3
          // 166 -> 145 us at b1024)
          if (p.strip) {
            // tap (i, j) of sub-tile sub: strip rows 2 sub + i .., shifted by j pixels (64 bytes
            // each); SW64 descriptors, base offset 0 for every 64-byte row shift (conv_tc.cu)
            const std::uint32_t sa0 = (sa >> 4) | (1u << 16);
#pragma unroll 1
            for (int q = 0; q < p.mt * 3; q++) {
              const int sub = q / 3, i = q - sub * 3;
              const std::uint32_t ds = d + sub * p.bn, ar = sa0 + (sub * 2 + i) * 256, br = b0 + i * 3 * bs;
#pragma unroll
              for (int j = 0; j < 3; j++)
#pragma unroll
                for (int ks = 0; ks < 2; ks++)
                  umma_i8(ds, ar + j * 4 + ks * 2, hi, br + j * bs + ks * 2, hi, idesc, (i | j | ks) ? 1u : 0u);
            }
          } else if (p.band) {
            // folded row j of the band (overlapping-row A, a_hi) against banded filter block j
            const std::uint32_t rs = static_cast<std::uint32_t>(p.band_rowb >> 4), ab = (sa >> 4) | (1u << 16);
#pragma unroll 1
            for (int j = 0; j < p.kblocks; j++)
#pragma unroll
              for (int ks = 0; ks < 2; ks++)
                umma_i8(d, ab + j * rs + ks * 2, p.a_hi, b0 + j * bs + ks * 2, hi, idesc, (j | ks) ? 1u : 0u);
          } else {
            // sub-tile sub: rows 128 sub .. of every k-block's A, accumulator columns + sub * bn
#pragma unroll 1
            for (int q = 0; q < p.mt * p.kpb; q++) {
              const int sub = q / p.kpb, j = q - sub * p.kpb;
              const std::uint32_t ds = d + sub * p.bn, ar = a0 + sub * ((BM * p.bk) >> 4) + j * as, br = b0 + j * bs;
              const bool f = first && j == 0;
              if (ksteps == 2) {
#pragma unroll
                for (int ks = 0; ks < 2; ks++) umma_i8(ds, ar + ks * 2, hi, br + ks * 2, hi, idesc, (f && ks == 0) ? 0u : 1u);
              } else {
#pragma unroll
                for (int ks = 0; ks < 4; ks++) umma_i8(ds, ar + ks * 2, hi, br + ks * 2, hi, idesc, (f && ks == 0) ? 0u : 1u);
              }
            }
          }
        }
        if (issuer) STAGE_STAMP(iter, kb0 / p.kpb, 2);
        if (issuer) umma_commit(&empty[stage]);
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (p.res_mma) {
        // + residual: D[:, 32 g + n] += R[:, 32 g + k] * I32[n, k], one N = 32 instruction per
        // 32 output channels (the residual's K = 32 chunk g against the 32 x 32 identity)
        const int rb = p.res1 ? 0 : acc;
        mbar_wait(&rfull[rb], p.res1 ? iter & 1 : (iter >> 1) & 1);
        tc_fence_after();
        const int groups = min(p.bn, nrem + 31) / 32;
        const std::uint32_t hi128 = (1024u >> 4) | (1u << 14) | (2u << 29);
        const std::uint32_t id32 = (p.idesc & ~(0x3Fu << 17)) | ((32u >> 3) << 17);
        const std::uint32_t ra = smem_u32(base + p.res_off + rb * TM * p.bn), ib = smem_u32(base + p.ident_off);
        const std::uint32_t ib_lo = (ib >> 4) | ((128u >> 4) << 16), ib_hi = (256u >> 4) | (1u << 14);
        const int hcount = (p.bn + 127) / 128;
        for (int sub = 0; sub < p.mt; sub++)
          for (int g = 0; g < groups; g++)
            if (issuer)
              umma_i8(d + sub * p.bn + 32 * g,
                      (((ra + (sub * hcount + (g >> 2)) * 16384) >> 4) | (1u << 16)) + (g & 3) * 2, hi128, ib_lo, ib_hi,
                      id32, 1);
        if (issuer) umma_commit(&rempty[rb]);
        __syncwarp();
      }
      if (issuer) umma_commit(&tfull[acc]);
      __syncwarp();
      if (issuer) TILE_STAMP(2, iter);
    }
  } else if (p.gather && warp >= 2 + p.epi_warps) {
    // gather producers: row r of every A stage = the packed (i, j, c) taps of pixel m0 + r,
    // zero where a constraint skips the tap; written in the TMA swizzle layout
    const int gt = threadIdx.x - 64 - 32 * p.epi_warps;  // 0..255: row r = gt / 2, half = gt % 2
    const int r = gt >> 1, half = gt & 1;
    std::int32_t* toff = reinterpret_cast<std::int32_t*>(base + p.tab_off);
    std::int8_t* tdi = reinterpret_cast<std::int8_t*>(toff + p.kblocks * p.bk);
    std::int8_t* tdj = tdi + p.kblocks * p.bk;
    for (int kk = gt; kk < p.kblocks * p.bk; kk += 256) {
      if (kk < p.rsc) {
        const int c = kk % p.g_C, ij = kk / p.g_C, i = ij / p.g_S, j = ij - i * p.g_S;
        toff[kk] = static_cast<std::int32_t>(p.g_ax * i + p.g_ay * j + c);
        tdi[kk] = static_cast<std::int8_t>(i);
        tdj[kk] = static_cast<std::int8_t>(j);
      } else {
        toff[kk] = 0;
        tdi[kk] = -128;  // never valid
        tdj[kk] = 0;
      }
    }
    if (p.pdl_wait) asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("bar.sync 2, 256;" ::: "memory");
    const int PQ = p.P * p.Q;
    const int sw = p.bk == 128 ? (r & 7) : ((r >> 1) & 3);
    int stage = 0;
    std::uint32_t phase = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m = (t / p.tiles_n) * BM + r;
      const bool live = m < p.M;
      const int img = live ? m / PQ : 0, rem = m - img * PQ;
      const int ox = rem / p.Q, oy = rem - ox * p.Q;
      const int u0 = p.sx * ox, v0 = p.sy * oy;
      const std::int8_t* pix = p.g_in + p.g_a0 + p.g_an * img + p.g_ax * u0 + p.g_ay * v0;
      for (int kb = 0; kb < p.kblocks; kb++) {
        std::uint8_t* rowp = ring + stage * sstride + r * p.bk;
        if (p.g_run) {
          // run layout: tap row i's S*C input bytes are contiguous (a_y == C); copy them with
          // aligned word loads + funnel shifts, zeroing bytes whose column j is skipped.
          // Both of this thread's runs issue their loads before the stage wait, so one L2
          // round trip per k-block overlaps the ring back-pressure.
          const int RUN = p.g_run;
          const int jlo = max(0, p.g_vlo - v0), jhi = min(p.g_S - 1, p.g_vhi - v0);
          const int d0 = jlo * p.g_C, dlen = (jhi - jlo + 1) * p.g_C;
          const int nruns = p.bk / RUN;
          for (int rb = half; rb < nruns; rb += 4) {
            std::uint32_t wd[2][17];
            int sh[2];
#pragma unroll
            for (int z = 0; z < 2; z++) {
              const int ri = rb + 2 * z;
              const int i = kb * nruns + ri;
              const int u = u0 + i;
              const bool ok = ri < nruns && live && i < p.g_R && u >= p.g_ulo && u <= p.g_uhi && dlen > 0;
              const long long src = static_cast<long long>(reinterpret_cast<std::uintptr_t>(pix)) + p.g_ax * i;
              const long long first_w = (src + d0) >> 2, last_w = (src + d0 + dlen - 1) >> 2;
              const long long A0 = src >> 2;
              sh[z] = static_cast<int>(src & 3) * 8;
              // words e in [e_lo, e_hi] hold valid bytes (the others are never dereferenced)
              const int e_lo = ok ? static_cast<int>(first_w - A0) : 1 << 20;
              const int e_hi = ok ? min(static_cast<int>(last_w - A0), RUN / 4) : -1;
              const std::uint32_t* wp = reinterpret_cast<const std::uint32_t*>(A0 << 2);
#pragma unroll
              for (int e = 0; e < 17; e++) wd[z][e] = (e >= e_lo && e <= e_hi) ? __ldg(wp + e) : 0u;
            }
            if (rb == half) mbar_wait(&empty[stage], phase ^ 1);  // stage free before the first store
            auto below = [](int x) -> std::uint32_t { return x <= 0 ? 0u : x >= 4 ? ~0u : ((1u << (8 * x)) - 1u); };
#pragma unroll
            for (int z = 0; z < 2; z++) {
              const int ri = rb + 2 * z;
              if (ri >= nruns) break;
#pragma unroll
              for (int ch = 0; ch < 4; ch++) {
                if (ch >= RUN / 16) break;
                std::uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; e++) {
                  const int ow = ch * 4 + e;
                  const std::uint32_t v = __funnelshift_r(wd[z][ow], wd[z][ow + 1], sh[z]);
                  const int lb = d0 - 4 * ow, hb = d0 + dlen - 4 * ow;
                  w[e] = v & below(hb) & ~below(lb);
                }
                const int q = (ri * RUN) / 16 + ch;
                *reinterpret_cast<uint4*>(rowp + ((q ^ sw) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
          }
          if (half >= nruns) mbar_wait(&empty[stage], phase ^ 1);
        } else {
          mbar_wait(&empty[stage], phase ^ 1);
        }
        if (!p.g_run)
        for (int q = half; q < p.bk / 16; q += 2) {
          std::uint32_t w[4];
#pragma unroll
          for (int e4 = 0; e4 < 4; e4++) {
            std::uint32_t word = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) {
              const int kk = kb * p.bk + q * 16 + e4 * 4 + e;
              const int u = u0 + tdi[kk], v = v0 + tdj[kk];
              std::int8_t val = 0;
              if (live && tdi[kk] != -128 && u >= p.g_ulo && u <= p.g_uhi && v >= p.g_vlo && v <= p.g_vhi)
                val = __ldg(pix + toff[kk]);
              word |= static_cast<std::uint32_t>(static_cast<std::uint8_t>(val)) << (8 * e);
            }
            w[e4] = word;
          }
          *reinterpret_cast<uint4*>(rowp + ((q ^ sw) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tcgen05 reads
        mbar_arrive(&full[stage]);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31 (warp % 4 rule)
    const int row = quarter * 32 + lane;
    const int ethreads = 32 * p.epi_warps;
    const int hgroups = p.epi_warps / 4, hgroup = (warp - 2) / 4;  // column halves when 8 warps
    const int sw = row & 7;  // 128B swizzle phase of this staging row
    // split: group g = hgroup owns TMEM accumulator g, staging/residual buffer g and tiles
    // blockIdx.x + g*grid, + 2*grid, ... (its own barrier and store leader), so the two
    // groups' per-tile chains (TMEM wait, math, barrier, TMA store) overlap
    const bool split = p.epi_split != 0;
    const int gthreads = split ? 128 : ethreads;
    const int gbar = split && hgroup ? 3 : 1;
    const bool leader = threadIdx.x == 64 + (split ? 128 * hgroup : 0);
    std::int32_t* thr_s = vec_s + kMaxVecK;
    if (p.epi_vec || p.fast_clamp) {
      // per-output-channel vector (e.g. the bias) as int32 in smem, read with ld.shared.v4; with
      // fast_clamp also the threshold t[k] = clamp32(lo - vec[k]): acc + res + vec >= lo
      // <=> acc + res >= t[k] exactly, because |acc + res| < 2^31 - 1
      if (p.pdl_wait) asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
      for (int k = threadIdx.x - 64; k < p.N; k += ethreads) {
        const long long vi = static_cast<long long>(p.vec_mod ? k % p.vec_mod : k) * p.vec_k;
        const std::int32_t b = !p.epi_vec ? 0
                               : p.vec_kind == kI8 ? static_cast<const std::int8_t*>(p.vec)[vi]
                               : p.vec_kind == kI16 ? static_cast<const std::int16_t*>(p.vec)[vi]
                                                    : static_cast<const std::int32_t*>(p.vec)[vi];
        vec_s[k] = b;
        if (p.fast8 && p.epi_lo && (b > p.bias_bound || b < -p.bias_bound)) atomicOr(reinterpret_cast<int*>(bars + 41), 1);
        if (p.fast_clamp) {
          const long long t = p.lo - b;
          thr_s[k] = static_cast<std::int32_t>(t < INT_MIN ? INT_MIN : t > INT_MAX ? INT_MAX : t);
        }
      }
    }
    if (p.epi_vec)  // zero tail: chunk loads past N need no bounds select
      for (int k = p.N + threadIdx.x - 64; k < (p.N + p.bn - 1) / p.bn * p.bn && k < kMaxVecK; k += ethreads) vec_s[k] = 0;
    const bool eres = p.epi_res && !p.res_mma;  // residual read by the epilogue (else added by the MMAs)
    if (eres && leader && p.pdl_wait) asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(ethreads) : "memory");
    // fast8 clamp: max(acc + res + vec, lo) in int32 when no |vec[k]| can overflow it, else the
    // exact threshold form acc + res >= clamp32(lo - vec[k]) (both keep the wrapped low byte)
    const bool fast8 = p.fast8 != 0;
    const bool thr8 = p.epi_lo && (p.thr_always || *reinterpret_cast<volatile int*>(bars + 41));
    const std::uint32_t lo32u = static_cast<std::uint32_t>(p.lo);
    const std::int32_t lo8 = p.epi_lo ? static_cast<std::int32_t>(p.lo) : INT_MIN;
    const long long lo = p.epi_lo ? p.lo : LLONG_MIN;
    const bool relu0 = p.epi_lo && p.lo == 0;
    // residual tile [128 pixels x bn channels] i8 of tile t into buffer b, as 128-channel halves
    const int hcnt = (p.bn + 127) / 128;  // 16 KB staging boxes per 128-row sub-tile
    // band mode with 64 channels: one box per band row (the TMA store pads 64-byte inner rows
    // to the 128-byte swizzle span), two 32-column chunks per 128-byte row
    const int shsh = p.band && p.vec_mod == 64 ? 1 : 2, sbox = shsh == 1 ? p.band : hcnt;
    const int res_buf = TM * p.bn, stg_buf = p.mt * sbox * 16384;
    auto load_res = [&](int t, int b) {  // (epilogue-read residual: mt == 1 only)
      const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * p.bn;
      const int halves = min(p.bn, p.N - n0 + 127) / 128;
      mbar_expect_tx(&rfull[b], BM * 128 * halves);
      for (int hh = 0; hh < halves; hh++)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                "r"(smem_u32(rstg + b * res_buf + hh * 16384)),
            "l"(reinterpret_cast<std::uint64_t>(&rmap)), "r"(smem_u32(&rfull[b])), "r"(n0 + hh * 128), "r"(m0)
            : "memory");
    };
    const int g0 = split ? hgroup : 0, tstep = split ? 2 * static_cast<int>(gridDim.x) : static_cast<int>(gridDim.x);
    if (eres && leader && static_cast<int>(blockIdx.x) + g0 * static_cast<int>(gridDim.x) < tiles)
      load_res(blockIdx.x + g0 * gridDim.x, g0);
    int iter = g0;
    for (int t = blockIdx.x + g0 * gridDim.x; t < tiles; t += tstep, iter += split ? 2 : 1) {
      const int acc = iter & 1;
      const int m0 = (t / p.tiles_n) * TM, n0 = (t % p.tiles_n) * p.bn;
      if (leader) TILE_STAMP(8, iter);
      if (p.tma_out || eres) {
        // i32 staging is single-buffered, i8 staging double-buffered (one buffer per group when split)
        if (leader && (p.tma_out == 1 || (split && p.tma_out == 2 && !p.stg4)))
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (leader && ((!split && p.tma_out == 2) || p.stg4))
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("bar.sync %0, %1;" ::"r"(gbar), "r"(gthreads) : "memory");  // staging and the older residual buffer are free
      }
      if (!split && eres && leader && t + static_cast<int>(gridDim.x) < tiles) load_res(t + gridDim.x, (iter + 1) & 1);
      mbar_wait(&tfull[acc], (iter >> 1) & 1);
      tc_fence_after();
      if (leader) TILE_STAMP(3, iter);
      if (eres) mbar_wait(&rfull[iter & 1], (iter >> 1) & 1);
      std::uint8_t* rcur = rstg + (iter & 1) * res_buf;
      // i8 staging: buffer iter & 1 (one per group when split), or iter & 3 with stg4 (a group
      // alternates between its two buffers: tile t's TMA store drains while t + 2 is staged)
      std::uint8_t* scur = p.tma_out == 2 ? stg + (iter & (p.stg4 ? 3 : 1)) * stg_buf : stg;
      const int m = m0 + row;
      // this warp's 32-column chunks: all valid chunks (split), else the valid chunks of the
      // tile divided between the two column groups
      const int nch = min(p.bn, p.N - n0 + 31) / 32;
      const int c_lo = split || hgroups == 1 ? 0 : (hgroup * nch) >> 1;
      const int c_hi = split || hgroups == 1 ? nch : ((hgroup + 1) * nch) >> 1;
      if (EXPB(64)) {  // (trace builds: no epilogue math)
      } else if (fast8 && p.epi_pipe) {
        const std::uint32_t tbase = tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) +
                                    static_cast<std::uint32_t>(acc * p.mt * p.bn);
        const std::uint32_t vaddr = smem_u32(vec_s + n0), taddr = smem_u32(thr_s + n0);
        const std::uint32_t raddr = smem_u32(rcur) + row * 128, saddr = smem_u32(scur) + row * 128;
        const int per = c_hi - c_lo;
        if (thr8 && eres) epi8_pipelined<true, true>(tbase, p.bn, p.mt, c_lo, per, vaddr, taddr, raddr, saddr, sbox, shsh, sw, lo32u, lo8, EPI_EXP);
        else if (thr8) epi8_pipelined<true, false>(tbase, p.bn, p.mt, c_lo, per, vaddr, taddr, raddr, saddr, sbox, shsh, sw, lo32u, lo8, EPI_EXP);
        else if (eres) epi8_pipelined<false, true>(tbase, p.bn, p.mt, c_lo, per, vaddr, taddr, raddr, saddr, sbox, shsh, sw, lo32u, lo8, EPI_EXP);
        else epi8_pipelined<false, false>(tbase, p.bn, p.mt, c_lo, per, vaddr, taddr, raddr, saddr, sbox, shsh, sw, lo32u, lo8, EPI_EXP);
      } else
      for (int sub = 0; sub < p.mt; sub++)
      for (int h = c_lo; h < c_hi; h++) {
        const int msub = m + sub * BM;
        std::uint32_t v[32];
#ifdef SB_TILE_TRACE
        if (p.exp & 4) {
          for (int q = 0; q < 32; q++) v[q] = 0;
        } else
#endif
        {
          const std::uint32_t ta = tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) +
                                   static_cast<std::uint32_t>(acc * p.mt * p.bn + sub * p.bn + h * 32);
          // fast8: the TMEM load is waited for only after the bias loads below were issued
          if (fast8) tmem_ld32_async(ta, v);
          else tmem_ld32(ta, v);
        }
        const int kbase = n0 + h * 32;
        if (fast8) {
          // out = wrap8(max(acc + res + vec, lo)) in int32 (exact: see IgKParams::fast8)

          std::int32_t bv[32];
#pragma unroll
          for (int q = 0; q < 8; q++) {
            if (p.epi_vec)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(bv[4 * q]), "=r"(bv[4 * q + 1]), "=r"(bv[4 * q + 2]), "=r"(bv[4 * q + 3])
                           : "r"(smem_u32(vec_s + kbase + 4 * q)));
            else
              bv[4 * q] = bv[4 * q + 1] = bv[4 * q + 2] = bv[4 * q + 3] = 0;
          }
          std::uint32_t w[8];
          tmem_wait_ld(v);
          if (eres) {
            std::uint32_t rw[8];
            const std::uint32_t rrow = smem_u32(rcur + (sub * hcnt + (h >> 2)) * 16384 + row * 128);
#pragma unroll
            for (int u = 0; u < 2; u++)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(rw[4 * u]), "=r"(rw[4 * u + 1]), "=r"(rw[4 * u + 2]), "=r"(rw[4 * u + 3])
                           : "r"(rrow + (((2 * (h & 3) + u) ^ sw) << 4)));
#pragma unroll
            for (int q = 0; q < 32; q++) {
              std::int32_t r;  // sign-extended residual byte (prmt sign-replicate selector)
              asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(rw[q >> 2]), "r"(0x8880u + 0x1111u * (q & 3)));
              v[q] = static_cast<std::uint32_t>(static_cast<std::int32_t>(v[q]) + r);
            }
          }
          if (thr8) {
            std::int32_t tv[32];
#pragma unroll
            for (int q = 0; q < 8; q++)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(tv[4 * q]), "=r"(tv[4 * q + 1]), "=r"(tv[4 * q + 2]), "=r"(tv[4 * q + 3])
                           : "r"(smem_u32(thr_s + kbase + 4 * q)));
#pragma unroll
            for (int q = 0; q < 32; q++)
              v[q] = static_cast<std::int32_t>(v[q]) >= tv[q] ? v[q] + static_cast<std::uint32_t>(bv[q]) : lo32u;
          } else {
#pragma unroll
            for (int q = 0; q < 32; q++)
              v[q] = static_cast<std::uint32_t>(max(static_cast<std::int32_t>(v[q]) + bv[q], lo8));
          }
#pragma unroll
          for (int q = 0; q < 8; q++)
            w[q] = __byte_perm(__byte_perm(v[4 * q], v[4 * q + 1], 0x0040), __byte_perm(v[4 * q + 2], v[4 * q + 3], 0x0040),
                               0x5410);
          const std::uint32_t rbase = smem_u32(scur + (sub * hcnt + (h >> 2)) * 16384 + row * 128);
#pragma unroll
          for (int u = 0; u < 2; u++)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + (((2 * (h & 3) + u) ^ sw) << 4)),
                         "r"(w[4 * u]), "r"(w[4 * u + 1]), "r"(w[4 * u + 2]), "r"(w[4 * u + 3]));
          continue;
        }
        if (p.epi) {
          // exact s32 accumulator + vector + residual in int64 (the reference's temps),
          // clamped, wrapped by the store
          int bv[32];
#pragma unroll
          for (int q = 0; q < 8; q++) {
            if (p.epi_vec || p.fast_clamp)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(bv[4 * q]), "=r"(bv[4 * q + 1]), "=r"(bv[4 * q + 2]), "=r"(bv[4 * q + 3])
                           : "r"(smem_u32(vec_s + (kbase + 4 * q < p.N ? kbase + 4 * q : 0))));
            else
              bv[4 * q] = bv[4 * q + 1] = bv[4 * q + 2] = bv[4 * q + 3] = 0;
          }
          std::uint32_t rw[8];
          if (eres) {
            const std::uint32_t rrow = smem_u32(rcur + (sub * hcnt + (h >> 2)) * 16384 + row * 128);
#pragma unroll
            for (int u = 0; u < 2; u++)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(rw[4 * u]), "=r"(rw[4 * u + 1]), "=r"(rw[4 * u + 2]), "=r"(rw[4 * u + 3])
                           : "r"(rrow + (((2 * (h & 3) + u) ^ sw) << 4)));
          }
          if (!p.epi_lo) {
            // no clamp: only the wrapped low bits reach the store
#pragma unroll
            for (int q = 0; q < 32; q++) {
              const std::uint32_t r = eres ? static_cast<std::uint32_t>(
                                                      static_cast<std::int32_t>(static_cast<std::int8_t>(rw[q >> 2] >> (8 * (q & 3)))))
                                                : 0u;
              v[q] = v[q] + static_cast<std::uint32_t>(bv[q]) + r;
            }
          } else if (p.fast_clamp) {
            int tv[32];
#pragma unroll
            for (int q = 0; q < 8; q++)
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(tv[4 * q]), "=r"(tv[4 * q + 1]), "=r"(tv[4 * q + 2]), "=r"(tv[4 * q + 3])
                           : "r"(smem_u32(thr_s + (kbase + 4 * q < p.N ? kbase + 4 * q : 0))));
            const std::uint32_t lo32 = static_cast<std::uint32_t>(p.lo);
#pragma unroll
            for (int q = 0; q < 32; q++) {
              const std::int32_t r = eres ? static_cast<std::int32_t>(static_cast<std::int8_t>(rw[q >> 2] >> (8 * (q & 3))))
                                               : 0;
              const std::int32_t ar = static_cast<std::int32_t>(v[q]) + r;
              v[q] = ar >= tv[q] ? static_cast<std::uint32_t>(ar) + static_cast<std::uint32_t>(bv[q]) : lo32;
            }
          } else if (relu0) {
            // exact x = acc + vec (+ res) as a 64-bit (hi:lo) carry chain; ReLU keeps lo iff hi >= 0
#pragma unroll
            for (int q = 0; q < 32; q++) {
              const std::uint32_t r = eres ? static_cast<std::uint32_t>(
                                                      static_cast<std::int32_t>(static_cast<std::int8_t>(rw[q >> 2] >> (8 * (q & 3)))))
                                                : 0u;
              std::uint32_t lo32;
              std::int32_t hi32;
              asm("{\n\t.reg .s32 sa, sb, sr;\n\t"
                  "shr.s32 sa, %2, 31;\n\t"
                  "shr.s32 sb, %3, 31;\n\t"
                  "shr.s32 sr, %4, 31;\n\t"
                  "add.cc.u32 %0, %2, %3;\n\t"
                  "addc.cc.s32 %1, sa, sb;\n\t"
                  "add.cc.u32 %0, %0, %4;\n\t"
                  "addc.s32 %1, %1, sr;\n\t}"
                  : "=r"(lo32), "=r"(hi32)
                  : "r"(v[q]), "r"(bv[q]), "r"(r));
              v[q] = hi32 < 0 ? 0u : lo32;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 32; q++) {
              long long x = static_cast<long long>(static_cast<std::int32_t>(v[q])) + bv[q];
              if (eres) x += static_cast<std::int8_t>(rw[q >> 2] >> (8 * (q & 3)));
              v[q] = static_cast<std::uint32_t>(x < lo ? lo : x);
            }
          }
        }
        if (p.tma_out == 1) {
          const std::uint32_t rbase = smem_u32(stg + h * 16384 + row * 128);
#pragma unroll
          for (int q = 0; q < 8; q++)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((q ^ sw) << 4)), "r"(v[4 * q]),
                         "r"(v[4 * q + 1]), "r"(v[4 * q + 2]), "r"(v[4 * q + 3]));
        } else if (p.tma_out == 2) {
          // i8: this row's 32 channels -> two swizzled 16-byte chunks of a 128-byte row
          std::uint32_t w[8];
#pragma unroll
          for (int q = 0; q < 8; q++)
            w[q] = (v[4 * q] & 0xFF) | ((v[4 * q + 1] & 0xFF) << 8) | ((v[4 * q + 2] & 0xFF) << 16) |
                   (v[4 * q + 3] << 24);
          const std::uint32_t rbase = smem_u32(scur + (sub * sbox + (h >> shsh)) * 16384 + row * 128);
#pragma unroll
          for (int u = 0; u < 2; u++)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + (((2 * (h & ((1 << shsh) - 1)) + u) ^ sw) << 4)),
                         "r"(w[4 * u]), "r"(w[4 * u + 1]), "r"(w[4 * u + 2]), "r"(w[4 * u + 3]));
        } else if (msub < p.M) {
          const long long rowbase = static_cast<long long>(msub) * p.ldc;
          for (int q = 0; q < 32; q++) {
            const int n = kbase + q;
            if (n >= p.N) break;
            const long long idx = rowbase + n;
            if (p.out_kind == kI32) {
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
#ifdef SB_TILE_TRACE
      if (p.band && (p.exp & 32)) {
        // debug: staging row = (row, 100 + row) per band row p, same swizzle as the epilogue
        for (int c = 0; c < 8; c++) {
          const std::uint32_t val = (c < 4 ? row : 100 + row) & 0xFF;
          const std::uint32_t v4 = val * 0x01010101u;
          asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(smem_u32(scur) + row * 128 + ((c ^ sw) << 4)), "r"(v4));
        }
      }
#endif
      if (leader) TILE_STAMP(9, iter);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (p.tma_out || split) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync %0, %1;" ::"r"(gbar), "r"(gthreads) : "memory");
        // split: the group's residual buffer is free again -> prefetch its next tile's
        if (split && eres && leader && t + tstep < tiles) load_res(t + tstep, g0);
      }
      if (p.tma_out) {
        if (leader) {
          if (p.tma_out == 1) {
            for (int h = 0; h < BN / 32; h++)
              if (n0 + h * 32 < p.N)
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                 reinterpret_cast<std::uint64_t>(&cmap)),
                             "r"(smem_u32(stg + h * 16384)), "r"(n0 + h * 32), "r"(m0)
                             : "memory");
          } else if (p.strip) {
            // (k, pixel, row, image) per 128-row sub-tile (2 output rows x 64-pixel pitch):
            // pixels past the row width and rows past the image are clipped
            const int img = t / p.strip_tx, x0 = (t - img * p.strip_tx) * p.strip_rows;
            for (int sub = 0; sub < p.mt; sub++)
              for (int hh = 0; hh < p.bn / 128 || hh == 0; hh++) {
                if (n0 + hh * 128 >= p.N) break;
                asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                                 reinterpret_cast<std::uint64_t>(&cmap)),
                             "r"(smem_u32(scur + (sub * hcnt + hh) * 16384)), "r"(n0 + hh * 128), "r"(0),
                             "r"(x0 + sub * 2), "r"(img)
                             : "memory");
              }
          } else if (p.band) {
            // (k, row of the band, pixel, band index): pixels past the row width are clipped
            // one 16 KB box per band row
            for (int hh = 0; hh < p.band && !EXPB(2048); hh++)
              asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                               reinterpret_cast<std::uint64_t>(&cmap)),
                           "r"(smem_u32(scur + hh * 16384)), "r"(0), "r"(hh), "r"(0), "r"(t)
                           : "memory");
          } else {
            for (int sub = 0; sub < p.mt; sub++)
              for (int hh = 0; hh < p.bn / 128 && n0 + hh * 128 < p.N; hh++)
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                 reinterpret_cast<std::uint64_t>(&cmap)),
                             "r"(smem_u32(scur + (sub * hcnt + hh) * 16384)), "r"(n0 + hh * 128), "r"(m0 + sub * BM)
                             : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          TILE_STAMP(4, iter);
        }
      }
    }
    if (p.tma_out && leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

template <class F>
F driver_fn(const char* name) {
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<F>(f);
  return nullptr;
}

constexpr int kSmemMax = 227 * 1024;

struct Geometry {
  std::int64_t Hin, Win;       // input window extents (tensor map dims)
  int lower_h, lower_w, upper_h, upper_w;
  int bk;
};

bool geometry(const ConvPlan& cp, Geometry* g) {
  g->Hin = cp.u_hi - cp.u_lo + 1;
  g->Win = cp.v_hi - cp.v_lo + 1;
  // the window origin of output x is u = sx*x (+ tap i); relative to the map origin u_lo
  g->lower_h = static_cast<int>(-cp.u_lo);
  g->lower_w = static_cast<int>(-cp.v_lo);
  g->upper_h = static_cast<int>(cp.sx * (cp.H - 1) - cp.u_lo - (g->Hin - 1));
  g->upper_w = static_cast<int>(cp.sy * (cp.W - 1) - cp.v_lo - (g->Win - 1));
  g->bk = cp.C % 128 == 0 ? 128 : 64;
  auto corner = [](std::int64_t v) { return v >= -128 && v <= 127; };
  return corner(-cp.u_lo) && corner(-cp.v_lo) && corner(cp.sx * (cp.H - 1) - cp.u_lo - (g->Hin - 1)) &&
         corner(cp.sy * (cp.W - 1) - cp.v_lo - (g->Win - 1));
}

struct Prepared {
  ConvPlan cp;
  const void *a, *b, *vec, *res;
  void* c;
  IgKParams kp;
  CUtensorMap amap, bmap, cmap, rmap;
};

std::mutex g_mu;
std::vector<Prepared>* g_prep = nullptr;

bool same(const ConvPlan& x, const ConvPlan& y) {
  return x.N == y.N && x.H == y.H && x.W == y.W && x.C == y.C && x.K == y.K && x.R == y.R && x.S == y.S &&
         x.sx == y.sx && x.sy == y.sy && x.a_n == y.a_n && x.a_x == y.a_x && x.a_y == y.a_y && x.a0 == y.a0 &&
         x.u_lo == y.u_lo && x.u_hi == y.u_hi && x.v_lo == y.v_lo && x.v_hi == y.v_hi && x.b_i == y.b_i &&
         x.b_j == y.b_j && x.b_k == y.b_k && x.b0 == y.b0 && x.c_n == y.c_n && x.c_x == y.c_x && x.c_y == y.c_y &&
         x.c0 == y.c0 && x.c_dtype == y.c_dtype && x.fresh_output == y.fresh_output && x.epi == y.epi &&
         x.epi_vec == y.epi_vec && x.epi_lo == y.epi_lo && x.vec_k == y.vec_k && x.vec_c == y.vec_c && x.lo == y.lo &&
         x.epi_res == y.epi_res && x.res_c0 == y.res_c0 && x.res_pix == y.res_pix && x.fold_band == y.fold_band &&
         x.band_raw == y.band_raw && x.raw_a_n == y.raw_a_n && x.raw_a_x == y.raw_a_x && x.raw_a0 == y.raw_a0 &&
         x.raw_u_lo == y.raw_u_lo && x.raw_u_hi == y.raw_u_hi && x.raw_v_lo == y.raw_v_lo && x.raw_v_hi == y.raw_v_hi;
}

int kind_of(DType d) { return d == DType::I8 ? kI8 : d == DType::I16 ? kI16 : kI32; }

cudaError_t prepare(const ConvPlan& cp, const ConvArgs& args, Prepared* out) {
  out->cp = cp;
  out->a = args.a;
  out->b = args.b;
  out->c = args.c;
  out->vec = args.vec;
  out->res = args.res;
  auto enc_tiled = driver_fn<PFN_cuTensorMapEncodeTiled_v12000>("cuTensorMapEncodeTiled");
  auto enc_im2col = driver_fn<PFN_cuTensorMapEncodeIm2col_v12000>("cuTensorMapEncodeIm2col");
  if (!enc_tiled || !enc_im2col) return cudaErrorNotSupported;
  const ConvPlan gp = cp.packed ? packed_view(cp) : cp;  // GEMM geometry (B map, K blocks)
  Geometry g;
  if (!geometry(gp, &g)) return cudaErrorNotSupported;
  IgKParams& kp = out->kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.M = static_cast<int>(cp.N * cp.H * cp.W);
  kp.N = static_cast<int>(cp.K);
  kp.P = static_cast<int>(cp.H);
  kp.Q = static_cast<int>(cp.W);
  kp.sx = static_cast<int>(cp.sx);
  kp.sy = static_cast<int>(cp.sy);
  kp.lower_h = g.lower_h;
  kp.lower_w = g.lower_w;
  kp.S = static_cast<int>(gp.S);
  kp.bk = g.bk;
  kp.cblocks = static_cast<int>(gp.C / g.bk);
  kp.kblocks = static_cast<int>(gp.R * gp.S) * kp.cblocks;
  kp.epi_warps = cp.packed ? 4 : 8;
  if (cp.fold_band) {
    // band view (packed_view of a band-folded conv): cp.H x cp.W output rows/cols, cp.K =
    // band x the output channels, cp.a_x / cp.a_n = folded row / image bytes
    const int band = static_cast<int>(cp.fold_band);
    kp.band = band;
    kp.band_rowb = cp.a_x;
    kp.band_img = cp.a_n;
    kp.band_rpi = static_cast<int>(cp.H / band);
    // the band's kblocks folded rows; the last row up to pixel 127 + (C / a_y - 1) (junk rows
    // of the tile read past the row: finite, discarded by the clipped store)
    kp.band_bytes = static_cast<int>((kp.kblocks - 1) * cp.a_x + (BM + cp.C / cp.a_y - 1) * cp.a_y);
    kp.band_bytes = (kp.band_bytes + 15) / 16 * 16;
    // whole KB stages keep every later region (filter SW64, staging SW128) 1024-byte aligned
    kp.band_stage = (kp.band_bytes + 1023) / 1024 * 1024;
    kp.band_src = static_cast<const std::int8_t*>(args.a);
    kp.vec_mod = static_cast<int>(cp.K / band);
    if (cp.band_raw) {
      kp.band_raw = 1;
      kp.raw_fv = static_cast<int>(cp.fold_v);
      kp.raw_chunks = static_cast<int>((cp.raw_v_hi - cp.raw_v_lo + 1) * 3 / 16);
      kp.raw_col0 = static_cast<int>((3 * cp.raw_v_lo + 15) / 16 * 16);
      // bytes read per row: up to window column 2 fold_v - 1 plus the 12-byte word window
      kp.raw_rp = (kp.raw_col0 + 6 * kp.raw_fv + 16 + 15) / 16 * 16;
      kp.raw_stage = (2 * kp.kblocks * kp.raw_rp + 127) / 128 * 128;
      kp.r_an = cp.raw_a_n;
      kp.r_ax = cp.raw_a_x;
      kp.r_a0 = cp.raw_a0;
      kp.r_ulo = static_cast<int>(cp.raw_u_lo);
      kp.r_uhi = static_cast<int>(cp.raw_u_hi);
      kp.r_vlo = static_cast<int>(cp.raw_v_lo);
    }
    kp.M = static_cast<int>(cp.N * kp.band_rpi * BM);
    // K-major, no swizzle: core matrices of 8 rows x 16 bytes (rows 16 bytes apart), LBO (low
    // word, 16 bytes) between core matrices along K, SBO (high word, 128 bytes) between 8-row
    // groups along M -- measured on B200 by tools/microbench/desc_probe.cu -- so row m, byte q
    // of the operand is at start + 16 m + q: overlapping 64-byte windows
    kp.a_hi = (128u >> 4) | (1u << 14);
  }
  if (cp.packed) {
    kp.gather = 1;
    kp.rsc = static_cast<int>(cp.R * cp.S * cp.C);
    kp.g_C = static_cast<int>(cp.C);
    kp.g_S = static_cast<int>(cp.S);
    kp.g_R = static_cast<int>(cp.R);
    kp.g_an = cp.a_n;
    kp.g_ax = cp.a_x;
    kp.g_ay = cp.a_y;
    kp.g_a0 = cp.a0;
    kp.g_ulo = static_cast<int>(cp.u_lo);
    kp.g_uhi = static_cast<int>(cp.u_hi);
    kp.g_vlo = static_cast<int>(cp.v_lo);
    kp.g_vhi = static_cast<int>(cp.v_hi);
    kp.g_in = static_cast<const std::int8_t*>(args.a);
    kp.g_run = static_cast<int>(cp.pack_run);
  }
  kp.mt = 1;
  kp.tiles_m = (kp.M + BM - 1) / BM;  // final value from layout() below
  kp.bn = 128;
  kp.tiles_n = (kp.N + BN - 1) / BN;  // final value from layout() below
  kp.fresh = cp.fresh_output ? 1 : 0;
  kp.out_kind = kind_of(cp.c_dtype);
  kp.ldc = cp.c_y;
  const int ob = kp.out_kind == kI8 ? 1 : kp.out_kind == kI16 ? 2 : 4;
  kp.c = static_cast<char*>(args.c) + cp.c0 * ob;
  kp.epi = cp.epi ? 1 : 0;
  kp.epi_vec = cp.epi_vec ? 1 : 0;
  kp.epi_lo = cp.epi_lo ? 1 : 0;
  kp.epi_res = cp.epi_res ? 1 : 0;
  {
    const long long taps = cp.packed ? cp.R * cp.S * cp.C : gp.R * gp.S * gp.C;
    kp.fast_clamp = cp.epi_lo && cp.K <= kMaxVecK && taps * 128 * 128 + 128 < (1ll << 31) - 1 ? 1 : 0;
  }
  kp.lo = cp.lo;
  kp.vec_k = cp.vec_k;
  kp.vec_kind = args.vec_kind;
  if (cp.epi_vec) {
    const int vb = args.vec_kind == kI8 ? 1 : args.vec_kind == kI16 ? 2 : 4;
    kp.vec = static_cast<const char*>(args.vec) + cp.vec_c * vb;
  }
  {
    const std::uintptr_t cbase = reinterpret_cast<std::uintptr_t>(kp.c);
    if (kp.fresh && kp.out_kind == kI32 && (kp.ldc * 4) % 16 == 0 && cbase % 16 == 0) kp.tma_out = 1;
    else if (kp.fresh && kp.out_kind == kI8 && kp.ldc % 16 == 0 && cbase % 16 == 0) kp.tma_out = 2;
    else kp.tma_out = 0;
  }
  {
    const long long taps = cp.packed ? cp.R * cp.S * cp.C : gp.R * gp.S * gp.C;
    const long long T = taps * 128 * 128 + 128;  // bound on |acc + res|
    const bool lo_ok = !cp.epi_lo || (cp.lo >= INT_MIN && cp.lo <= INT_MAX && T < INT_MAX);
    // i8 epilogue in int32: no clamp (wrapped low bits), or a clamp decided exactly by max()
    // (small biases, lo in int32) or by the per-channel threshold (needs the fast_clamp bound)
    kp.fast8 = kp.tma_out == 2 && cp.K <= kMaxVecK && (!cp.epi_lo || kp.fast_clamp) ? 1 : 0;
    kp.thr_always = cp.epi_lo && !lo_ok ? 1 : 0;
    kp.epi_pipe = kp.fast8;
    kp.epi_split = kp.epi_warps == 8 && kp.tma_out != 1 && !std::getenv("SB_IG_NOSPLIT") ? 1 : 0;
    kp.bias_bound = T < INT_MAX ? INT_MAX - T : 0;
  }
  // strip mode (see IgKParams::strip): stride-1 3x3 over exactly 64 channels, rows fit a
  // 64-pixel pitch, fresh i8 output written by the TMA store, resident filter
  if (!kp.gather && !cp.fold_band && cp.R == 3 && cp.S == 3 && cp.sx == 1 && cp.sy == 1 && cp.C == 64 &&
      cp.W + 2 <= 64 && kp.tma_out == 2 && !cp.epi_res && cp.K <= 256 && !std::getenv("SB_IG_NOSTRIP") &&
      cp.c_x == cp.W * cp.c_y && (cp.N == 1 || cp.c_n == cp.H * cp.c_x) && cp.c_y % 16 == 0)
    kp.strip = 1;
  // dynamic smem: A/B ring (up to 128 KB) | resident filter | output staging | residual tiles |
  // vector | gather table | barriers, for tile width bn (false: does not fit)
  const int bres_cap = (std::getenv("SB_IG_BRES_KB") ? std::atoi(std::getenv("SB_IG_BRES_KB")) : 96) * 1024;
  auto layout = [&](int bn, int mt) -> bool {
    kp.bn = bn;
    kp.mt = mt;
    kp.tiles_n = (kp.N + bn - 1) / bn;
    kp.tiles_m = (kp.M + BM * mt - 1) / (BM * mt);
    const int sboxes = kp.band && kp.vec_mod == 64 ? kp.band : bn / 128;  // 16 KB staging boxes per sub-tile
    const int stg = kp.tma_out == 1 ? kStgBytes : kp.tma_out == 2 ? (kp.stg4 ? 4 : 2) * mt * sboxes * 16384 : 0;
    const int res = kp.epi_res ? (kp.res1 ? 1 : 2) * BM * mt * bn : 0;
    const int vec = kp.fast_clamp ? 2 * kVecBytes : kp.epi_vec ? kVecBytes : 0;
    const int tab = kp.gather ? (kp.kblocks * kp.bk * 6 + 15) / 16 * 16 : 0;
    const int ident = kp.res_mma ? 1024 : 0;
    const int rawb = kp.band_raw ? kRawStages * kp.raw_stage : 0;
    // the filter stays resident when there is one n-tile and it is small (<= 96 KB)
    kp.bn_box = kp.N <= 64 ? 64 : bn;
    const int bres = (kp.tiles_n == 1 || kp.nstat) && kp.kblocks * kp.bn_box * g.bk <= bres_cap &&
                             !std::getenv("SB_IG_NOBRES")
                         ? kp.kblocks * kp.bn_box * g.bk : 0;
    kp.b_res = bres ? 1 : 0;
    if (kp.nstat && !bres) return false;
    const int kstage = (BM * mt + (bres ? 0 : kp.bn_box)) * g.bk;  // one k-block's A (+ B)
    const int avail = std::min(kRingBytes, kSmemMax - 1024 - 512 - stg - res - vec - tab - bres - ident - rawb);
    // k-blocks per stage: up to 4 while three stages still fit (gather mode: 1)
    kp.kpb = 1;
    if (kp.band || kp.strip) kp.kpb = kp.kblocks;  // one load per tile feeds every k-block
    else if (!kp.gather && !std::getenv("SB_IG_KPB1"))
      for (int c : {4, 3, 2})
        if (kp.kblocks % c == 0 && (std::getenv("SB_IG_KPB3") ? 3 : 2) * c * kstage <= avail) {
          kp.kpb = c;
          break;
        }
    if (kp.strip) {
      kp.strip_rows = 2 * mt;
      kp.strip_tx = static_cast<int>((cp.H + kp.strip_rows - 1) / kp.strip_rows);
      kp.strip_stage = (kp.strip_rows + 2) * 64 * 64;
      kp.tiles_m = static_cast<int>(cp.N) * kp.strip_tx;
    }
    const int stage = kp.band ? kp.band_stage : kp.strip ? kp.strip_stage : kp.kpb * kstage;
    if (avail < 2 * stage) return false;
    int ring = avail / stage * stage;
    kp.stages = std::min(16, ring / stage);
    ring = kp.stages * stage;
    kp.bres_off = ring;
    ring += bres;
    kp.stg_off = ring;
    kp.res_off = ring + stg;
    kp.ident_off = ring + stg + res;
    ring += ident;
    kp.vec_off = ring + stg + res;
    kp.tab_off = ring + stg + res + vec;
    kp.raw_off = kp.tab_off + tab;
    kp.bar_off = kp.raw_off + rawb;
    kp.smem = 1024 + kp.bar_off + 512;
    return true;
  };
  kp.res_mma = kp.epi_res && !kp.gather && kp.epi_split && !std::getenv("SB_IG_RESEPI") ? 1 : 0;
  // 256-wide tiles (N = 256 MMAs: half the instructions and A re-reads) for wide outputs
  const bool wide = kp.epi_split && kp.N >= 256 && cp.K <= kMaxVecK && !std::getenv("SB_IG_BN128");
  // two 128-row sub-tiles per tile (one stage handshake and one filter tile feed twice the
  // MMAs) for narrow outputs with enough tiles left for every SM
  const bool tall = !kp.band && kp.epi_split && kp.tma_out != 1 && kp.N <= 128 && !(kp.epi_res && !kp.res_mma) &&
                    (kp.M + 2 * BM - 1) / (2 * BM) >= 2 * 148 && !std::getenv("SB_IG_MT1");
  // split i8 epilogue: two staging buffers per group when the ring keeps >= 3 stages
  // (band mode: the ring depth matters more -- one bulk copy per tile with DRAM latency to hide)
  const bool stg4_ok = kp.epi_split && kp.tma_out == 2 && (!kp.band || std::getenv("SB_IG_BAND_STG4")) &&
                       !std::getenv("SB_IG_STG2");
  // n-stationary resident filter slices when several n-tiles each fit (see IgKParams::nstat)
  const bool nstat_ok = !kp.gather && !kp.band && !kp.strip && !std::getenv("SB_IG_NONSTAT");
  auto try_layout = [&](int bn, int mt, bool nstat, bool stg4, bool res1, int min_stages) {
    kp.nstat = nstat ? 1 : 0;
    kp.stg4 = stg4 ? 1 : 0;
    kp.res1 = res1 ? 1 : 0;
    return layout(bn, mt) && kp.stages >= min_stages;
  };
  const int max_tn = std::getenv("SB_IG_NSTAT8") ? 8 : 16;
  // the second staging buffer per epilogue group (stg4) only when the ring keeps >= 3 stages
  // AND as many k-blocks per stage as without it (fewer, larger handshakes win: measured)
  auto pick = [&](int bn, int mt, bool nstat, bool res1, int min_stages) {
    if (!try_layout(bn, mt, nstat, false, res1, min_stages)) return false;
    const int kpb2 = kp.kpb;
    if (stg4_ok && try_layout(bn, mt, nstat, true, res1, 3) && (kp.kpb >= kpb2 || std::getenv("SB_IG_STG4_ANY")))
      return true;
    return try_layout(bn, mt, nstat, false, res1, min_stages);
  };
  auto shape_nstat = [&](int bn, int mt) {
    const int tn = (kp.N + bn - 1) / bn;
    if (!nstat_ok || tn < 2 || tn > max_tn) return false;
    if (pick(bn, mt, true, false, 2)) return true;
    return kp.res_mma && pick(bn, mt, true, true, 2);
  };
  auto shape = [&](int bn, int mt) { return pick(bn, mt, false, false, 0); };
  // one 256-wide n-tile with the whole filter resident first, then n-stationary slices
  // (256-wide, then 128-wide tiles), then the streamed shapes
  const bool single_res = wide && (kp.N + 255) / 256 == 1 && shape(256, 1) && kp.b_res;
  if (!single_res && !(wide && shape_nstat(256, 1)) && !shape_nstat(128, 1) && !(wide && shape(256, 1)) &&
      !(tall && shape(128, 2)) && !shape(128, 1))
    return cudaErrorNotSupported;
  // idesc: S32 accumulate, signed A/B, both K-major, N = 128, M = 128
  kp.idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  // descriptor high word: SBO = 8 rows x row bytes, version 1, swizzle 128B (2) / 64B (4)
  kp.desc_hi = g.bk == 128 ? ((1024u >> 4) | (1u << 14) | (2u << 29)) : ((512u >> 4) | (1u << 14) | (4u << 29));
  const CUtensorMapSwizzle sw = g.bk == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;

  std::memset(&out->amap, 0, sizeof(out->amap));
  if (kp.band && (kp.tma_out != 2 || !kp.b_res || kp.bn != kp.N || kp.mt != 1)) return cudaErrorNotSupported;
  if (kp.strip && (!kp.b_res || kp.tiles_n != 1)) kp.strip = 0;  // (layout() ran with strip: redo without)
  if (!kp.strip && kp.strip_stage) {
    kp.strip_stage = 0;
    if (!(wide && shape(256, 1)) && !(tall && shape(128, 2)) && !shape(128, 1)) return cudaErrorNotSupported;
  }
  if (kp.band && reinterpret_cast<std::uintptr_t>(args.a) % 16) return cudaErrorMisalignedAddress;
  if (kp.strip) {
    // A: the input window as (c, v, u, n) from the corner (u_lo, v_lo); box = haloed strip
    const std::int8_t* abase = static_cast<const std::int8_t*>(args.a) + cp.a0 + cp.a_x * cp.u_lo + cp.a_y * cp.v_lo;
    if (reinterpret_cast<std::uintptr_t>(abase) % 16 || cp.a_y % 16 || cp.a_x % 16 || cp.a_n % 16)
      return cudaErrorMisalignedAddress;
    cuuint64_t adim[4] = {64, static_cast<cuuint64_t>(cp.v_hi - cp.v_lo + 1), static_cast<cuuint64_t>(cp.u_hi - cp.u_lo + 1),
                          static_cast<cuuint64_t>(cp.N)};
    cuuint64_t astr[3] = {static_cast<cuuint64_t>(cp.a_y), static_cast<cuuint64_t>(cp.a_x),
                          static_cast<cuuint64_t>(cp.a_n)};
    cuuint32_t abox[4] = {64u, 64u, static_cast<cuuint32_t>(kp.strip_rows + 2), 1u};
    cuuint32_t aes[4] = {1, 1, 1, 1};
    kp.strip_uoff = static_cast<int>(cp.ox - cp.u_lo);
    kp.strip_voff = static_cast<int>(cp.oy - cp.v_lo);
    if (enc_tiled(&out->amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<std::int8_t*>(abase), adim, astr, abox, aes,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (!kp.gather && !kp.band && !kp.strip) {
  // A: im2col over (c, v, u, n) from the window corner (u_lo, v_lo)
  const std::int8_t* abase = static_cast<const std::int8_t*>(args.a) + cp.a0 + cp.a_x * cp.u_lo + cp.a_y * cp.v_lo;
  if (reinterpret_cast<std::uintptr_t>(abase) % 16) return cudaErrorMisalignedAddress;
  cuuint64_t adim[4] = {static_cast<cuuint64_t>(cp.C), static_cast<cuuint64_t>(g.Win), static_cast<cuuint64_t>(g.Hin),
                        static_cast<cuuint64_t>(cp.N)};
  cuuint64_t astr[3] = {static_cast<cuuint64_t>(cp.a_y), static_cast<cuuint64_t>(cp.a_x),
                        static_cast<cuuint64_t>(cp.a_n)};
  int lower[2] = {g.lower_w, g.lower_h};  // innermost first: {W, H}
  int upper[2] = {g.upper_w, g.upper_h};
  cuuint32_t aes[4] = {1, static_cast<cuuint32_t>(cp.sy), static_cast<cuuint32_t>(cp.sx), 1};
  if (enc_im2col(&out->amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<std::int8_t*>(abase), adim, astr, lower,
                 upper, static_cast<cuuint32_t>(g.bk), static_cast<cuuint32_t>(BM * kp.mt), aes,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  }
  // B: filter as (c, k, j, i), box (bk, 128, 1, 1) (the packed [K, pack_k] filter in gather mode)
  const std::int8_t* bbase = static_cast<const std::int8_t*>(args.b) + gp.b0;
  if (reinterpret_cast<std::uintptr_t>(bbase) % 16) return cudaErrorMisalignedAddress;
  cuuint64_t bdim[4] = {static_cast<cuuint64_t>(gp.C), static_cast<cuuint64_t>(gp.K), static_cast<cuuint64_t>(gp.S),
                        static_cast<cuuint64_t>(gp.R)};
  cuuint64_t bstr[3] = {static_cast<cuuint64_t>(gp.b_k), static_cast<cuuint64_t>(gp.S > 1 ? gp.b_j : gp.b_k * gp.K),
                        static_cast<cuuint64_t>(gp.R > 1 ? gp.b_i : gp.b_k * gp.K * gp.S)};
  cuuint32_t bbox[4] = {static_cast<cuuint32_t>(g.bk), static_cast<cuuint32_t>(kp.bn_box), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (enc_tiled(&out->bmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<std::int8_t*>(bbase), bdim, bstr, bbox, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  std::memset(&out->cmap, 0, sizeof(out->cmap));
  if (kp.tma_out == 1) {
    cuuint64_t cdim[2] = {static_cast<cuuint64_t>(kp.N), static_cast<cuuint64_t>(kp.M)};
    cuuint64_t cstr[1] = {static_cast<cuuint64_t>(kp.ldc * 4)};
    cuuint32_t cbox[2] = {32, BM};
    if (enc_tiled(&out->cmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, kp.c, cdim, cstr, cbox, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else if (kp.tma_out == 2 && kp.strip) {
    // (k, pixel, row, image), box (<= 128 channels, 64 pixels, 2 rows, 1): 128-byte padded rows
    cuuint64_t cdim[4] = {static_cast<cuuint64_t>(cp.K), static_cast<cuuint64_t>(cp.W), static_cast<cuuint64_t>(cp.H),
                          static_cast<cuuint64_t>(cp.N)};
    cuuint64_t cstr[3] = {static_cast<cuuint64_t>(cp.c_y), static_cast<cuuint64_t>(cp.c_x),
                          static_cast<cuuint64_t>(cp.N > 1 ? cp.c_n : cp.c_x * cp.H)};
    cuuint32_t cbox[4] = {static_cast<cuuint32_t>(std::min<long long>(cp.K, 128)), 64, 2, 1};
    if (enc_tiled(&out->cmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, kp.c, cdim, cstr, cbox, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else if (kp.tma_out == 2 && kp.band) {
    // (k, band row p, pixel y, band index nu): element (n, band * u + p, y, k) of the NHWC output
    const long long ko = cp.K / kp.band;
    cuuint64_t cdim[4] = {static_cast<cuuint64_t>(ko), static_cast<cuuint64_t>(kp.band), static_cast<cuuint64_t>(cp.W),
                          static_cast<cuuint64_t>(cp.N * kp.band_rpi)};
    cuuint64_t cstr[3] = {static_cast<cuuint64_t>(cp.c_x), static_cast<cuuint64_t>(cp.c_y),
                          static_cast<cuuint64_t>(kp.band * cp.c_x)};
    cuuint32_t cbox[4] = {static_cast<cuuint32_t>(ko), 1, BM, 1};
    if (enc_tiled(&out->cmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, kp.c, cdim, cstr, cbox, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else if (kp.tma_out == 2) {
    cuuint64_t cdim[2] = {static_cast<cuuint64_t>(kp.N), static_cast<cuuint64_t>(kp.M)};
    cuuint64_t cstr[1] = {static_cast<cuuint64_t>(kp.ldc)};
    cuuint32_t cbox[2] = {BN, BM};
    if (enc_tiled(&out->cmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, kp.c, cdim, cstr, cbox, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  std::memset(&out->rmap, 0, sizeof(out->rmap));
  if (kp.epi_res) {
    const std::int8_t* rbase = static_cast<const std::int8_t*>(args.res) + cp.res_c0;
    if (reinterpret_cast<std::uintptr_t>(rbase) % 16 || cp.res_pix % 16) return cudaErrorMisalignedAddress;
    cuuint64_t rdim[2] = {static_cast<cuuint64_t>(kp.N), static_cast<cuuint64_t>(kp.M)};
    cuuint64_t rstr[1] = {static_cast<cuuint64_t>(cp.res_pix)};
    cuuint32_t rbox[2] = {BN, BM};
    if (enc_tiled(&out->rmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<std::int8_t*>(rbase), rdim, rstr, rbox, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (std::getenv("SB_IG_SHOW"))  // development aid: the chosen layout per prepared conv
    std::fprintf(stderr,
                 "igemm M=%d N=%d C=%lld R=%lld bn=%d mt=%d tiles=%dx%d kblocks=%d kpb=%d stages=%d b_res=%d nstat=%d "
                 "stg4=%d res1=%d res_mma=%d split=%d band=%d strip=%d gather=%d tma_out=%d smem=%d\n",
                 kp.M, kp.N, static_cast<long long>(cp.C), static_cast<long long>(cp.R), kp.bn, kp.mt, kp.tiles_m,
                 kp.tiles_n, kp.kblocks, kp.kpb, kp.stages, kp.b_res, kp.nstat, kp.stg4, kp.res1, kp.res_mma,
                 kp.epi_split, kp.band, kp.strip, kp.gather, kp.tma_out, kp.smem);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(conv_igemm_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return cudaSuccess;
}

// kk layout: dense (i, j, c) when run == 0, else i * run + (j * C + c) with zero padding
__global__ void conv_pack_filter_kernel(const std::int8_t* __restrict__ b, std::int8_t* __restrict__ pb, int K, int C,
                                        int R, int S, int run, int kp, long long b_i, long long b_j, long long b_k,
                                        long long b_c, long long b0) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < K * kp; g += gridDim.x * blockDim.x) {
    const int k = g / kp, kk = g - k * kp;
    int i, jc;
    if (run) {
      i = kk / run;
      jc = kk - i * run;
    } else {
      i = kk / (S * C);
      jc = kk - i * S * C;
    }
    std::int8_t val = 0;
    if (i < R && jc < S * C) {
      const int c = jc % C, j = jc / C;
      val = b[b0 + b_i * i + b_j * j + b_k * k + b_c * c];
    }
    pb[g] = val;
  }
}

// Folded pixels F[n, U, V, kf], kf = (di*fy + dj)*C + c: I[n, fx*U + di, fy*V + dj, c] (zero
// outside the constraint window and on the padding bytes up to fold_c).  Specialised: one
// thread per folded pixel, unrolled (the ResNet stem is FX = FY = 2, C = 3: 12 of 16 bytes).
// ROWS (fold_c == 16): the folded pixel (n, U, V) is scattered into the materialised rows
// T[n, U, y, b] = F[n, U, y + b] for b < NB, 0 <= y < Q (every row slot written once).
template <int FX, int FY, int CC, bool ROWS>
__global__ void __launch_bounds__(256) conv_fold_fixed(const std::int8_t* __restrict__ a, uint4* __restrict__ F, int pixels,
                                                       int FU, int FV, long long a_n, long long a_x, long long a_y,
                                                       long long a0, int u_lo, int u_hi, int v_lo, int v_hi, int Q, int NB) {
  constexpr int FC = (FX * FY * CC + 15) / 16 * 16;
  for (int pix = blockIdx.x * blockDim.x + threadIdx.x; pix < pixels; pix += gridDim.x * blockDim.x) {
    const int nu = pix / FV, V = pix - nu * FV;
    const int n = nu / FU, U = nu - n * FU;
    std::uint32_t w[FC / 4];
#pragma unroll
    for (int i = 0; i < FC / 4; i++) w[i] = 0;
#pragma unroll
    for (int di = 0; di < FX; di++) {
      const int u = FX * U + di;
      const bool uok = u >= u_lo && u <= u_hi;
      const std::int8_t* rp = a + a0 + a_n * n + a_x * u;
#pragma unroll
      for (int dj = 0; dj < FY; dj++) {
        const int v = FY * V + dj;
        if (uok && v >= v_lo && v <= v_hi) {
#pragma unroll
          for (int c = 0; c < CC; c++) {
            const int q = (di * FY + dj) * CC + c;
            w[q / 4] |= static_cast<std::uint32_t>(static_cast<std::uint8_t>(__ldg(rp + a_y * v + c))) << (8 * (q % 4));
          }
        }
      }
    }
    if (ROWS) {
      const uint4 val = make_uint4(w[0], w[1], w[2], w[3]);
      for (int b = 0; b < NB; b++) {
        const int y = V - b;
        if (y >= 0 && y < Q) F[(static_cast<long long>(nu) * Q + y) * NB + b] = val;
      }
    } else {
#pragma unroll
      for (int i = 0; i < FC / 16; i++)
        F[static_cast<long long>(pix) * (FC / 16) + i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
    }
  }
}

// Rows layout, one block per folded row (n, U): the row's FV folded pixels are built in shared
// memory (one thread each), then the Q x NB 16-byte row slots are written contiguously
// (coalesced 16-byte stores; the scatter form above writes them 64 bytes apart).
template <int FX, int FY, int CC>
__global__ void __launch_bounds__(256) conv_fold_rows_block(const std::int8_t* __restrict__ a, uint4* __restrict__ T,
                                                            int rows, int FU, int FV, long long a_n, long long a_x,
                                                            long long a_y, long long a0, int u_lo, int u_hi, int v_lo,
                                                            int v_hi, int Q, int NB) {
  extern __shared__ uint4 fp[];  // [FV]
  for (int nu = blockIdx.x; nu < rows; nu += gridDim.x) {
    const int n = nu / FU, U = nu - n * FU;
    for (int V = threadIdx.x; V < FV; V += blockDim.x) {
      std::uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int di = 0; di < FX; di++) {
        const int u = FX * U + di;
        const bool uok = u >= u_lo && u <= u_hi;
        const std::int8_t* rp = a + a0 + a_n * n + a_x * u;
#pragma unroll
        for (int dj = 0; dj < FY; dj++) {
          const int v = FY * V + dj;
          if (uok && v >= v_lo && v <= v_hi) {
#pragma unroll
            for (int c = 0; c < CC; c++) {
              const int q = (di * FY + dj) * CC + c;
              w[q / 4] |= static_cast<std::uint32_t>(static_cast<std::uint8_t>(__ldg(rp + a_y * v + c))) << (8 * (q % 4));
            }
          }
        }
      }
      fp[V] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncthreads();
    uint4* dst = T + static_cast<long long>(nu) * Q * NB;
    for (int i = threadIdx.x; i < Q * NB; i += blockDim.x) {
      const int y = i / NB, b = i - y * NB;
      dst[i] = fp[y + b];
    }
    __syncthreads();
  }
}

// Rows layout for any fold with 16-byte folded pixels (fx*fy*C <= 16): one thread per pixel.
__global__ void __launch_bounds__(256) conv_fold_rows_any(const std::int8_t* __restrict__ a, uint4* __restrict__ T,
                                                          int pixels, int FU, int FV, int fx, int fy, int C,
                                                          long long a_n, long long a_x, long long a_y, long long a0,
                                                          int u_lo, int u_hi, int v_lo, int v_hi, int Q, int NB) {
  for (int pix = blockIdx.x * blockDim.x + threadIdx.x; pix < pixels; pix += gridDim.x * blockDim.x) {
    const int nu = pix / FV, V = pix - nu * FV;
    const int n = nu / FU, U = nu - n * FU;
    std::uint32_t w[4] = {0, 0, 0, 0};
    int q = 0;
    for (int di = 0; di < fx; di++)
      for (int dj = 0; dj < fy; dj++)
        for (int c = 0; c < C; c++, q++) {
          const int u = fx * U + di, v = fy * V + dj;
          if (u >= u_lo && u <= u_hi && v >= v_lo && v <= v_hi)
            w[q >> 2] |= static_cast<std::uint32_t>(static_cast<std::uint8_t>(__ldg(a + a0 + a_n * n + a_x * u + a_y * v + c)))
                         << (8 * (q & 3));
        }
    const uint4 val = make_uint4(w[0], w[1], w[2], w[3]);
    for (int b = 0; b < NB; b++) {
      const int y = V - b;
      if (y >= 0 && y < Q) T[(static_cast<long long>(nu) * Q + y) * NB + b] = val;
    }
  }
}

// Any fold: one thread per 4 bytes of a folded pixel, per-byte (di, dj, c) from a shared table.
__global__ void __launch_bounds__(256) conv_fold_any(const std::int8_t* __restrict__ a, std::uint32_t* __restrict__ F,
                                                     long long words, int FU, int FV, int FCW, int fx, int fy, int C,
                                                     long long a_n, long long a_x, long long a_y, long long a0, int u_lo,
                                                     int u_hi, int v_lo, int v_hi) {
  __shared__ int tab[1024];  // di | c << 8 | dj << 16, or -1
  const int fc = 4 * FCW, fyc = fy * C;
  for (int q = threadIdx.x; q < fc; q += blockDim.x) {
    int e = -1;
    if (q < fx * fyc) {
      const int di = q / fyc, r = q - di * fyc, dj = r / C, c = r - dj * C;
      e = di | (c << 8) | (dj << 16);
    }
    tab[q] = e;
  }
  __syncthreads();
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < words;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long pix = g / FCW;
    const int wi = static_cast<int>(g - pix * FCW);
    const long long nu = pix / FV;
    const int V = static_cast<int>(pix - nu * FV);
    const long long n = nu / FU;
    const int U = static_cast<int>(nu - n * FU);
    std::uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int t = tab[4 * wi + e];
      if (t >= 0) {
        const int u = fx * U + (t & 0xFF), v = fy * V + (t >> 16), c = (t >> 8) & 0xFF;
        if (u >= u_lo && u <= u_hi && v >= v_lo && v <= v_hi)
          word |= static_cast<std::uint32_t>(static_cast<std::uint8_t>(__ldg(a + a0 + a_n * n + a_x * u + a_y * v + c)))
                  << (8 * e);
      }
    }
    F[g] = word;
  }
}

// Folded filter: G[a, k, q], q = b*fold_c + kf -> F[fx*a + di, fy*b + dj, k, c] (zero when the
// tap is past R/S or kf is padding).  Banded (band > 1, ConvPlan::fold_band): rows r of
// [fr + band - 1][band * K][cv], block (r, p) = G[r - p] (zero outside 0 <= r - p < fr).
__global__ void conv_fold_filter_kernel(const std::int8_t* __restrict__ b, std::int8_t* __restrict__ pb, int K, int C,
                                        int R, int S, int fx, int fy, int fc, int cv, int fr, int band, long long b_i,
                                        long long b_j, long long b_k, long long b_c, long long b0) {
  const int rows = band * K, total = (fr + band - 1) * rows * cv, fyc = fy * C;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int q = g % cv, rk = g / cv, row = rk % rows, r = rk / rows;
    const int pband = row / K, k = row - pband * K, ta = r - pband;
    const int tb = q / fc, kf = q - tb * fc;
    std::int8_t val = 0;
    if (ta >= 0 && ta < fr && kf < fx * fyc) {
      const int di = kf / fyc, r = kf - di * fyc, dj = r / C, c = r - dj * C;
      const int i = fx * ta + di, j = fy * tb + dj;
      if (i < R && j < S) val = b[b0 + b_i * i + b_j * j + b_k * k + b_c * c];
    }
    pb[g] = val;
  }
}

}  // namespace

cudaError_t launch_conv_fold(const ConvPlan& cp, const void* a, void* f, cudaStream_t s) {
  const long long pixels = cp.N * cp.fold_u * cp.fold_v;
  const auto* in = static_cast<const std::int8_t*>(a);
  const int lo_u = static_cast<int>(cp.u_lo), hi_u = static_cast<int>(cp.u_hi);
  const int lo_v = static_cast<int>(cp.v_lo), hi_v = static_cast<int>(cp.v_hi);
  // one thread per folded pixel, no grid-stride cap: the stem fold (12.8 M pixels at b1024)
  // streams better with every block in flight (stem step 437.9 -> 431.9 us against 32 blocks
  // per SM); SB_FOLD_GRID=<blocks per SM> caps it
  const long long fold_cap = 148ll * (std::getenv("SB_FOLD_GRID") ? std::atoi(std::getenv("SB_FOLD_GRID")) : 4096);
  const int blocks = static_cast<int>(std::min<long long>((pixels + 255) / 256, fold_cap));
  const int Q = static_cast<int>(cp.W), NB = static_cast<int>(cp.fold_cv / 16);
  auto fixed = [&](auto kern) {
    kern<<<blocks, 256, 0, s>>>(in, static_cast<uint4*>(f), static_cast<int>(pixels), static_cast<int>(cp.fold_u),
                                static_cast<int>(cp.fold_v), cp.a_n, cp.a_x, cp.a_y, cp.a0, lo_u, hi_u, lo_v, hi_v, Q, NB);
  };
  const bool stem = cp.fold_x == 2 && cp.fold_y == 2 && cp.C == 3 && cp.fold_c == 16;
  const bool c3s1 = cp.fold_x == 1 && cp.fold_y == 1 && cp.C == 3 && cp.fold_c == 16;
  if (stem && cp.fold_rows) {
    const int rows = static_cast<int>(cp.N * cp.fold_u);
    conv_fold_rows_block<2, 2, 3><<<std::min(rows, 148 * 16), 128, static_cast<int>(cp.fold_v) * 16, s>>>(
        in, static_cast<uint4*>(f), rows, static_cast<int>(cp.fold_u), static_cast<int>(cp.fold_v), cp.a_n, cp.a_x,
        cp.a_y, cp.a0, lo_u, hi_u, lo_v, hi_v, Q, NB);
  } else if (stem) {
    fixed(conv_fold_fixed<2, 2, 3, false>);
  } else if (c3s1 && cp.fold_rows) {
    fixed(conv_fold_fixed<1, 1, 3, true>);
  } else if (c3s1) {
    fixed(conv_fold_fixed<1, 1, 3, false>);
  } else if (cp.fold_rows) {
    conv_fold_rows_any<<<blocks, 256, 0, s>>>(in, static_cast<uint4*>(f), static_cast<int>(pixels),
                                              static_cast<int>(cp.fold_u), static_cast<int>(cp.fold_v),
                                              static_cast<int>(cp.fold_x), static_cast<int>(cp.fold_y),
                                              static_cast<int>(cp.C), cp.a_n, cp.a_x, cp.a_y, cp.a0, lo_u, hi_u, lo_v,
                                              hi_v, Q, NB);
  } else {
    const int FCW = static_cast<int>(cp.fold_c / 4);
    const long long words = pixels * FCW;
    const long long wblocks = std::min<long long>((words + 255) / 256, 148 * 32);
    conv_fold_any<<<static_cast<int>(wblocks), 256, 0, s>>>(
        in, static_cast<std::uint32_t*>(f), words, static_cast<int>(cp.fold_u), static_cast<int>(cp.fold_v), FCW,
        static_cast<int>(cp.fold_x), static_cast<int>(cp.fold_y), static_cast<int>(cp.C), cp.a_n, cp.a_x, cp.a_y, cp.a0,
        lo_u, hi_u, lo_v, hi_v);
  }
  return cudaGetLastError();
}

cudaError_t launch_conv_pack_filter(const ConvPlan& cp, const void* b, void* pb, cudaStream_t s) {
  if (cp.fold_x) {
    const int band = cp.fold_band ? static_cast<int>(cp.fold_band) : 1;
    const int total = static_cast<int>((cp.fold_r + band - 1) * band * cp.K * cp.fold_cv);
    conv_fold_filter_kernel<<<std::min(1024, (total + 255) / 256), 256, 0, s>>>(
        static_cast<const std::int8_t*>(b), static_cast<std::int8_t*>(pb), static_cast<int>(cp.K),
        static_cast<int>(cp.C), static_cast<int>(cp.R), static_cast<int>(cp.S), static_cast<int>(cp.fold_x),
        static_cast<int>(cp.fold_y), static_cast<int>(cp.fold_c), static_cast<int>(cp.fold_cv),
        static_cast<int>(cp.fold_r), band, cp.b_i, cp.b_j, cp.b_k, cp.b_c, cp.b0);
    return cudaGetLastError();
  }
  const int kp = static_cast<int>(cp.pack_k), rsc = static_cast<int>(cp.R * cp.S * cp.C);
  const int fb = static_cast<int>(std::min<long long>((cp.K * kp + 255) / 256, 1024));
  (void)rsc;
  conv_pack_filter_kernel<<<fb, 256, 0, s>>>(static_cast<const std::int8_t*>(b), static_cast<std::int8_t*>(pb),
                                             static_cast<int>(cp.K), static_cast<int>(cp.C), static_cast<int>(cp.R),
                                             static_cast<int>(cp.S), static_cast<int>(cp.pack_run), kp, cp.b_i, cp.b_j,
                                             cp.b_k, cp.b_c, cp.b0);
  return cudaGetLastError();
}

const char* conv_igemm_unsupported(const ConvPlan& cp) {
  if (cp.packed && cp.fold_x) {
    if (cp.fold_x != cp.sx || cp.fold_y != cp.sy || cp.fold_c % 16 || cp.fold_cv % 64 ||
        cp.fold_x * cp.fold_y * cp.C > cp.fold_c || cp.fold_s * cp.fold_c > cp.fold_cv ||
        cp.fold_u < cp.H + cp.fold_r - 1 || (cp.fold_v - cp.W + 1) * cp.fold_c < cp.fold_cv)
      return "inconsistent phase fold";
    if (cp.N * cp.fold_u * cp.fold_v >= (1ll << 31) || cp.fold_c > 1024 || cp.fold_r > 127 || cp.C > 255)
      return "folded input too large";
    return conv_igemm_unsupported(packed_view(cp));
  }
  if (cp.packed) {
    // gather mode: the kernel builds A rows from the original input; the GEMM is packed_view
    if (cp.pack_run && (cp.a_y != cp.C || cp.S * cp.C > cp.pack_run || (cp.pack_run != 16 && cp.pack_run != 32 &&
                                                                          cp.pack_run != 64)))
      return "run layout needs contiguous pixels";
    if (cp.R > 127 || cp.S > 127 || cp.pack_k > 1024 || cp.pack_k % 64 ||
        cp.a_x * (cp.R - 1) + cp.a_y * (cp.S - 1) + cp.C >= (1ll << 30))
      return "gathered taps out of range";
    return conv_igemm_unsupported(packed_view(cp));
  }
  if (cp.fold_band) {
    // band view (see prepare()): one 128-pixel tile per output row, stacked rows along N
    if (cp.W > BM || cp.H % cp.fold_band || cp.fold_band != 2 || (cp.K != 128 && cp.K != 256) || cp.C != 64 ||
        cp.a_y != 16 || cp.a_x % 16 ||
        cp.R * cp.S * 64 * cp.K > 96 * 1024)
      return "band geometry";
    if (cp.c_dtype != DType::I8 || !cp.fresh_output || cp.epi_res || cp.c_y != cp.K / cp.fold_band ||
        cp.c_x != cp.W * cp.c_y || cp.c_x % 16 || cp.c0 % 16)
      return "band output not a fresh dense NHWC i8 activation";
    if (cp.N * (cp.H / cp.fold_band) >= (1ll << 31) || cp.a_n >= (1ll << 40)) return "extent too large";
    if (cp.epi_vec && cp.K > kMaxVecK) return "epilogue vector longer than 2048";
    return nullptr;
  }
  Geometry g;
  if (!geometry(cp, &g)) return "padding halo outside the im2col corner range";
  if (cp.C % 64 != 0) return "channels not a multiple of 64";
  if (cp.sx < 1 || cp.sx > 8 || cp.sy < 1 || cp.sy > 8) return "stride outside [1, 8]";
  if (cp.R > 16 || cp.S > 16) return "filter taps beyond 16";
  if (cp.a_y % 16 || cp.a_x % 16 || cp.a_n % 16) return "input strides not 16-byte multiples";
  if (cp.b_c != 1 || cp.b_k % 16 || (cp.S > 1 && cp.b_j % 16) || (cp.R > 1 && cp.b_i % 16) || cp.b0 % 16)
    return "filter layout not channel-contiguous with 16-byte aligned rows";
  if (cp.N * cp.H * cp.W >= (1ll << 31) || cp.K >= (1 << 20)) return "extent too large";
  // output rows must follow the (n, x, y) pixel order with a uniform pitch
  if (cp.c_y < cp.K || (cp.H > 1 && cp.c_x != cp.W * cp.c_y) || (cp.N > 1 && cp.c_n != cp.H * cp.W * cp.c_y))
    return "output not pixel-major";
  if (cp.R * cp.S * cp.C * 128 * 128 >= (1ll << 31)) return "reduction too long for exact s32 accumulation";
  if (cp.epi_vec && cp.K > kMaxVecK) return "epilogue vector longer than 2048";
  if (cp.epi_res && (cp.res_pix % 16 || cp.res_c0 % 16)) return "residual rows not 16-byte aligned";

  return nullptr;
}

cudaError_t launch_conv_igemm(const ConvPlan& cp, const ConvArgs& args, cudaStream_t s, int num_sms) {
  Prepared prep;  // copied under the lock: another thread's push_back may move the cache
  {
    Prepared* pr = nullptr;
    std::lock_guard<std::mutex> lock(g_mu);
    if (!g_prep) g_prep = new std::vector<Prepared>();
    for (auto& e : *g_prep)
      if (e.a == args.a && e.b == args.b && e.c == args.c && e.vec == args.vec && e.res == args.res && same(e.cp, cp))
        pr = &e;
    if (!pr) {
      if (g_prep->size() >= 512) g_prep->clear();
      Prepared fresh;
      cudaError_t err = prepare(cp, args, &fresh);
      if (err != cudaSuccess) return err;
      g_prep->push_back(fresh);
      pr = &g_prep->back();
    }
    prep = *pr;
  }
  IgKParams kp = prep.kp;
  kp.pdl = args.pdl_mode != kPdlOff ? 1 : 0;
  kp.pdl_wait = args.pdl_mode == kPdlWait ? 1 : 0;
  kp.b_early = args.b_immutable ? 1 : 0;
  if (kp.fast8 && std::getenv("SB_IG_NOPIPE")) kp.epi_pipe = 0;  // A/B switch, read per launch
  const int tiles = kp.tiles_m * kp.tiles_n;
  cudaLaunchConfig_t cfg = {};
  int grid = tiles < num_sms ? tiles : num_sms;
  if (kp.nstat) grid = grid / kp.tiles_n * kp.tiles_n;  // CTA c keeps n-tile c % tiles_n
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(64 + 32 * kp.epi_warps + (kp.gather ? 256 : 96 + (kp.res_mma || kp.band_raw ? 32 : 0)));
  cfg.dynamicSmemBytes = static_cast<unsigned>(kp.smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kp.pdl ? 1 : 0;
#ifdef SB_TILE_TRACE
  static long long* tr = nullptr;
  if (!tr) cudaMalloc(&tr, (640 + 32 * 4 * 3 + 256 + 512) * 8);
  cudaMemsetAsync(tr, 0, (640 + 32 * 4 * 3 + 256 + 512) * 8, s);
  kp.trace = tr;
  kp.exp = std::getenv("SB_IG_EXP") ? std::atoi(std::getenv("SB_IG_EXP")) : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, conv_igemm_i8_kernel, prep.amap, prep.bmap, prep.cmap, prep.rmap, kp);
  long long h[640 + 32 * 4 * 3 + 256 + 512];
  cudaStreamSynchronize(s);
  cudaMemcpy(h, tr, sizeof(h), cudaMemcpyDeviceToHost);
  std::fprintf(stderr, "igemm M=%d N=%d kblocks=%d kpb=%d stages=%d b_res=%d nstat=%d res1=%d split=%d tiles=%d\n", kp.M, kp.N, kp.kblocks,
               kp.kpb, kp.stages, kp.b_res, kp.nstat, kp.res1, kp.epi_split, tiles);
  if (kp.band && (kp.exp & 16)) {
    const unsigned char* b = reinterpret_cast<const unsigned char*>(h + 1280);
    std::fprintf(stderr, "band stage smem 0x%llx stage %lld rowb %lld bytes %d\n", h[1536], h[1537], kp.band_rowb, kp.band_bytes);
    for (int r = 0; r < 128; r++) {
      std::fprintf(stderr, "  %5d:", r * 16);
      for (int q = 0; q < 16; q++) std::fprintf(stderr, " %3d", static_cast<signed char>(b[r * 16 + q]));
      std::fprintf(stderr, "\n");
    }
  }
  for (int i = 0; i < 128; i++)
    if (h[128 + i])
      std::fprintf(stderr, "tile %3d prod %8lld mma0 %8lld mma1 %8lld | etop %8lld epi0 %8lld math %8lld epi1 %8lld\n", i,
                   h[i] ? h[i] - h[128] : -1, h[128 + i] - h[128], h[256 + i] - h[128], h[1024 + i] - h[128],
                   h[384 + i] - h[128], h[1152 + i] - h[128], h[512 + i] - h[128]);
  for (int i = 0; i < 32; i++)
    for (int st = 0; st < 4; st++) {
      const long long* q = h + 640 + (i * 4 + st) * 3;
      if (q[0]) std::fprintf(stderr, "  tile %2d stage %d: wait %6lld..%6lld  mma issue %5lld\n", i, st, q[0] - h[128], q[1] - h[128], q[2] - q[1]);
    }
  return e;
#else
  return cudaLaunchKernelEx(&cfg, conv_igemm_i8_kernel, prep.amap, prep.bmap, prep.cmap, prep.rmap, kp);
#endif
}

}  // namespace sb
