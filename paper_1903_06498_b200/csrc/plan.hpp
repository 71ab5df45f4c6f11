// Host-side execution plan: the lowering of a Stripe Program into a serial
// list of device steps (identity fills and kernel launches).
//
// This is the B200 replacement for the reference's Executor::compile
// (proj/src/interp.cpp:201-347): instead of a slot-form tree walked per point
// on one CPU thread, each root-to-leaf chain of blocks becomes ONE flat launch
// whose dims are every ranged index on the chain, whose constraints are all the
// chain's predicates, and whose accesses are the composed refinement chains
// (flat base = sum over levels of stride*offset, interp.cpp:227-233, 449-451).
// Multi-statement blocks become consecutive launches (kernel boundaries are
// the phase barriers); per-iteration local allocations become per-point
// slices of a zero-filled scratch buffer (interp.cpp:239-247, 442-447).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "desc.hpp"
#include "ir.hpp"

namespace sb {

struct FAff {
  std::int64_t c = 0;
  std::vector<std::int64_t> k;  // dense over the launch dims
  std::int64_t at(std::size_t d) const { return d < k.size() ? k[d] : 0; }
  bool uses(std::size_t d) const { return at(d) != 0; }
  bool operator==(const FAff& o) const;
};

struct PDim {
  std::string name;
  std::int64_t range = 1;
  bool pinned = false;  // host-unrolled (serial fallback); value folded into constants
  std::int64_t value = 0;
};

struct PBuffer {
  std::string name;
  DType dtype = DType::I32;
  std::int8_t kind = kI32;  // device storage kind (kI64 for temp spills)
  std::int64_t elements = 0;
  bool root = false;
  int root_index = -1;  // index into Program::buffers
  Dir dir = Dir::In;
};

struct PAccess {
  int buf = 0;
  FAff addr;
};

struct PSpecial {
  bool gather = true;
  int dst = 0, src = 0, idx = 0;  // access indices
  std::vector<std::int64_t> walk, sdst, ssrc, sidx;
  std::int64_t bound = 0;
  Agg dst_agg = Agg::Assign;
  DType dst_dtype = DType::I32;
};

// Specialised kernel families the matcher can route a launch to.
enum class KernelKind { Generic, ConvI8TC, Map, Reduce, GemmI8TC, ConvIgemmTC, Pool, GemmF32 };

// Windowed max/min (pooling) leaf: $v = load(I); O = store($v) with O:max|min, taps
// bounded by interval constraints (kernels/pool.cu).
struct PoolPlan {
  int in_buf = -1, out_buf = -1;
  int kind = 0;  // element kind (in == out)
  int agg = 0;
  std::int64_t N = 1, H = 1, W = 1, C = 1, R = 1, S = 1, sx = 1, sy = 1;
  std::int64_t a_n = 0, a_x = 0, a_y = 0, a0 = 0;  // input: a0 + a_n*n + a_x*u + a_y*v + c, u = sx*x + i
  std::int64_t u_lo = 0, u_hi = 0, v_lo = 0, v_hi = 0;
  std::int64_t o_n = 0, o_x = 0, o_y = 0, o0 = 0;  // output: o0 + o_n*n + o_x*x + o_y*y + c
  // the output's only earlier touch is a fill (elided): start every element from fill_value
  // instead of reading it back
  bool fresh = false;
  std::int64_t fill_value = 0;
};

// tcgen05 GEMM (kernels/gemm_tc.cu): C[m,n] (+)= sum_k A[m,k] B[k,n], i8 operands.
struct GemmPlan {
  long long M = 0, N = 0, K = 0, lda = 0, ldb = 0, ldc = 0, a0 = 0, b0 = 0, c0 = 0;  // keep first, contiguous
  bool b_kmajor = false, fresh = false;
  DType c_dtype = DType::I32;
  int a_buf = -1, b_buf = -1, c_buf = -1;
  bool unsigned_ab = false;  // u8 x u8 operands (byte limbs)
  bool f32 = false;          // fp32 numeric mode (kernels/gemm_f32.cu)
  bool tf32x3 = false;       // fp32 via 3xTF32 on tensor cores (PlanOptions::fp32_tc)
  // byte-limb mode (i16/i32 operands, exact modulo 2^(8*bytes(C))): A = sum_i a_i 256^i with
  // unsigned byte planes; S_s = sum_{i+j=s} a_i b_j runs as ONE u8 GEMM per s over operands
  // concatenated along k (planes_a / planes_b), C (+)= sum_s S_s << 8s wrapped at the store
  int limbs_a = 0, limbs_b = 0, a_kind = 0, b_kind = 0;
  int planes_a = -1, planes_b = -1, sums = -1;  // scratch buffers
  // fused (default): planes [limb][rows][Kp] and ONE kernel keeping every S_s in TMEM and
  // combining them in its epilogue (gemm_tc.cu gemm_limb_kernel); else the per-sum GEMMs
  bool limb_fused = false;
};

// Number of (i, j) limb pairs with i + j = s.
inline int limb_pairs(const GemmPlan& g, int s) {
  int n = 0;
  for (int i = 0; i < g.limbs_a; i++)
    if (s - i >= 0 && s - i < g.limbs_b) n++;
  return n;
}
// Output bytes that matter (sums s = 0 .. limb_smax).
inline int limb_smax(const GemmPlan& g) {
  const int ob = g.c_dtype == DType::I8 ? 1 : g.c_dtype == DType::I16 ? 2 : 4;
  return std::min(ob, g.limbs_a + g.limbs_b - 1) - 1;
}

// Streaming reduce/copy ($v = load(I); O = store($v)): kernels/reduce.cu.
struct ReducePlan {
  int in_buf = -1, out_buf = -1;
  int in_kind = 0, out_kind = 0, agg = 0;
  bool fresh = false;
  std::int64_t identity = 0;
  int np = 0, nr = 0;
  std::int64_t prange[kMaxDims] = {}, pin[kMaxDims] = {}, pout[kMaxDims] = {};
  std::int64_t rrange[kMaxDims] = {}, rstep[kMaxDims] = {};
  std::int64_t in_c = 0, out_c = 0, pcount = 0;
  int rcount = 0;
};

// Parameters of the tcgen05 implicit-GEMM convolution (kernels/conv_tc.cu).
struct ConvPlan {
  int a_buf = -1, b_buf = -1, c_buf = -1;
  DType c_dtype = DType::I32;
  std::int64_t N = 1, H = 1, W = 1, C = 1, K = 1, R = 1, S = 1;
  std::int64_t sx = 1, sy = 1;  // conv strides (input rows/cols per output row/col)
  // A (input) element address = a_n*n + a_x*u + a_y*v + c + a0, u = sx*x + i + ox, v = sy*y + j + oy
  std::int64_t a_n = 0, a_x = 0, a_y = 0, a0 = 0;
  std::int64_t ox = 0, oy = 0;
  std::int64_t u_lo = 0, u_hi = 0, v_lo = 0, v_hi = 0;  // valid input window from constraints
  // B (filter) element address = b_i*i + b_j*j + b_k*k + b_c*c + b0
  std::int64_t b_i = 0, b_j = 0, b_k = 0, b_c = 0, b0 = 0;
  // C (output) element address = c_n*n + c_x*x + c_y*y + k + c0
  std::int64_t c_n = 0, c_x = 0, c_y = 0, c0 = 0;
  bool fresh_output = false;  // output known identity-filled: overwrite instead of accumulate
  bool overwrites = false;    // fused epilogue stores with assign (program semantics overwrite)
  bool b_immutable = false;   // filter is a root `in` buffer that no plan step writes
  // fused element-wise epilogue (K3e): out = wrap(max(acc + vec[k], lo)) with the optional parts
  bool epi = false, epi_vec = false, epi_lo = false;
  int vec_buf = -1;
  std::int64_t vec_c = 0, vec_k = 0, lo = 0;
  // + res[pixel, k] (i8, pixel-major like the output): residual add (im2col kernel only)
  bool epi_res = false;
  int res_buf = -1;
  std::int64_t res_c0 = 0, res_pix = 0;
  // small-channel lowering (the 7x7x3 stem): taps x channels packed per output pixel into
  // a scratch [pixels, pack_k] (zero where a constraint skips the tap), the filter into
  // [K, pack_k]; the im2col kernel then runs the 1x1 conv packed_view() describes
  bool packed = false;
  int pack_a = -1, pack_b = -1;
  std::int64_t pack_k = 0;
  std::int64_t pack_run = 0;  // >0: kk = i * pack_run + (j * C + c) (contiguous S*C-byte runs per tap row)
  // phase fold (fold_x/fold_y > 0, pack_a = the folded input): the strided small-channel conv
  // becomes a stride-1 valid conv over folded pixels F[n, U, V, (di, dj, c)] =
  // I[n, sx*U + di, sy*V + dj, c] (zero outside the constraint window; fold_c bytes each,
  // fold_u x fold_v of them per image): fold_r tap rows of one fold_cv-byte "pixel" each,
  // the fold_cv / fold_c folded pixels from (U, y) on (see packed_view())
  std::int64_t fold_x = 0, fold_y = 0, fold_c = 0, fold_r = 0, fold_s = 0, fold_cv = 0, fold_u = 0, fold_v = 0;
  // fold_rows: the folded input is materialised as rows T[n, U, y] = F[n, U, y .. y + fold_cv /
  // fold_c - 1] (fold_cv bytes, 64-byte aligned TMA rows; ~2x the im2col rate of the
  // overlapping-stride view) instead of the folded pixels themselves
  bool fold_rows = false;
  // fold_band (> 0, compact folded pixels): one tile = fold_band consecutive output rows x 128
  // pixel columns; A = the (fold_r + fold_band - 1) folded rows the band needs, one bulk copy,
  // read by UMMA descriptors whose rows overlap (row m at 16 m bytes, no swizzle); the band's
  // output rows stacked along N against a banded filter [fold_r + band - 1][band * K][fold_cv]
  // (block (r, p) = folded tap row r - p): N = band * K columns per MMA instead of K
  std::int64_t fold_band = 0;
  // band_raw (with fold_band, the 2x2-folded 3-channel stem): no folded copy -- the conv's
  // producer warps build each band's folded rows in shared memory from the raw input rows
  // (raw_* = the unfolded input's geometry: a_n, a_x, a0, window [u_lo, u_hi] x [v_lo, v_hi],
  // 3-byte pixels)
  bool band_raw = false;
  std::int64_t raw_a_n = 0, raw_a_x = 0, raw_a0 = 0, raw_u_lo = 0, raw_u_hi = 0, raw_v_lo = 0, raw_v_hi = 0;
};

// Statement-DAG concurrency (schedule.cpp): independent steps on up to N streams.
struct PStep;
struct Plan;
struct LaneSchedule {
  int nlanes = 1;
  std::vector<int> lane;                // per step
  std::vector<std::vector<int>> waits;  // per step: steps on other lanes to wait for
  std::vector<char> signal;             // per step: record an event after it
};

// The 1x1 conv over the packed operands of a `packed` conv (same output and epilogue); for a
// phase-folded conv, the fold_r x 1 stride-1 conv over the folded input whose pixel rows
// overlap (pixel stride fold_c bytes, fold_cv "channels" per pixel).
ConvPlan packed_view(const ConvPlan& c);

struct PLaunch {
  std::string path;  // dot path of the leaf block ("0.1.0")
  std::vector<PDim> dims;
  std::vector<FAff> cons;
  std::vector<PAccess> acc;
  std::vector<DInstr> code;
  std::vector<std::int64_t> consts;
  std::vector<PSpecial> specials;
  std::vector<std::pair<Agg, DType>> priv;  // leaf-level private allocs
  int ntemps = 0;
  bool has_spill = false;

  // analysis (analyze())
  std::int8_t mode = kModeOwner;
  bool is_float = false;  // f32 numeric mode (every data buffer F32)
  std::vector<int> pdims, rdims;
  std::vector<std::int8_t> acc_mode, acc_cell;
  int ncells = 0;
  std::int64_t pcount = 1, points = 1;
  std::string why;  // reason for a non-owner mode

  KernelKind kernel = KernelKind::Generic;
  ConvPlan conv;
  ReducePlan reduce;
  GemmPlan gemm;
  PoolPlan pool;
  int fused_fill_root = -1;  // root buffer whose prepare_outputs fill this launch performs itself
  // map kernel (vectorised owner mode): vdim = thread dim split into kVec-lane vectors
  int vdim = -1;
  std::vector<std::int8_t> vkind;
  std::int64_t vcount = 0;
};

struct PStep {
  enum Kind { Fill, Launch } kind = Launch;
  bool elided = false;  // absorbed into another step (fused epilogue / fused identity fill)
  int buf = -1;
  std::int64_t value = 0;
  PLaunch launch;
};

struct Plan {
  std::vector<PBuffer> bufs;  // roots first (Program::buffers order), then scratch
  std::vector<PStep> steps;
  std::vector<std::string> notes;
  std::string describe() const;  // human-readable plan dump (tests / logs)
};

struct PlanOptions {
  bool enable_tc = true;           // route matched contractions to tcgen05 kernels
  std::vector<bool> fresh_outputs; // per root buffer: contents are prepare_outputs' identity
  std::int64_t max_unroll = 1 << 16;
  bool fp32_tc = false;            // fp32 matmuls as 3xTF32 tensor-core GEMMs (stated bound)
};

Plan build_plan(const Program& p, const PlanOptions& opt);

// Fills a device descriptor for a generic launch.
// bufmap receives the plan buffer id of every launch-local buffer slot.
void to_desc(const PLaunch& l, GenericDesc* d, std::vector<int>* bufmap);

// Plan buffers a step reads / writes (aggregating stores count as both).
void step_access(const PStep& s, std::vector<int>* reads, std::vector<int>* writes);
// `alias(a, b)`: distinct plan buffers that share device memory (scratch arena reuse).
LaneSchedule schedule_lanes(const Plan& plan, int max_lanes, const std::function<bool(int, int)>& alias);

}  // namespace sb
