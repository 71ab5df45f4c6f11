// Host-callable launchers of the sm_100a kernels (kernels/*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "desc.hpp"
#include "plan.hpp"

namespace sb {

// fp32 numeric mode (kernels/generic_f32.cu)
cudaError_t launch_generic_f32(const GenericDesc* d_desc, std::int64_t pcount, const BufTable& t, DevError* err,
                               int launch_id, cudaStream_t s);
cudaError_t launch_generic(const GenericDesc* d_desc, std::int64_t pcount, const BufTable& t,
                           DevError* err, int launch_id, cudaStream_t s);
cudaError_t launch_fill(void* p, int kind, std::int64_t n, std::int64_t v, cudaStream_t s);
// Vectorised owner-mode block kernel (kernels/map.cu): memory-bound map / reduce blocks.
cudaError_t launch_map(const GenericDesc* d_desc, std::int64_t vcount, const BufTable& t, DevError* err,
                       int launch_id, cudaStream_t s);

// Streaming reduce/copy (kernels/reduce.cu).
struct ReduceArgs {
  const void* in;
  void* out;
  int in_kind, out_kind, agg, fresh;
  std::int64_t identity;
  int np, nr, rcount;
  std::int64_t prange[kMaxDims], pin[kMaxDims], pout[kMaxDims];
  std::int64_t rrange[kMaxDims], rstep[kMaxDims];
  std::int64_t in_c, out_c, pcount;
};
int reduce_vec_lanes(int in_kind);
cudaError_t launch_reduce(const ReduceArgs& a, cudaStream_t s);

// tcgen05 GEMM (kernels/gemm_tc.cu).
// Programmatic dependent launch per call (capi.cpp decides from buffer overlap with the
// launches that may still run): 0 plain stream order, 1 PDL + griddepcontrol.wait,
// 2 PDL without waiting (independent of every in-flight launch), 3 PDL whose loads may start
// at once (nothing in flight writes what it reads) but whose stores wait (resident-filter conv
// only; other kernels treat it as 1).
enum : int { kPdlOff = 0, kPdlWait = 1, kPdlFree = 2, kPdlLoadEarly = 3 };

struct GemmArgs {
  const void* a;
  const void* b;
  void* c;
  int pdl_mode = kPdlWait;
};
const char* gemm_tc_unsupported(const GemmPlan& g);
// fp32 mode: exact-order SIMT GEMM, bitwise equal to the F32 oracle (kernels/gemm_f32.cu)
cudaError_t launch_gemm_f32(const GemmPlan& g, const void* a, const void* b, void* c, cudaStream_t s);
// byte-limb mode: split A/B into concatenated unsigned byte planes, and the final combine
cudaError_t launch_limb_split(const GemmPlan& g, const void* a, const void* b, void* pa, void* pb, cudaStream_t s);
cudaError_t launch_limb_combine(const GemmPlan& g, const void* sums, void* c, cudaStream_t s);
// Fused byte-limb GEMM: planes (launch-internal split) + one kernel with the combine in its
// epilogue; pa / pb hold limbs_a * M * limb_fused_kp(g) / limbs_b * N * limb_fused_kp(g) bytes.
cudaError_t launch_limb_fused(const GemmPlan& g, const void* a, const void* b, void* pa, void* pb, void* c,
                              cudaStream_t s, int num_sms);
long long limb_fused_kp(const GemmPlan& g);
// The u8 GEMM computing S_s inside a limb plan.
GemmPlan limb_sum_plan(const GemmPlan& g, int s);
long long limb_plane_bytes_a(const GemmPlan& g);
// 3xTF32 mode for fp32 matmuls (opt-in, stated bound): split + one kind::tf32 GEMM
GemmPlan tf32_sum_plan(const GemmPlan& g, int t);
cudaError_t launch_tf32_combine(const GemmPlan& g, const void* sums, void* c, cudaStream_t s);
cudaError_t launch_tf32_split(const GemmPlan& g, const void* a, const void* b, void* pa, void* pb, cudaStream_t s);
long long limb_a_off(const GemmPlan& g, int s);
long long limb_b_off(const GemmPlan& g, int s);
long long limb_plane_bytes_b(const GemmPlan& g);
cudaError_t launch_gemm_tc(const GemmPlan& g, const GemmArgs& args, cudaStream_t s, int num_sms);

// Constraint-satisfying points of one block (kernels/count.cu); cons_k is [nc][nd].
cudaError_t launch_count_points(int nd, const long long* ranges, int nc, const long long* cons_c,
                                const long long* cons_k, void* scratch, unsigned long long* h_out, cudaStream_t s);
std::size_t count_points_scratch_bytes();

// Distinct cache lines per tile for every residue of the tile base (kernels/tilecost.cu): one
// (candidate, refinement) item of tile_cost (tile.cpp:413-453).  F = cst + one value from each
// axis list (len[a] values at val_off, axis 0 fastest); run != 0: the last axis is the unit-step
// run [v, v + len - 1] given by its single stored value v.  Per-q min/max slots live in shared
// memory (scratch_off < 0) or at scratch_off words of the global scratch (2 * nq words).
constexpr int kTileMaxAxes = 32;
struct TileLineItem {
  long long cst, qbase, prefixes, scratch_off;
  int nq, naxes, run, val_off;
  int len[kTileMaxAxes];
};
// Split-aggregation combine over NCCL (kernels/collective.cu; NCCL loaded at first use).
void nccl_unique_id(char (&id)[128]);
void* nccl_comm_init(int nranks, const char* id, int rank);
void nccl_comm_destroy(void* comm);
void split_allreduce(void* comm, void* data, long long count, DType dt, Agg agg, cudaStream_t s);
int tile_lines_smem_q();
cudaError_t launch_tile_lines(const std::vector<TileLineItem>& items, const std::vector<long long>& values,
                              long long scratch_words, int L, std::vector<long long>* counts, cudaStream_t s);

// Windowed max/min over constraint-bounded taps, 16-byte channel vectors (kernels/pool.cu).
const char* pool_unsupported(const PoolPlan& pp);
cudaError_t launch_pool(const PoolPlan& pp, const void* in, void* out, cudaStream_t s);

// tcgen05 implicit-GEMM convolution, i8 x i8 -> i32 accumulate (kernels/conv_tc.cu).
struct ConvArgs {
  const void* a;  // input activations (i8)
  const void* b;  // filter (i8)
  void* c;        // output (i8/i16/i32)
  std::int64_t a_elems, b_elems, c_elems;
  bool b_immutable = false;  // filter is a root `in` buffer no plan step writes
  const void* vec = nullptr;  // fused-epilogue per-channel vector buffer
  int vec_kind = 0;
  const void* res = nullptr;  // fused-epilogue residual (i8, pixel-major)
  int pdl_mode = kPdlWait;
};
// Host-side checks that the plan fits the kernel's tiling; empty string = ok.
const char* conv_tc_unsupported(const ConvPlan& cp);
cudaError_t launch_conv_tc(const ConvPlan& cp, const ConvArgs& args, cudaStream_t s, int num_sms);
// General im2col-TMA implicit GEMM (kernels/conv_igemm.cu): strides, 1x1, streamed filters.
const char* conv_igemm_unsupported(const ConvPlan& cp);
cudaError_t launch_conv_igemm(const ConvPlan& cp, const ConvArgs& args, cudaStream_t s, int num_sms);
// Packs a small-channel conv's filter for gather mode ([K, pack_k] rows) or the phase fold
// ([fold_r][K][fold_cv]) (ConvPlan::packed).
cudaError_t launch_conv_pack_filter(const ConvPlan& cp, const void* b, void* pb, cudaStream_t s);
// Phase-folds the input of a folded small-channel conv (ConvPlan::fold_x) into f.
cudaError_t launch_conv_fold(const ConvPlan& cp, const void* a, void* f, cudaStream_t s);

}  // namespace sb
