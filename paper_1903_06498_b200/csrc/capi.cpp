// C ABI + device executor (see include/stripe_b200.h).
//
// sb_execute is the B200 counterpart of stripe::execute (interp.h:68,
// interp.cpp:613-615): the buffer-table check of Executor::run
// (interp.cpp:183-198) happens on the host, the Program is lowered once into a
// cached plan (planner.cpp), buffers are moved to HBM at native width, the
// plan's steps run in stream order, and outputs come back.  Errors map 1:1 to
// the reference's ExecError codes.
#include <cuda_runtime.h>

#include <atomic>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/stripe_b200.h"
#include "ir.hpp"
#include "kernels.hpp"
#include "tilecost.hpp"
#include "plan.hpp"

namespace {

thread_local std::string g_last_error;

int status_of(const std::string& code) {
  static const std::map<std::string, int> m = {
      {"MissingBuffer", SB_ERR_MISSING_BUFFER},   {"UnknownIntrinsic", SB_ERR_UNKNOWN_INTRINSIC},
      {"UnknownSpecial", SB_ERR_UNKNOWN_SPECIAL}, {"UndefinedTemp", SB_ERR_UNDEFINED_TEMP},
      {"OutOfBoundsAccess", SB_ERR_OUT_OF_BOUNDS}, {"UnboundIndex", SB_ERR_UNBOUND_INDEX},
      {"SyntaxError", SB_ERR_SYNTAX},             {"ScopeError", SB_ERR_SCOPE},
      {"Unsupported", SB_ERR_UNSUPPORTED},        {"CudaError", SB_ERR_CUDA},
      {"NcclError", SB_ERR_NCCL},                 {"Invalid", SB_ERR_INVALID},
      {"InvalidTile", SB_ERR_PASS},               {"NotTileable", SB_ERR_PASS}};
  auto it = m.find(code);
  return it == m.end() ? SB_ERR_INVALID : it->second;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return SB_OK;
  } catch (const sb::Error& e) {
    g_last_error = e.code + ": " + e.what();
    return status_of(e.code);
  } catch (const std::exception& e) {
    g_last_error = std::string("Invalid: ") + e.what();
    return SB_ERR_INVALID;
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw sb::Error("CudaError", std::string(what) + ": " + cudaGetErrorString(e));
}

std::size_t kind_bytes(int kind) {
  switch (kind) {
    case sb::kI8: return 1;
    case sb::kI16: return 2;
    case sb::kI64: return 8;
    default: return 4;
  }
}

std::size_t padded(std::size_t bytes) { return (bytes + 15) / 16 * 16; }

struct Compiled {
  std::uint64_t id = 0;  // unique: device state is keyed by it, never by address
  sb::Plan plan;
  std::vector<sb::GenericDesc> descs;
  std::vector<std::vector<int>> bufmaps;
  std::vector<int> desc_of_step;
  sb::LaneSchedule lanes;
  std::vector<long long> arena_off, arena_bytes;  // scratch buffer -> arena range (-1: none)
  std::size_t arena_total = 0;
};

}  // namespace

struct sb_program {
  sb::Program prog;
  std::mutex mu;
  std::map<std::string, std::unique_ptr<Compiled>> plans;
  ~sb_program();
};

struct sb_context {
  // One execute at a time per context: the staging buffers, root buffers, plan states and
  // the PDL window below are mutated by every execute ("execute is reentrant",
  // concurrent callers on one context serialize here; callers wanting
  // concurrency use one context per thread, as stripe::b200::execute does).
  std::recursive_mutex mu;
  int device = 0;
  int num_sms = 148;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  sb::DevError* d_err = nullptr;
  sb::DevError* h_err = nullptr;
  std::uint64_t launches = 0;
  struct State {
    sb::GenericDesc* d_descs = nullptr;
    void* arena = nullptr;       // one allocation for every live scratch buffer
    std::size_t arena_bytes = 0;
    std::vector<void*> scratch;  // by plan buffer id (scratch only; null when never touched)
  };
  std::map<std::uint64_t, State> states;  // by Compiled::id
  cudaStream_t lane_streams[8] = {};       // statement-DAG lanes 1..7 (lane 0 = stream)
  std::vector<cudaEvent_t> step_events;    // per plan step (reused across runs)
  cudaEvent_t fork_event = nullptr, join_events[8] = {};
  cudaStream_t aux_streams[4] = {};        // intra-step forks (byte-limb sums)
  // Launches that may still be running on `stream` since the last serialization point
  // (programmatic dependent launches that did not wait): byte ranges read / written.
  struct Span {
    std::uintptr_t lo, hi;
  };
  struct InFlight {
    std::vector<Span> rd, wr;
  };
  std::vector<InFlight> window;
  cudaEvent_t aux_fork = nullptr, aux_join[4] = {};
  std::vector<std::pair<void*, std::size_t>> roots;  // host-path device buffers
  std::vector<std::pair<void*, std::size_t>> pinned;  // host-path staging
  // sb_context_set_kernel_order: this context's kernel phases queue behind the last kernel
  // phase of every other ordered context on the device (its copies do not)
  bool ordered = false;
  cudaEvent_t kernels_done = nullptr;
  bool profile = false;      // per-step device times (sb_context_set_profile)
  std::string profile_text;  // "step ms kernel path points" lines since the last read

  static void release(State& st) {
    cudaFree(st.d_descs);
    cudaFree(st.arena);
  }
  ~sb_context();
  void body_dtor() {
    cudaSetDevice(device);
    for (auto& [c, st] : states) release(st);
    for (auto& r : roots) cudaFree(r.first);
    for (auto& r : pinned) cudaFreeHost(r.first);
    cudaFree(d_err);
    cudaFreeHost(h_err);
    for (auto& s : lane_streams)
      if (s) cudaStreamDestroy(s);
    for (auto& e : step_events) cudaEventDestroy(e);
    for (auto& s : aux_streams)
      if (s) cudaStreamDestroy(s);
    if (aux_fork) cudaEventDestroy(aux_fork);
    for (auto& e : aux_join)
      if (e) cudaEventDestroy(e);
    if (fork_event) cudaEventDestroy(fork_event);
    for (auto& e : join_events)
      if (e) cudaEventDestroy(e);
    if (own) cudaStreamDestroy(own);
    // teardown is best effort: a failing destroy must not surface later as the "last error"
    // of an unrelated launch on this thread (non-sticky errors are consumed here)
    cudaGetLastError();
  }
};

namespace {

std::mutex g_registry_mu;
std::set<sb_context*> g_contexts;
std::atomic<std::uint64_t> g_next_plan_id{1};

}  // namespace

// Device-wide order of the kernel phases of ordered contexts (sb_context_set_kernel_order).
struct KernelOrder {
  std::mutex mu;
  cudaEvent_t last = nullptr;  // the kernels_done event of the last ordered kernel phase
};
KernelOrder g_kernel_order[64];

sb_context::~sb_context() {
  {
    std::lock_guard<std::mutex> lock(g_registry_mu);
    g_contexts.erase(this);
  }
  if (kernels_done) {
    std::lock_guard<std::mutex> lock(g_kernel_order[device & 63].mu);
    if (g_kernel_order[device & 63].last == kernels_done) g_kernel_order[device & 63].last = nullptr;
    cudaEventDestroy(kernels_done);
  }
  body_dtor();
}

sb_program::~sb_program() {
  // drop the device state every context holds for this program's plans
  std::lock_guard<std::mutex> lock(g_registry_mu);
  for (auto& [key, c] : plans) {
    for (sb_context* ctx : g_contexts) {
      std::lock_guard<std::recursive_mutex> cl(ctx->mu);
      auto it = ctx->states.find(c->id);
      if (it == ctx->states.end()) continue;
      cudaSetDevice(ctx->device);
      cudaStreamSynchronize(ctx->stream);
      sb_context::release(it->second);
      ctx->states.erase(it);
    }
  }
}

namespace {

// Plan buffers a step reads or writes.
std::vector<int> step_buffers(const sb::PStep& s) {
  std::vector<int> out;
  if (s.kind == sb::PStep::Fill) {
    out.push_back(s.buf);
    return out;
  }
  const sb::PLaunch& l = s.launch;
  switch (l.kernel) {
    case sb::KernelKind::ConvI8TC:
    case sb::KernelKind::ConvIgemmTC:
      out = {l.conv.a_buf, l.conv.b_buf, l.conv.c_buf};
      if (l.conv.epi_vec) out.push_back(l.conv.vec_buf);
      if (l.conv.epi_res) out.push_back(l.conv.res_buf);
      if (l.conv.packed) {
        out.push_back(l.conv.pack_a);
        out.push_back(l.conv.pack_b);
      }
      break;
    case sb::KernelKind::GemmF32:
    case sb::KernelKind::GemmI8TC:
      out = {l.gemm.a_buf, l.gemm.b_buf, l.gemm.c_buf, l.gemm.planes_a, l.gemm.planes_b, l.gemm.sums};
      break;
    case sb::KernelKind::Reduce:
      out = {l.reduce.in_buf, l.reduce.out_buf};
      break;
    case sb::KernelKind::Pool:
      out = {l.pool.in_buf, l.pool.out_buf};
      break;
    default:
      for (const auto& a : l.acc) out.push_back(a.buf);
  }
  return out;
}

// Scratch (locals, spills) lives in one arena.  Offsets come from live intervals over
// the non-elided steps: buffers whose [first, last] step ranges are disjoint share bytes
// (greedy first-fit, largest first); locals a fused epilogue never materialises get
// nothing.  Shared bytes are dependencies for the lane scheduler (alias()).
void layout_arena(Compiled* c) {
  const auto& plan = c->plan;
  const std::size_t nb = plan.bufs.size();
  std::vector<int> first(nb, -1), last(nb, -1);
  for (std::size_t i = 0; i < plan.steps.size(); i++) {
    const auto& s = plan.steps[i];
    if (s.elided) continue;
    for (int b : step_buffers(s)) {
      if (b < 0 || plan.bufs[b].root) continue;
      if (first[b] < 0) first[b] = static_cast<int>(i);
      last[b] = static_cast<int>(i);
    }
  }
  struct Slot {
    int buf;
    std::size_t off, bytes;
  };
  std::vector<int> order;
  for (std::size_t b = 0; b < nb; b++)
    if (first[b] >= 0) order.push_back(static_cast<int>(b));
  auto bytes_of = [&](int b) { return (plan.bufs[b].elements * kind_bytes(plan.bufs[b].kind) + 255) / 256 * 256; };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return bytes_of(a) > bytes_of(b); });
  std::vector<Slot> placed;
  std::size_t total = 0;
  for (int b : order) {
    std::vector<std::pair<std::size_t, std::size_t>> busy;
    for (const auto& q : placed)
      if (!(last[q.buf] < first[b] || last[b] < first[q.buf])) busy.emplace_back(q.off, q.off + q.bytes);
    std::sort(busy.begin(), busy.end());
    std::size_t off = 0, need = bytes_of(b);
    for (const auto& [lo, hi] : busy) {
      if (off + need <= lo) break;
      off = std::max(off, hi);
    }
    placed.push_back({b, off, need});
    total = std::max(total, off + need);
  }
  c->arena_off.assign(nb, -1);
  c->arena_bytes.assign(nb, 0);
  for (const auto& q : placed) {
    c->arena_off[q.buf] = static_cast<long long>(q.off);
    c->arena_bytes[q.buf] = static_cast<long long>(q.bytes);
  }
  c->arena_total = total;
}

Compiled* get_plan(sb_program* p, const std::vector<bool>& fresh, bool tc, int fp32_mode = 0) {
  std::string key(tc ? "T" : "G");
  key += fp32_mode == 1 ? 'x' : 'e';
  for (bool f : fresh) key += f ? '1' : '0';
  std::lock_guard<std::mutex> lock(p->mu);
  auto it = p->plans.find(key);
  if (it != p->plans.end()) return it->second.get();
  auto c = std::make_unique<Compiled>();
  c->id = g_next_plan_id++;
  sb::PlanOptions opt;
  opt.enable_tc = tc;
  opt.fresh_outputs = fresh;
  opt.fp32_tc = fp32_mode == 1;
  c->plan = sb::build_plan(p->prog, opt);
  for (const auto& s : c->plan.steps) {
    if (s.kind == sb::PStep::Launch &&
        (s.launch.kernel == sb::KernelKind::Generic || s.launch.kernel == sb::KernelKind::Map)) {
      c->desc_of_step.push_back(static_cast<int>(c->descs.size()));
      c->descs.emplace_back();
      c->bufmaps.emplace_back();
      sb::to_desc(s.launch, &c->descs.back(), &c->bufmaps.back());
    } else {
      c->desc_of_step.push_back(-1);
    }
  }
  {
    static const int max_lanes = [] {
      const char* e = std::getenv("SB_LANES");
      int v = e ? std::atoi(e) : 4;
      return v < 1 ? 1 : v > 8 ? 8 : v;
    }();
    layout_arena(c.get());
    const Compiled* cc = c.get();
    auto alias = [cc](int a, int b) {
      if (a < 0 || b < 0 || cc->arena_off[a] < 0 || cc->arena_off[b] < 0) return false;
      return cc->arena_off[a] < cc->arena_off[b] + cc->arena_bytes[b] &&
             cc->arena_off[b] < cc->arena_off[a] + cc->arena_bytes[a];
    };
    c->lanes = sb::schedule_lanes(c->plan, max_lanes, alias);
  }
  Compiled* raw = c.get();
  p->plans[key] = std::move(c);
  return raw;
}

sb_context::State& ensure_state(sb_context* ctx, const Compiled* c) {
  auto it = ctx->states.find(c->id);
  if (it != ctx->states.end()) return it->second;
  sb_context::State st;
  if (!c->descs.empty()) {
    cuda_check(cudaMalloc(&st.d_descs, sizeof(sb::GenericDesc) * c->descs.size()), "cudaMalloc(desc)");
    cuda_check(cudaMemcpy(st.d_descs, c->descs.data(), sizeof(sb::GenericDesc) * c->descs.size(),
                          cudaMemcpyHostToDevice),
               "upload desc");
  }
  const std::size_t nb = c->plan.bufs.size();
  st.scratch.assign(nb, nullptr);
  if (c->arena_total) cuda_check(cudaMalloc(&st.arena, c->arena_total), "cudaMalloc(scratch arena)");
  for (std::size_t b = 0; b < nb; b++)
    if (c->arena_off[b] >= 0) st.scratch[b] = static_cast<char*>(st.arena) + c->arena_off[b];
  st.arena_bytes = c->arena_total;
  return ctx->states.emplace(c->id, std::move(st)).first->second;
}

// Runs every plan step on the context stream.  root_ptr/root_elems indexed by root buffer.
void run_plan(sb_context* ctx, const Compiled* c, const std::vector<void*>& root_ptr) {
  auto& st = ensure_state(ctx, c);
  const auto& plan = c->plan;
  auto ptr_of = [&](int b) { return plan.bufs[b].root ? root_ptr[plan.bufs[b].root_index] : st.scratch[b]; };
  const bool single_lane = c->lanes.nlanes <= 1;
  auto span_of = [&](int b) {
    const auto lo = reinterpret_cast<std::uintptr_t>(ptr_of(b));
    return sb_context::Span{lo, lo + static_cast<std::uintptr_t>(plan.bufs[b].elements * kind_bytes(plan.bufs[b].kind))};
  };
  // writes of launches of earlier executes that may still run on this stream
  std::vector<sb_context::Span> carried_wr;
  for (const auto& w : ctx->window) carried_wr.insert(carried_wr.end(), w.wr.begin(), w.wr.end());
  // Dependency-aware PDL: a tensor-core launch that touches nothing an in-flight launch writes
  // (and writes nothing one reads) need not wait for its predecessor at all, so consecutive
  // independent executes overlap completely (the previous grid's tail wave is filled).
  // The kernels release their dependents only after their own griddepcontrol.wait has
  // returned (then their predecessor has completed), so after a waiting launch only that
  // launch may still run when the next one starts; the window holds it.  Free launches (no
  // wait) release at entry and accumulate in the window.
  // `early_b` (in/out): the launch wants to fetch plan buffer `early_b_buf` before its wait;
  // cleared when any launch that may still run writes bytes of it (e.g. the previous
  // execute's kernel producing this program's filter).
  auto pdl_mode = [&](std::size_t i, bool load_early_ok, int early_b_buf = -1, bool* early_b = nullptr) -> int {
    // Free is opt-in (SB_PDL_FREE=1): measured no gain on the configs. LoadEarly (default
    // for the resident-filter conv): when only the immediately preceding launch may still run
    // and it writes nothing this launch reads, the loads and MMAs start at once and only the
    // stores wait for the predecessor (WAW / WAR ordering kept).
    static const bool allow_free = std::getenv("SB_PDL_FREE") != nullptr;
    static const bool load_early = std::getenv("SB_PDL_NO_EARLY") == nullptr;
    auto ov = [](const std::vector<sb_context::Span>& x, const std::vector<sb_context::Span>& y) {
      for (const auto& a : x)
        for (const auto& b : y)
          if (a.lo < b.hi && b.lo < a.hi) return true;
      return false;
    };
    if (early_b && *early_b && early_b_buf >= 0) {
      // b_immutable: no step of this plan writes it; only earlier executes on this stream can
      const std::vector<sb_context::Span> bs{span_of(early_b_buf)};
      if (ov(carried_wr, bs)) *early_b = false;
      for (const auto& w : ctx->window)
        if (ov(w.wr, bs)) *early_b = false;
    }
    if (!single_lane) {
      ctx->window.clear();
      return sb::kPdlWait;
    }
    std::vector<int> rd, wr;
    sb::step_access(plan.steps[i], &rd, &wr);
    sb_context::InFlight me;
    for (int b : rd) me.rd.push_back(span_of(b));
    for (int b : wr) me.wr.push_back(span_of(b));
    bool raw = false, any = false;
    for (const auto& w : ctx->window) {
      raw |= ov(w.wr, me.rd);
      any |= ov(w.wr, me.rd) || ov(w.wr, me.wr) || ov(w.rd, me.wr);
    }
    if (allow_free && !any && ctx->window.size() < 64) {
      ctx->window.push_back(std::move(me));
      return sb::kPdlFree;
    }
    const std::size_t inflight = ctx->window.size();  // 0/1: only the preceding launch may still run
    ctx->window.clear();
    ctx->window.push_back(std::move(me));
    if (inflight <= 1 && !raw && load_early && load_early_ok) return sb::kPdlLoadEarly;
    return inflight <= 1 ? sb::kPdlWait : sb::kPdlOff;
  };
  auto step = [&](std::size_t i) {
    const auto& s = plan.steps[i];
    if (s.elided) return;
    const bool tc_single = s.kind == sb::PStep::Launch &&
                           ((s.launch.kernel == sb::KernelKind::ConvI8TC) ||
                            (s.launch.kernel == sb::KernelKind::ConvIgemmTC && !s.launch.conv.packed) ||
                            (s.launch.kernel == sb::KernelKind::GemmI8TC && !s.launch.gemm.limbs_a));
    if (!tc_single) ctx->window.clear();  // plain stream-ordered launches serialize everything
    if (s.kind == sb::PStep::Fill) {
      const auto& pb = plan.bufs[s.buf];
      cuda_check(sb::launch_fill(ptr_of(s.buf), pb.kind, pb.elements, s.value, ctx->stream), "fill");
      ctx->launches++;
      return;
    }
    const sb::PLaunch& l = s.launch;
    if (l.kernel == sb::KernelKind::ConvI8TC || l.kernel == sb::KernelKind::ConvIgemmTC) {
      sb::ConvArgs a;
      a.a = ptr_of(l.conv.a_buf);
      a.b = ptr_of(l.conv.b_buf);
      a.c = ptr_of(l.conv.c_buf);
      a.a_elems = plan.bufs[l.conv.a_buf].elements;
      a.b_elems = plan.bufs[l.conv.b_buf].elements;
      a.c_elems = plan.bufs[l.conv.c_buf].elements;
      bool b_early = l.conv.b_immutable;
      if (l.conv.epi_vec) {
        a.vec = ptr_of(l.conv.vec_buf);
        a.vec_kind = plan.bufs[l.conv.vec_buf].kind;
      }
      if (l.conv.epi_res) a.res = ptr_of(l.conv.res_buf);
      if (tc_single) a.pdl_mode = pdl_mode(i, l.kernel == sb::KernelKind::ConvI8TC, l.conv.b_buf, &b_early);
      a.b_immutable = b_early;
      if (l.kernel == sb::KernelKind::ConvI8TC) {
        cuda_check(sb::launch_conv_tc(l.conv, a, ctx->stream, ctx->num_sms), "conv_tc");
      } else if (l.conv.packed && l.conv.fold_x) {
        // phase-folded small-channel conv: fold the input and the filter, then the stride-1
        // im2col conv over the folded copy (packed_view)
        // (band_raw: the conv's producer warps fold the raw rows themselves)
        void* fa = ptr_of(l.conv.pack_a);
        void* pb = ptr_of(l.conv.pack_b);
        if (!l.conv.band_raw) {
          cuda_check(sb::launch_conv_fold(l.conv, a.a, fa, ctx->stream), "conv_fold");
          ctx->launches++;
          a.a = fa;
        }
        cuda_check(sb::launch_conv_pack_filter(l.conv, a.b, pb, ctx->stream), "conv_pack_filter");
        ctx->launches++;
        a.b = pb;
        cuda_check(sb::launch_conv_igemm(sb::packed_view(l.conv), a, ctx->stream, ctx->num_sms), "conv_igemm");
      } else if (l.conv.packed) {
        // small-channel conv: filter packed to [K, pack_k]; A rows gathered inside the kernel
        void* pb = ptr_of(l.conv.pack_b);
        cuda_check(sb::launch_conv_pack_filter(l.conv, a.b, pb, ctx->stream), "conv_pack_filter");
        ctx->launches++;
        a.b = pb;
        cuda_check(sb::launch_conv_igemm(l.conv, a, ctx->stream, ctx->num_sms), "conv_igemm");
      } else {
        cuda_check(sb::launch_conv_igemm(l.conv, a, ctx->stream, ctx->num_sms), "conv_igemm");
      }
      ctx->launches++;
      return;
    }
    if (l.kernel == sb::KernelKind::GemmF32 && l.gemm.tf32x3) {
      const sb::GemmPlan& g = l.gemm;
      void* pa = ptr_of(g.planes_a);
      void* pb = ptr_of(g.planes_b);
      char* sums = static_cast<char*>(ptr_of(g.sums));
      cuda_check(sb::launch_tf32_split(g, ptr_of(g.a_buf), ptr_of(g.b_buf), pa, pb, ctx->stream), "tf32_split");
      ctx->launches++;
      auto ev = [](cudaEvent_t* e) {
        if (!*e) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        return *e;
      };
      cuda_check(cudaEventRecord(ev(&ctx->aux_fork), ctx->stream), "tf32 fork");
      for (int t = 0; t < 3; t++) {
        cudaStream_t s = ctx->stream;
        if (t > 0) {
          if (!ctx->aux_streams[t]) cuda_check(cudaStreamCreateWithFlags(&ctx->aux_streams[t], cudaStreamNonBlocking), "aux");
          s = ctx->aux_streams[t];
          cuda_check(cudaStreamWaitEvent(s, ctx->aux_fork, 0), "tf32 fork wait");
        }
        sb::GemmArgs a{pa, pb, sums + 4ll * t * g.M * g.N};
        cuda_check(sb::launch_gemm_tc(sb::tf32_sum_plan(g, t), a, s, ctx->num_sms), "gemm_tc(tf32x3)");
        ctx->launches++;
        if (t > 0) cuda_check(cudaEventRecord(ev(&ctx->aux_join[t]), s), "tf32 join");
      }
      for (int t = 1; t < 3; t++) cuda_check(cudaStreamWaitEvent(ctx->stream, ctx->aux_join[t], 0), "tf32 join wait");
      cuda_check(sb::launch_tf32_combine(g, sums, ptr_of(g.c_buf), ctx->stream), "tf32_combine");
      ctx->launches++;
      return;
    }
    if (l.kernel == sb::KernelKind::GemmF32) {
      cuda_check(sb::launch_gemm_f32(l.gemm, ptr_of(l.gemm.a_buf), ptr_of(l.gemm.b_buf), ptr_of(l.gemm.c_buf),
                                     ctx->stream),
                 "gemm_f32");
      ctx->launches++;
      return;
    }
    if (l.kernel == sb::KernelKind::GemmI8TC && l.gemm.limbs_a && l.gemm.limb_fused) {
      const sb::GemmPlan& g = l.gemm;
      cuda_check(sb::launch_limb_fused(g, ptr_of(g.a_buf), ptr_of(g.b_buf), ptr_of(g.planes_a), ptr_of(g.planes_b),
                                       ptr_of(g.c_buf), ctx->stream, ctx->num_sms),
                 "gemm_limb");
      ctx->launches += 3;
      return;
    }
    if (l.kernel == sb::KernelKind::GemmI8TC && l.gemm.limbs_a) {
      const sb::GemmPlan& g = l.gemm;
      char* pa = static_cast<char*>(ptr_of(g.planes_a));
      char* pb = static_cast<char*>(ptr_of(g.planes_b));
      char* sums = static_cast<char*>(ptr_of(g.sums));
      cuda_check(sb::launch_limb_split(g, ptr_of(g.a_buf), ptr_of(g.b_buf), pa, pb, ctx->stream), "limb_split");
      ctx->launches += 2;
      // the sums are independent GEMMs: run them side by side (each alone fills only
      // ceil(M/128) * ceil(N/128) CTAs), joined before the combine
      auto ev = [](cudaEvent_t* e) {
        if (!*e) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        return *e;
      };
      const int ns = sb::limb_smax(g) + 1;
      cuda_check(cudaEventRecord(ev(&ctx->aux_fork), ctx->stream), "limb fork");
      for (int t = 0; t < ns; t++) {
        cudaStream_t s = ctx->stream;
        if (t > 0) {
          if (!ctx->aux_streams[t]) cuda_check(cudaStreamCreateWithFlags(&ctx->aux_streams[t], cudaStreamNonBlocking), "aux");
          s = ctx->aux_streams[t];
          cuda_check(cudaStreamWaitEvent(s, ctx->aux_fork, 0), "limb fork wait");
        }
        sb::GemmArgs a{pa + sb::limb_a_off(g, t), pb + sb::limb_b_off(g, t), sums + 4ll * t * g.M * g.N};
        cuda_check(sb::launch_gemm_tc(sb::limb_sum_plan(g, t), a, s, ctx->num_sms), "gemm_tc(limb)");
        ctx->launches++;
        if (t > 0) cuda_check(cudaEventRecord(ev(&ctx->aux_join[t]), s), "limb join");
      }
      for (int t = 1; t < ns; t++) cuda_check(cudaStreamWaitEvent(ctx->stream, ctx->aux_join[t], 0), "limb join wait");
      cuda_check(sb::launch_limb_combine(g, sums, ptr_of(g.c_buf), ctx->stream), "limb_combine");
      ctx->launches++;
      return;
    }
    if (l.kernel == sb::KernelKind::GemmI8TC) {
      sb::GemmArgs a{ptr_of(l.gemm.a_buf), ptr_of(l.gemm.b_buf), ptr_of(l.gemm.c_buf)};
      a.pdl_mode = pdl_mode(i, false);
      cuda_check(sb::launch_gemm_tc(l.gemm, a, ctx->stream, ctx->num_sms), "gemm_tc");
      ctx->launches++;
      return;
    }
    if (l.kernel == sb::KernelKind::Pool) {
      cuda_check(sb::launch_pool(l.pool, ptr_of(l.pool.in_buf), ptr_of(l.pool.out_buf), ctx->stream), "pool");
      ctx->launches++;
      return;
    }
    if (l.kernel == sb::KernelKind::Reduce) {
      sb::ReduceArgs a;
      std::memset(&a, 0, sizeof(a));
      const sb::ReducePlan& r = l.reduce;
      a.in = ptr_of(r.in_buf);
      a.out = ptr_of(r.out_buf);
      a.in_kind = r.in_kind;
      a.out_kind = r.out_kind;
      a.agg = r.agg;
      a.fresh = r.fresh ? 1 : 0;
      a.identity = r.identity;
      a.np = r.np;
      a.nr = r.nr;
      a.rcount = r.rcount;
      for (int k = 0; k < r.np; k++) {
        a.prange[k] = r.prange[k];
        a.pin[k] = r.pin[k];
        a.pout[k] = r.pout[k];
      }
      for (int k = 0; k < r.nr; k++) {
        a.rrange[k] = r.rrange[k];
        a.rstep[k] = r.rstep[k];
      }
      a.in_c = r.in_c;
      a.out_c = r.out_c;
      a.pcount = r.pcount;
      cuda_check(sb::launch_reduce(a, ctx->stream), "reduce");
      ctx->launches++;
      return;
    }
    int di = c->desc_of_step[i];
    sb::BufTable t;
    std::memset(&t, 0, sizeof(t));
    const auto& map = c->bufmaps[di];
    for (std::size_t k = 0; k < map.size(); k++) {
      t.ptr[k] = ptr_of(map[k]);
      t.elems[k] = plan.bufs[map[k]].elements;
      t.kind[k] = plan.bufs[map[k]].kind;
    }
    if (l.is_float)
      cuda_check(sb::launch_generic_f32(st.d_descs + di, l.pcount, t, ctx->d_err, static_cast<int>(i), ctx->stream),
                 "generic_f32");
    else if (l.kernel == sb::KernelKind::Map)
      cuda_check(sb::launch_map(st.d_descs + di, l.vcount, t, ctx->d_err, static_cast<int>(i), ctx->stream), "map");
    else
      cuda_check(sb::launch_generic(st.d_descs + di, l.pcount, t, ctx->d_err, static_cast<int>(i), ctx->stream),
                 "generic");
    ctx->launches++;
  };
  static const bool profile_env = std::getenv("SB_PROFILE_STEPS") != nullptr;
  const bool profile = profile_env || ctx->profile;
  const sb::LaneSchedule& ls = c->lanes;
  if (!profile && ls.nlanes > 1) {
    // independent steps on parallel lanes (events only where a step depends across lanes)
    const cudaStream_t main = ctx->stream;
    auto ev = [](cudaEvent_t* e) {
      if (!*e) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
      return *e;
    };
    if (ctx->step_events.size() < plan.steps.size()) ctx->step_events.resize(plan.steps.size(), nullptr);
    cuda_check(cudaEventRecord(ev(&ctx->fork_event), main), "fork");
    for (int L = 1; L < ls.nlanes; L++) {
      if (!ctx->lane_streams[L]) cuda_check(cudaStreamCreateWithFlags(&ctx->lane_streams[L], cudaStreamNonBlocking), "lane");
      cuda_check(cudaStreamWaitEvent(ctx->lane_streams[L], ctx->fork_event, 0), "fork wait");
    }
    for (std::size_t i = 0; i < plan.steps.size(); i++) {
      if (plan.steps[i].elided) continue;
      const cudaStream_t s = ls.lane[i] == 0 ? main : ctx->lane_streams[ls.lane[i]];
      for (int w : ls.waits[i]) cuda_check(cudaStreamWaitEvent(s, ctx->step_events[w], 0), "dep wait");
      ctx->stream = s;
      step(i);
      ctx->stream = main;
      if (ls.signal[i]) cuda_check(cudaEventRecord(ev(&ctx->step_events[i]), s), "dep record");
    }
    for (int L = 1; L < ls.nlanes; L++) {
      cuda_check(cudaEventRecord(ev(&ctx->join_events[L]), ctx->lane_streams[L]), "join");
      cuda_check(cudaStreamWaitEvent(main, ctx->join_events[L], 0), "join wait");
    }
    // conservatively, any of this execute's launches may still run when the next one starts:
    // its reads and writes form one in-flight entry for the next execute's PDL decisions
    sb_context::InFlight all;
    for (std::size_t i = 0; i < plan.steps.size(); i++) {
      if (plan.steps[i].elided) continue;
      std::vector<int> rd, wr;
      sb::step_access(plan.steps[i], &rd, &wr);
      for (int b : rd) all.rd.push_back(span_of(b));
      for (int b : wr) all.wr.push_back(span_of(b));
    }
    ctx->window.clear();
    ctx->window.push_back(std::move(all));
    return;
  }
  if (!profile) {
    for (std::size_t i = 0; i < plan.steps.size(); i++) step(i);
    return;
  }
  // tracing aid: per-step device time (events on the context stream), printed to stderr
  std::vector<cudaEvent_t> ev(plan.steps.size() + 1);
  for (auto& e : ev) cudaEventCreate(&e);
  for (std::size_t i = 0; i < plan.steps.size(); i++) {
    cudaEventRecord(ev[i], ctx->stream);
    step(i);
  }
  cudaEventRecord(ev.back(), ctx->stream);
  cudaEventSynchronize(ev.back());
  static const char* kinds[] = {"generic", "conv_i8_tc", "map", "reduce", "gemm_i8_tc", "conv_igemm_tc", "pool", "gemm_f32"};
  for (std::size_t i = 0; i < plan.steps.size(); i++) {
    const auto& s = plan.steps[i];
    if (s.elided) continue;
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
    char line[512];
    if (s.kind == sb::PStep::Fill)
      std::snprintf(line, sizeof(line), "%zu %.6f fill %s %lld\n", i, ms, plan.bufs[s.buf].name.c_str(),
                    static_cast<long long>(plan.bufs[s.buf].elements));
    else
      std::snprintf(line, sizeof(line), "%zu %.6f %s %s %lld\n", i, ms, kinds[static_cast<int>(s.launch.kernel)],
                    s.launch.path.c_str(), static_cast<long long>(s.launch.points));
    if (ctx->profile) ctx->profile_text += line;
    if (profile_env) std::fprintf(stderr, "[sb step] %s", line);
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

void check_device_error(sb_context* ctx, const Compiled* c) {
  cuda_check(cudaStreamSynchronize(ctx->stream), "stream sync");
  if (ctx->h_err->code == 0) return;
  cuda_check(cudaMemcpy(ctx->h_err, ctx->d_err, sizeof(sb::DevError), cudaMemcpyDeviceToHost), "err read");
  sb::DevError e = *ctx->h_err;
  sb::DevError zero{};
  cudaMemcpy(ctx->d_err, &zero, sizeof(zero), cudaMemcpyHostToDevice);
  ctx->h_err->code = 0;
  if (e.code == 0) return;
  std::string where = c && e.launch >= 0 && e.launch < static_cast<int>(c->plan.steps.size())
                          ? c->plan.steps[e.launch].launch.path
                          : "?";
  if (e.code == 2)
    throw sb::Error("OutOfBoundsAccess", "gather/scatter index " + std::to_string(e.addr) +
                                             " outside range in block " + where);
  throw sb::Error("OutOfBoundsAccess", "access at element " + std::to_string(e.addr) +
                                           " outside buffer in block " + where);
}

std::vector<bool> fresh_flags(const sb::Program& prog, const std::vector<int>& slot_of_root,
                              const std::vector<int>& flags) {
  std::vector<bool> fresh(prog.buffers.size(), false);
  for (std::size_t r = 0; r < prog.buffers.size(); r++)
    fresh[r] = slot_of_root[r] >= 0 && (flags[slot_of_root[r]] & SB_BUF_PREPARE) &&
               prog.buffers[r].dir != sb::Dir::In;
  return fresh;
}

void check_opts(const sb_exec_options* o) {
  if (o && o->observer)
    throw sb::Error("Unsupported", "execution observers are not supported by the device executor");
}

}  // namespace

extern "C" {

const char* sb_last_error(void) { return g_last_error.c_str(); }
int sb_abi_version(void) { return SB_ABI_VERSION; }

const char* sb_status_name(int s) {
  static const char* names[] = {"Ok",           "MissingBuffer",  "UnknownIntrinsic", "UnknownSpecial",
                                "UndefinedTemp", "OutOfBoundsAccess", "UnboundIndex",   "SyntaxError",
                                "ScopeError",   "Unsupported",    "CudaError",        "NcclError",
                                "Invalid",      "PassError"};
  return s >= 0 && s <= 13 ? names[s] : "Invalid";
}

int sb_program_parse(const char* text, sb_program** out) {
  return guarded([&] {
    if (!text || !out) throw sb::Error("Invalid", "null argument");
    auto p = std::make_unique<sb_program>();
    p->prog = sb::parse_program(text);
    *out = p.release();
  });
}

void sb_program_free(sb_program* p) { delete p; }

int sb_program_print(const sb_program* p, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::string s = sb::print_program(p->prog);
    if (len) *len = s.size();
    if (buf && cap) {
      std::size_t n = std::min(s.size(), cap - 1);
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

int sb_program_buffer_count(const sb_program* p) { return static_cast<int>(p->prog.buffers.size()); }

int sb_program_buffer_info(const sb_program* p, int i, const char** name, int* dtype,
                           int64_t* elements, int* dir) {
  return guarded([&] {
    if (i < 0 || i >= static_cast<int>(p->prog.buffers.size())) throw sb::Error("Invalid", "buffer index");
    const auto& b = p->prog.buffers[i];
    if (name) *name = b.name.c_str();
    if (dtype) *dtype = b.dtype == sb::DType::F32 ? SB_F32 : sb::dtype_bits(b.dtype);
    if (elements) *elements = b.elements;
    if (dir) *dir = static_cast<int>(b.dir);
  });
}

int sb_program_output_identity(const sb_program* p, const char* name, int64_t* value) {
  return guarded([&] { *value = sb::output_identity(p->prog, name); });
}

int sb_program_output_aggregation(const sb_program* p, const char* name, int* agg) {
  return guarded([&] { *agg = static_cast<int>(sb::output_aggregation(p->prog, name)); });
}

namespace {
const sb::Block* block_at(const sb_program* p, const char* block_path) {
  const sb::Block* b = &p->prog.root;
  std::string path = block_path ? block_path : "";
  std::stringstream ss(path);
  std::string part;
  while (!path.empty() && std::getline(ss, part, '.')) {
    const std::size_t k = static_cast<std::size_t>(std::stoll(part));
    if (k >= b->stmts.size() || b->stmts[k].kind != sb::StmtKind::Block)
      throw sb::Error("Unsupported", "no block at path '" + path + "'");
    b = b->stmts[k].block.get();
  }
  return b;
}

void put_report(const sb::TileReport& r, sb_tile_report* out) {
  out->lines_total = r.lines_total;
  out->useful_ops = r.useful_ops;
  out->tile_elements = r.tile_elements;
  out->excluded = r.excluded ? 1 : 0;
}
}  // namespace

int sb_tile_cost(sb_context* ctx, const sb_program* p, const char* block_path, const char* tiles, int interleaved,
                 int64_t line, int64_t mem_cap, sb_tile_report* out) {
  return guarded([&] {
    if (!out) throw sb::Error("Invalid", "null report");
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    const auto shape = sb::parse_tile_shape_text(tiles ? tiles : "");
    sb::TileCoster tc(*block_at(p, block_path), line, mem_cap, ctx->stream);
    put_report(tc.tile_cost(shape, interleaved != 0), out);
  });
}

int sb_autotile(sb_context* ctx, const sb_program* p, const char* block_path, int64_t line, int64_t mem_cap,
                int power_of_two, char* chosen, size_t cap, size_t* len, int* found, sb_tile_report* report,
                int64_t* candidates, int64_t* excluded) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    sb::TileCoster tc(*block_at(p, block_path), line, mem_cap, ctx->stream);
    const sb::AutotileResult r = tc.autotile(power_of_two != 0);
    const std::string text = r.found ? tc.shape_text(r.chosen) : "";
    if (len) *len = text.size();
    if (chosen && cap) {
      const std::size_t n = std::min(cap - 1, text.size());
      std::memcpy(chosen, text.data(), n);
      chosen[n] = 0;
    }
    if (found) *found = r.found ? 1 : 0;
    if (report) put_report(r.report, report);
    if (candidates) *candidates = r.candidates;
    if (excluded) *excluded = r.excluded;
  });
}

int sb_count_valid_points(sb_context* ctx, const sb_program* p, const char* block_path, int64_t* count) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    const sb::Block* b = block_at(p, block_path);
    // the reference's definition: the block's own ranged indexes, its own constraints
    std::vector<long long> ranges;
    std::vector<std::string> names;
    for (const auto& idx : b->indexes) {
      if (idx.is_alias) throw sb::Error("InvalidTile", "count_valid_points requires alias-free blocks");
      names.push_back(idx.name);
      ranges.push_back(idx.range);
    }
    std::int64_t total = 1;
    for (auto r : ranges) total *= r;
    if (ranges.empty()) {
      ranges.push_back(1);
      names.push_back("");
    }
    const int nd = static_cast<int>(ranges.size()), nc = static_cast<int>(b->constraints.size());
    std::vector<long long> cc(nc), ck(static_cast<std::size_t>(nc) * nd, 0);
    for (int c = 0; c < nc; c++) {
      cc[c] = b->constraints[c].constant;
      for (const auto& [name, k] : b->constraints[c].terms) {
        auto it = std::find(names.begin(), names.end(), name);
        if (it == names.end()) throw sb::Error("UnboundIndex", "unbound index '" + name + "'");
        ck[static_cast<std::size_t>(c) * nd + (it - names.begin())] = k;
      }
    }
    if (total == 0) {
      *count = 0;
      return;
    }
    void* scratch = nullptr;
    cuda_check(cudaMalloc(&scratch, sb::count_points_scratch_bytes()), "cudaMalloc(count)");
    unsigned long long h = 0;
    cudaError_t e = sb::launch_count_points(nd, ranges.data(), nc, cc.data(), ck.data(), scratch, &h, ctx->stream);
    cudaFree(scratch);
    cuda_check(e, "count_points");
    *count = static_cast<std::int64_t>(h);
  });
}

int sb_nccl_unique_id(char* id) {
  return guarded([&] {
    if (!id) throw sb::Error("Invalid", "null id buffer");
    char buf[128];
    sb::nccl_unique_id(buf);
    std::memcpy(id, buf, 128);
  });
}

int sb_nccl_comm_init(sb_context* ctx, int nranks, const char* id, int rank, void** comm) {
  return guarded([&] {
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) throw sb::Error("Invalid", "bad communicator arguments");
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    *comm = sb::nccl_comm_init(nranks, id, rank);
  });
}

int sb_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (comm) sb::nccl_comm_destroy(comm);
  });
}

int sb_split_allreduce(sb_context* ctx, const sb_program* p, const char* name, void* data, int64_t count,
                       void* nccl_comm) {
  return guarded([&] {
    if (!name || !nccl_comm || (count > 0 && !data)) throw sb::Error("Invalid", "null argument");
    const int r = p->prog.buffer_index(name);
    if (r < 0) throw sb::Error("MissingBuffer", std::string("no buffer '") + name + "'");
    const auto& b = p->prog.buffers[r];
    if (b.dir == sb::Dir::In) throw sb::Error("Unsupported", std::string("'") + name + "' is an input");
    if (count != b.elements)
      throw sb::Error("MissingBuffer", "buffer '" + b.name + "' has " + std::to_string(count) + " elements, expected " +
                                           std::to_string(b.elements));
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    ctx->window.clear();  // a collective is a serialization point of the stream
    sb::split_allreduce(nccl_comm, data, count, b.dtype, sb::output_aggregation(p->prog, name), ctx->stream);
  });
}

int sb_program_restrict_index(const sb_program* p, const char* block_path, const char* index, int64_t lo, int64_t hi,
                              sb_program** out) {
  return guarded([&] {
    auto q = std::make_unique<sb_program>();
    q->prog = sb::restrict_index(p->prog, block_path ? block_path : "", index, lo, hi);
    *out = q.release();
  });
}

int sb_program_check_split(const sb_program* p, const char* block_path, const char* index) {
  return guarded([&] { sb::check_split(p->prog, block_path ? block_path : "", index ? index : ""); });
}

int sb_program_describe_plan(sb_program* p, int fresh_outputs, int disable_tc, char* buf, size_t cap,
                             size_t* len) {
  return guarded([&] {
    std::vector<bool> fresh(p->prog.buffers.size(), false);
    for (std::size_t r = 0; r < fresh.size(); r++) fresh[r] = fresh_outputs && p->prog.buffers[r].dir != sb::Dir::In;
    Compiled* c = get_plan(p, fresh, !(disable_tc & 1), (disable_tc & 2) ? 1 : 0);
    std::string s = c->plan.describe();
    if (c->lanes.nlanes > 1) {
      s += "lanes " + std::to_string(c->lanes.nlanes) + ":";
      for (std::size_t i = 0; i < c->plan.steps.size(); i++)
        if (!c->plan.steps[i].elided) s += " " + std::to_string(c->lanes.lane[i]);
      s += "\n";
    }
    s += "arena " + std::to_string(c->arena_total) + " bytes\n";
    if (len) *len = s.size();
    if (buf && cap) {
      std::size_t n = std::min(s.size(), cap - 1);
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

int sb_context_create(int device, sb_context** out) {
  return guarded([&] {
    int count = 0;
    cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) throw sb::Error("CudaError", "no such device");
    cudaDeviceProp prop;
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
      throw sb::Error("CudaError", std::string("device is not sm_100 (Blackwell): ") + prop.name);
    auto ctx = std::make_unique<sb_context>();
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking), "cudaStreamCreate");
    ctx->stream = ctx->own;
    cuda_check(cudaMalloc(&ctx->d_err, sizeof(sb::DevError)), "cudaMalloc(err)");
    cuda_check(cudaMemset(ctx->d_err, 0, sizeof(sb::DevError)), "memset(err)");
    cuda_check(cudaMallocHost(&ctx->h_err, sizeof(sb::DevError)), "cudaMallocHost");
    // h_err->code doubles as a "maybe dirty" hint; the authoritative copy is read on sync.
    ctx->h_err->code = 1;
    {
      std::lock_guard<std::mutex> lock(g_registry_mu);
      g_contexts.insert(ctx.get());
    }
    *out = ctx.release();
  });
}

void sb_context_destroy(sb_context* ctx) { delete ctx; }

int sb_context_set_stream(sb_context* ctx, void* s) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
    ctx->window.clear();
  });
}

void* sb_context_stream(sb_context* ctx) { return ctx->stream; }

int sb_context_set_kernel_order(sb_context* ctx, int enable) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (enable && !ctx->kernels_done)
      cuda_check(cudaEventCreateWithFlags(&ctx->kernels_done, cudaEventDisableTiming), "cudaEventCreate(order)");
    ctx->ordered = enable != 0;
  });
}

int sb_context_sync(sb_context* ctx) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    ctx->window.clear();
    ctx->h_err->code = 1;
    check_device_error(ctx, nullptr);
  });
}

int sb_context_set_profile(sb_context* ctx, int enable) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    ctx->profile = enable != 0;
    ctx->profile_text.clear();
  });
}

int sb_context_profile_read(sb_context* ctx, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    if (len) *len = ctx->profile_text.size();
    if (buf && cap) {
      std::size_t n = std::min(ctx->profile_text.size(), cap - 1);
      std::memcpy(buf, ctx->profile_text.data(), n);
      buf[n] = 0;
      ctx->profile_text.clear();
    }
  });
}

uint64_t sb_context_launch_count(sb_context* ctx) {
  std::lock_guard<std::recursive_mutex> lock(ctx->mu);
  return ctx->launches;
}

int sb_device_alloc(sb_context* ctx, int64_t bytes, void** dptr) {
  return guarded([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_check(cudaMalloc(dptr, padded(static_cast<std::size_t>(bytes))), "cudaMalloc");
  });
}

int sb_device_free(sb_context* ctx, void* dptr) {
  return guarded([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_check(cudaFree(dptr), "cudaFree");
  });
}

int sb_host_alloc_pinned(int64_t bytes, void** ptr) {
  return guarded([&] { cuda_check(cudaMallocHost(ptr, padded(static_cast<std::size_t>(bytes))), "cudaMallocHost"); });
}

int sb_host_free_pinned(void* ptr) { return guarded([&] { cuda_check(cudaFreeHost(ptr), "cudaFreeHost"); }); }

int sb_execute_device(sb_context* ctx, sb_program* p, const sb_device_buffer* bufs, int n,
                      const sb_exec_options* opts) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    check_opts(opts);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaGetLastError();  // a stale non-sticky error of an unrelated earlier runtime call is not ours
    const auto& prog = p->prog;
    std::vector<int> slot(prog.buffers.size(), -1);
    std::vector<int> flags(n);
    for (int i = 0; i < n; i++) {
      flags[i] = bufs[i].flags;
      int r = prog.buffer_index(bufs[i].name ? bufs[i].name : "");
      if (r >= 0) slot[r] = i;
    }
    std::vector<void*> ptrs(prog.buffers.size(), nullptr);
    for (std::size_t r = 0; r < prog.buffers.size(); r++) {
      if (slot[r] < 0)
        throw sb::Error("MissingBuffer", "buffer '" + prog.buffers[r].name + "' not present in store");
      if (bufs[slot[r]].count != prog.buffers[r].elements)
        throw sb::Error("MissingBuffer", "buffer '" + prog.buffers[r].name + "' has " +
                                             std::to_string(bufs[slot[r]].count) + " elements, expected " +
                                             std::to_string(prog.buffers[r].elements));
      ptrs[r] = bufs[slot[r]].dptr;
    }
    Compiled* c = get_plan(p, fresh_flags(prog, slot, flags), !(opts && opts->disable_tensor_cores),
                           opts ? opts->fp32_mode : 0);
    for (std::size_t r = 0; r < prog.buffers.size(); r++) {
      if ((flags[slot[r]] & SB_BUF_PREPARE) && prog.buffers[r].dir != sb::Dir::In) {
        const auto& b = prog.buffers[r];
        bool consumed = false;  // a matched kernel overwrites fresh outputs itself
        for (const auto& s : c->plan.steps)
          if (s.kind == sb::PStep::Launch && s.launch.fused_fill_root == static_cast<int>(r)) consumed = true;
        if (!consumed) {
          cuda_check(sb::launch_fill(ptrs[r], c->plan.bufs[r].kind, b.elements, sb::output_identity(prog, b.name),
                                     ctx->stream),
                     "prepare_outputs");
          ctx->launches++;
          ctx->window.clear();  // a plain stream-ordered launch: everything before it has completed
        }
      }
    }
    run_plan(ctx, c, ptrs);
  });
}

}  // extern "C"

namespace {
// int64 carriers <-> native width on the host (the drop-in boundary's BufferStore, interp.h:14-17):
// memory-bound loops split over host threads for large buffers.
template <typename F>
void parallel_elems(std::int64_t n, F&& f) {
  const std::int64_t kMin = 1 << 20;
  unsigned hw = std::thread::hardware_concurrency();
  int nt = static_cast<int>(std::min<std::int64_t>(std::max(1u, std::min(hw, 16u)), (n + kMin - 1) / kMin));
  if (nt <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const std::int64_t chunk = (n + nt - 1) / nt;
  for (int t = 1; t < nt; t++) {
    const std::int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  f(0, std::min(n, chunk));
  for (auto& x : th) x.join();
}

void narrow_from_i64(const std::int64_t* in, void* out, int kind, std::int64_t n) {
  parallel_elems(n, [&](std::int64_t lo, std::int64_t hi) {
    switch (kind) {
      case sb::kI8: for (std::int64_t e = lo; e < hi; e++) static_cast<std::int8_t*>(out)[e] = static_cast<std::int8_t>(in[e]); break;
      case sb::kI16: for (std::int64_t e = lo; e < hi; e++) static_cast<std::int16_t*>(out)[e] = static_cast<std::int16_t>(in[e]); break;
      default: for (std::int64_t e = lo; e < hi; e++) static_cast<std::int32_t*>(out)[e] = static_cast<std::int32_t>(in[e]); break;
    }
  });
}

void widen_to_i64(const void* in, std::int64_t* out, int kind, std::int64_t n) {
  parallel_elems(n, [&](std::int64_t lo, std::int64_t hi) {
    switch (kind) {
      case sb::kI8: for (std::int64_t e = lo; e < hi; e++) out[e] = static_cast<const std::int8_t*>(in)[e]; break;
      case sb::kI16: for (std::int64_t e = lo; e < hi; e++) out[e] = static_cast<const std::int16_t*>(in)[e]; break;
      default: for (std::int64_t e = lo; e < hi; e++) out[e] = static_cast<const std::int32_t*>(in)[e]; break;
    }
  });
}

int execute_host(sb_context* ctx, sb_program* p, sb_host_buffer* bufs, int n, const sb_exec_options* opts, bool async) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cudaSetDevice(ctx->device);
    cudaGetLastError();   // a stale non-sticky error of an unrelated earlier runtime call is not ours
    ctx->window.clear();  // host copies serialize the stream
    if (async)
      for (int i = 0; i < n; i++)
        if (bufs[i].carrier != SB_CARRIER_NATIVE)
          throw sb::Error("Unsupported", "sb_execute_async needs native-width carriers (pinned host memory)");
    check_opts(opts);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    const auto& prog = p->prog;
    std::vector<int> slot(prog.buffers.size(), -1);
    std::vector<int> flags(n);
    for (int i = 0; i < n; i++) {
      flags[i] = bufs[i].flags;
      int r = prog.buffer_index(bufs[i].name ? bufs[i].name : "");
      if (r >= 0) slot[r] = i;
    }
    // Executor::run's buffer-table check (interp.cpp:184-194).
    for (std::size_t r = 0; r < prog.buffers.size(); r++) {
      if (slot[r] < 0)
        throw sb::Error("MissingBuffer", "buffer '" + prog.buffers[r].name + "' not present in store");
      if (bufs[slot[r]].count != prog.buffers[r].elements)
        throw sb::Error("MissingBuffer", "buffer '" + prog.buffers[r].name + "' has " +
                                             std::to_string(bufs[slot[r]].count) + " elements, expected " +
                                             std::to_string(prog.buffers[r].elements));
    }
    Compiled* c = get_plan(p, fresh_flags(prog, slot, flags), !(opts && opts->disable_tensor_cores),
                           opts ? opts->fp32_mode : 0);
    const std::size_t nr = prog.buffers.size();
    if (ctx->roots.size() < nr) ctx->roots.resize(nr, {nullptr, 0});
    if (ctx->pinned.size() < nr) ctx->pinned.resize(nr, {nullptr, 0});
    std::vector<void*> ptrs(nr);
    std::vector<sb_device_buffer> dev(nr);
    for (std::size_t r = 0; r < nr; r++) {
      const auto& b = prog.buffers[r];
      const sb_host_buffer& hb = bufs[slot[r]];
      int kind = c->plan.bufs[r].kind;
      std::size_t bytes = padded(b.elements * kind_bytes(kind));
      if (ctx->roots[r].second < bytes) {
        cudaFree(ctx->roots[r].first);
        cuda_check(cudaMalloc(&ctx->roots[r].first, bytes), "cudaMalloc(root)");
        ctx->roots[r].second = bytes;
      }
      ptrs[r] = ctx->roots[r].first;
      dev[r] = sb_device_buffer{b.name.c_str(), hb.flags, 0, ptrs[r], b.elements};
      if ((hb.flags & SB_BUF_PREPARE) && b.dir != sb::Dir::In) continue;
      const void* src = hb.data;
      if (hb.carrier == SB_CARRIER_I64) {
        if (ctx->pinned[r].second < bytes) {
          cudaFreeHost(ctx->pinned[r].first);
          cuda_check(cudaMallocHost(&ctx->pinned[r].first, bytes), "cudaMallocHost");
          ctx->pinned[r].second = bytes;
        }
        void* st = ctx->pinned[r].first;
        narrow_from_i64(static_cast<const std::int64_t*>(hb.data), st, kind, b.elements);
        src = st;
      }
      cuda_check(cudaMemcpyAsync(ptrs[r], src, b.elements * kind_bytes(kind), cudaMemcpyHostToDevice, ctx->stream),
                 "H2D");
    }
    {
      // reuse the device path for prepare-fills + plan execution; an ordered context's
      // kernels wait for the previous ordered kernel phase on this device (two contexts
      // ping-ponging steps then overlap copies with kernels without running two steps'
      // kernels at once, which would split L2 between their activations)
      std::unique_lock<std::mutex> order;
      if (ctx->ordered) {
        KernelOrder& ko = g_kernel_order[ctx->device & 63];
        order = std::unique_lock<std::mutex>(ko.mu);
        if (ko.last) cuda_check(cudaStreamWaitEvent(ctx->stream, ko.last, 0), "cudaStreamWaitEvent(order)");
      }
      int rc = sb_execute_device(ctx, p, dev.data(), static_cast<int>(nr), opts);
      if (rc != SB_OK) throw sb::Error(sb_status_name(rc), g_last_error);
      if (ctx->ordered) {
        cuda_check(cudaEventRecord(ctx->kernels_done, ctx->stream), "cudaEventRecord(order)");
        g_kernel_order[ctx->device & 63].last = ctx->kernels_done;
      }
    }
    for (std::size_t r = 0; r < nr; r++) {
      const auto& b = prog.buffers[r];
      if (b.dir == sb::Dir::In) continue;
      sb_host_buffer& hb = bufs[slot[r]];
      int kind = c->plan.bufs[r].kind;
      void* dst = hb.data;
      if (hb.carrier == SB_CARRIER_I64) {
        std::size_t bytes = padded(b.elements * kind_bytes(kind));
        if (ctx->pinned[r].second < bytes) {
          cudaFreeHost(ctx->pinned[r].first);
          cuda_check(cudaMallocHost(&ctx->pinned[r].first, bytes), "cudaMallocHost");
          ctx->pinned[r].second = bytes;
        }
        dst = ctx->pinned[r].first;
      }
      cuda_check(cudaMemcpyAsync(dst, ptrs[r], b.elements * kind_bytes(kind), cudaMemcpyDeviceToHost, ctx->stream),
                 "D2H");
    }
    if (async) return;  // errors surface at sb_context_sync
    ctx->h_err->code = 1;
    check_device_error(ctx, c);
    for (std::size_t r = 0; r < nr; r++) {
      const auto& b = prog.buffers[r];
      if (b.dir == sb::Dir::In) continue;
      sb_host_buffer& hb = bufs[slot[r]];
      if (hb.carrier != SB_CARRIER_I64) continue;
      int kind = c->plan.bufs[r].kind;
      widen_to_i64(ctx->pinned[r].first, static_cast<std::int64_t*>(hb.data), kind, b.elements);
    }
  });
}
}  // namespace

extern "C" {

int sb_execute(sb_context* ctx, sb_program* p, sb_host_buffer* bufs, int n, const sb_exec_options* opts) {
  return execute_host(ctx, p, bufs, n, opts, false);
}

int sb_execute_async(sb_context* ctx, sb_program* p, sb_host_buffer* bufs, int n, const sb_exec_options* opts) {
  return execute_host(ctx, p, bufs, n, opts, true);
}

}  // extern "C"

// ---- CUDA graphs -----------------------------------------------------------------
struct sb_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::uint64_t kernels = 0;  // library kernels per launch of this graph
  ~sb_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

namespace {
thread_local std::uint64_t g_capture_mark = 0;
}

extern "C" {

int sb_graph_begin(sb_context* ctx) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    g_capture_mark = ctx->launches;
    ctx->window.clear();
    cuda_check(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  });
}

int sb_graph_end(sb_context* ctx, sb_graph** out) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    ctx->window.clear();
    auto g = std::make_unique<sb_graph>();
    cuda_check(cudaStreamEndCapture(ctx->stream, &g->graph), "cudaStreamEndCapture");
    cuda_check(cudaGraphInstantiate(&g->exec, g->graph, 0), "cudaGraphInstantiate");
    g->kernels = ctx->launches - g_capture_mark;
    ctx->launches = g_capture_mark;  // captured, not launched
    *out = g.release();
  });
}

int sb_graph_launch(sb_context* ctx, sb_graph* g) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lock(ctx->mu);
    cuda_check(cudaGraphLaunch(g->exec, ctx->stream), "cudaGraphLaunch");
    ctx->launches += g->kernels;
  });
}

void sb_graph_free(sb_graph* g) { delete g; }

}  // extern "C"
