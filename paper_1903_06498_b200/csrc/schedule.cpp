// Statement-DAG concurrency (the reference's build_dependency_dag,
// analysis.cpp:331-371, and schedule pass, passes.cpp:563-666, order statements on the
// CPU).  Plan steps run in program order on one stream by default; here every step's read
// and write sets (plan buffers) give the true dependencies, and independent steps are
// placed on up to `max_lanes` CUDA streams (lanes) by a list scheduler over estimated step
// times.  A step waits only for the latest conflicting step on each other lane (events);
// same-lane order needs nothing.  Under CUDA-graph capture the lanes become parallel graph
// branches.  Programs whose steps form a chain keep one lane (no events at all), and so do
// steps that saturate the GPU alone.
#include <algorithm>
#include <cmath>
#include <functional>
#include <set>

#include "plan.hpp"

namespace sb {

void step_access(const PStep& s, std::vector<int>* reads, std::vector<int>* writes) {
  reads->clear();
  writes->clear();
  auto R = [&](int b) {
    if (b >= 0) reads->push_back(b);
  };
  auto W = [&](int b) {
    if (b >= 0) writes->push_back(b);
  };
  if (s.kind == PStep::Fill) {
    W(s.buf);
    return;
  }
  const PLaunch& l = s.launch;
  switch (l.kernel) {
    case KernelKind::ConvI8TC:
    case KernelKind::ConvIgemmTC:
      R(l.conv.a_buf);
      R(l.conv.b_buf);
      if (l.conv.epi_vec) R(l.conv.vec_buf);
      if (l.conv.epi_res) R(l.conv.res_buf);
      if (!l.conv.fresh_output) R(l.conv.c_buf);
      W(l.conv.c_buf);
      if (l.conv.packed) {
        W(l.conv.pack_a);
        W(l.conv.pack_b);
      }
      return;
    case KernelKind::GemmI8TC:
    case KernelKind::GemmF32:
      R(l.gemm.a_buf);
      R(l.gemm.b_buf);
      if (!l.gemm.fresh) R(l.gemm.c_buf);
      W(l.gemm.c_buf);
      W(l.gemm.planes_a);
      W(l.gemm.planes_b);
      W(l.gemm.sums);
      return;
    case KernelKind::Reduce:
      R(l.reduce.in_buf);
      if (!l.reduce.fresh) R(l.reduce.out_buf);
      W(l.reduce.out_buf);
      return;
    case KernelKind::Pool:
      R(l.pool.in_buf);
      if (!l.pool.fresh) R(l.pool.out_buf);
      W(l.pool.out_buf);
      return;
    default:
      for (const auto& ins : l.code) {
        if (ins.op == kOpLoad) R(l.acc[ins.acc].buf);
        if (ins.op == kOpStore) {
          R(l.acc[ins.acc].buf);  // aggregation reads the current value
          W(l.acc[ins.acc].buf);
        }
      }
      for (const auto& sp : l.specials) {
        R(l.acc[sp.src].buf);
        R(l.acc[sp.idx].buf);
        R(l.acc[sp.dst].buf);
        W(l.acc[sp.dst].buf);
      }
      return;
  }
}

namespace {

// Rough device time of a step (µs): enough to order independent work sensibly.
double step_cost(const Plan& plan, const PStep& s) {
  if (s.kind == PStep::Fill) {
    const PBuffer& b = plan.bufs[s.buf];
    const int es = b.kind == kI8 ? 1 : b.kind == kI16 ? 2 : b.kind == kI64 ? 8 : 4;
    return 2.0 + static_cast<double>(b.elements) * es / 5e6;
  }
  const PLaunch& l = s.launch;
  switch (l.kernel) {
    case KernelKind::ConvI8TC:
    case KernelKind::ConvIgemmTC:
    case KernelKind::GemmI8TC:
      return 3.0 + static_cast<double>(l.points) / 1.5e9;
    case KernelKind::GemmF32:
      return 3.0 + static_cast<double>(l.points) / 1e7;
    default:
      return 3.0 + static_cast<double>(l.points) / 1e5;
  }
}

}  // namespace

LaneSchedule schedule_lanes(const Plan& plan, int max_lanes, const std::function<bool(int, int)>& alias) {
  auto intersects = [&](const std::vector<int>& a, const std::vector<int>& b) {
    for (int x : a)
      for (int y : b)
        if (x == y || alias(x, y)) return true;
    return false;
  };
  const int n = static_cast<int>(plan.steps.size());
  LaneSchedule ls;
  ls.lane.assign(n, 0);
  ls.waits.assign(n, {});
  ls.signal.assign(n, 0);
  std::vector<std::vector<int>> rd(n), wr(n);
  for (int i = 0; i < n; i++)
    if (!plan.steps[i].elided) step_access(plan.steps[i], &rd[i], &wr[i]);
  std::vector<double> finish(n, 0.0), lane_free(std::max(1, max_lanes), 0.0);
  std::vector<int> lane_tail(lane_free.size(), -1);
  int used = 1;
  for (int j = 0; j < n; j++) {
    if (plan.steps[j].elided) continue;
    std::vector<int> deps;
    double ready = 0.0;
    for (int i = 0; i < j; i++) {
      if (plan.steps[i].elided) continue;
      if (intersects(wr[i], rd[j]) || intersects(wr[i], wr[j]) || intersects(rd[i], wr[j])) {
        deps.push_back(i);
        ready = std::max(ready, finish[i]);
      }
    }
    // earliest start over lanes; prefer the lane that holds the latest dependency.  A step
    // long enough to fill the GPU on its own (est. >= 8 us) gains nothing from a second lane
    // and would lose programmatic-dependent-launch chaining: it stays on its dependency's lane.
    int best = -1;
    double best_start = 0.0;
    const int last_dep = deps.empty() ? -1 : deps.back();
    const bool saturating = step_cost(plan, plan.steps[j]) >= 8.0;
    if (saturating) {
      best = last_dep >= 0 ? ls.lane[last_dep] : 0;
      best_start = std::max(lane_free[best], ready);
    }
    for (int L = 0; L < static_cast<int>(lane_free.size()) && !saturating; L++) {
      if (L >= used + 1) break;  // open at most one new lane at a time
      const double start = std::max(lane_free[L], ready);
      const bool pref = last_dep >= 0 && ls.lane[last_dep] == L;
      if (best < 0 || start < best_start - 1e-9 || (std::abs(start - best_start) <= 1e-9 && pref)) {
        best = L;
        best_start = start;
      }
    }
    ls.lane[j] = best;
    used = std::max(used, best + 1);
    finish[j] = best_start + step_cost(plan, plan.steps[j]);
    lane_free[best] = finish[j];
    // cross-lane waits: the latest dependency on each other lane
    std::vector<int> latest(lane_free.size(), -1);
    for (int i : deps)
      if (ls.lane[i] != best) latest[ls.lane[i]] = std::max(latest[ls.lane[i]], i);
    for (int i : latest)
      if (i >= 0) {
        ls.waits[j].push_back(i);
        ls.signal[i] = 1;
      }
    lane_tail[best] = j;
  }
  ls.nlanes = used;
  return ls;
}

}  // namespace sb
