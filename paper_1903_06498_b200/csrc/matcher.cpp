// Kernel matcher: routes launches whose leaf body is a dense contraction of the
// convolution family to the tcgen05 implicit-GEMM kernel (kernels/conv_tc.cu).
// Everything else stays on the generic block kernel.
//
// Recognised body (the reference's conv leaf, tests/support.cpp:79-124):
//   $a = load(A); $b = load(B); $p = mul($a, $b) | mul($b, $a); C = store($p)  with C:add
// Index roles are read off the composed affine accesses:
//   k  (N)   : in B and C only                      -> output channel
//   c  (K)   : in A and B, coefficient 1 in A       -> input channel
//   i, j     : in A and B, same A coefficient as x/y -> filter taps
//   n, x, y  : in A and C only                      -> batch and spatial output dims
// Constraints must be exactly interval bounds on u = x + i and v = y + j: the
// kernel realises them as TMA out-of-bounds zero fill, which reproduces the
// skip-predicate semantics (interp.cpp:426-428) for a multiply-accumulate.
#include <algorithm>
#include <cstdlib>
#include <limits>

#include "kernels.hpp"
#include "plan.hpp"

namespace sb {
namespace {

bool match_conv(const Plan& plan, const PLaunch& l, const Program& prog, const PlanOptions& opt, std::size_t step,
                ConvPlan* cp, std::string* why) {
  if (l.mode != kModeOwner || !l.priv.empty() || l.has_spill || !l.specials.empty() || !l.consts.empty()) return false;
  if (l.code.size() != 4) return false;
  const DInstr& la = l.code[0];
  const DInstr& lb = l.code[1];
  const DInstr& mu = l.code[2];
  const DInstr& st = l.code[3];
  if (la.op != kOpLoad || lb.op != kOpLoad || mu.op != kOpMul || st.op != kOpStore) return false;
  bool order_ok = (mu.a == la.dst && mu.b == lb.dst) || (mu.a == lb.dst && mu.b == la.dst);
  if (!order_ok || st.a != mu.dst || la.dst == lb.dst) return false;
  if (st.agg != static_cast<std::int8_t>(Agg::Add)) return false;
  const PAccess* A = &l.acc[la.acc];
  const PAccess* B = &l.acc[lb.acc];
  const PAccess& C = l.acc[st.acc];
  if (A->buf == C.buf || B->buf == C.buf) return false;
  if (plan.bufs[A->buf].dtype != DType::I8 || plan.bufs[B->buf].dtype != DType::I8) return false;
  if (plan.bufs[A->buf].kind != kI8 || plan.bufs[B->buf].kind != kI8) return false;
  DType cdt = static_cast<DType>(st.dtype);
  if (cdt == DType::F32 || plan.bufs[C.buf].dtype != cdt) return false;

  const int nd = static_cast<int>(l.dims.size());
  auto roles = [&](const PAccess* a, const PAccess* b, int* kdim, int* cdim, std::vector<int>* mdims,
                   std::vector<int>* taps) {
    for (int d = 0; d < nd; d++) {
      bool ia = a->addr.uses(d), ib = b->addr.uses(d), ic = C.addr.uses(d);
      if (!ia && ib && ic) {
        if (*kdim >= 0) return false;
        *kdim = d;
      } else if (ia && ib && !ic) {
        taps->push_back(d);
      } else if (ia && !ib && ic) {
        mdims->push_back(d);
      } else {
        return false;
      }
    }
    return true;
  };
  int kdim = -1, cdim = -1;
  std::vector<int> mdims, taps;
  if (!roles(A, B, &kdim, &cdim, &mdims, &taps)) {
    // maybe the loads are in the other order (filter first)
    std::swap(A, B);
    kdim = -1;
    mdims.clear();
    taps.clear();
    if (!roles(A, B, &kdim, &cdim, &mdims, &taps)) return false;
  }
  if (kdim < 0 || mdims.empty() || mdims.size() > 3) return false;
  // input channel: the tap-role dim with A coefficient 1
  for (std::size_t t = 0; t < taps.size(); t++)
    if (A->addr.at(taps[t]) == 1) {
      cdim = taps[t];
      taps.erase(taps.begin() + static_cast<long>(t));
      break;
    }
  if (cdim < 0 || taps.size() > 2) return false;
  // spatial dims: the M dims ordered by A coefficient (y smallest, then x, then n)
  std::sort(mdims.begin(), mdims.end(), [&](int a, int b) { return A->addr.at(a) < A->addr.at(b); });
  int ydim = mdims[0];
  int xdim = mdims.size() > 1 ? mdims[1] : -1;
  int ndim = mdims.size() > 2 ? mdims[2] : -1;
  // taps: the smaller A coefficient pairs with y (j), the other with x (i); a spatial
  // coefficient that is s times its tap's is a stride-s conv (s in [1, 8])
  int idim = -1, jdim = -1;
  std::sort(taps.begin(), taps.end(), [&](int a, int b) { return A->addr.at(a) < A->addr.at(b); });
  auto stride_of = [&](int sp, int tp) -> std::int64_t {
    if (sp < 0 || tp < 0) return 0;
    std::int64_t a = A->addr.at(sp), t = A->addr.at(tp);
    if (t <= 0 || a % t != 0 || a / t < 1 || a / t > 8) return 0;
    return a / t;
  };
  if (taps.size() == 2) {
    jdim = taps[0];
    idim = taps[1];
    if (!stride_of(ydim, jdim) || !stride_of(xdim, idim)) return false;
  } else if (taps.size() == 1) {
    if (stride_of(ydim, taps[0])) jdim = taps[0];
    else if (stride_of(xdim, taps[0])) idim = taps[0];
    else return false;
  }
  // with a single M dim that has a tap but no batch: fine; taps must pair
  auto coef = [&](const PAccess* a, int d) -> std::int64_t { return d < 0 ? 0 : a->addr.at(d); };
  auto range = [&](int d) -> std::int64_t { return d < 0 ? 1 : l.dims[d].range; };
  for (int d = 0; d < nd; d++)
    if (A->addr.at(d) < 0 || B->addr.at(d) < 0 || C.addr.at(d) < 0) return false;
  if (C.addr.at(kdim) != 1) return false;

  ConvPlan c;
  c.a_buf = A->buf;
  c.b_buf = B->buf;
  c.c_buf = C.buf;
  c.c_dtype = cdt;
  c.N = range(ndim);
  c.H = range(xdim);
  c.W = range(ydim);
  c.C = range(cdim);
  c.K = range(kdim);
  c.R = range(idim);
  c.S = range(jdim);
  c.sx = idim >= 0 ? stride_of(xdim, idim) : 1;
  c.sy = jdim >= 0 ? stride_of(ydim, jdim) : 1;
  c.a_n = coef(A, ndim);
  c.a_x = idim >= 0 ? coef(A, idim) : coef(A, xdim);  // one input row
  c.a_y = jdim >= 0 ? coef(A, jdim) : coef(A, ydim);  // one input pixel
  c.a0 = A->addr.c;
  if (c.a_n == 0) c.a_n = std::max<std::int64_t>(16, (c.a_x ? c.a_x : c.a_y) * 1024);  // unused (N == 1)
  if (c.a_x == 0) c.a_x = std::max<std::int64_t>(16, c.a_y * c.W * 4);                // unused (H == 1)
  c.b_i = coef(B, idim);
  c.b_j = coef(B, jdim);
  c.b_k = coef(B, kdim);
  c.b_c = coef(B, cdim);
  c.b0 = B->addr.c;
  c.c_n = coef(&C, ndim);
  c.c_x = coef(&C, xdim);
  c.c_y = coef(&C, ydim);
  c.c0 = C.addr.c;
  // valid input window: u = sx*x + i in [u_lo, u_hi], v = sy*y + j in [v_lo, v_hi]
  c.u_lo = 0;
  c.u_hi = c.sx * (c.H - 1) + c.R - 1;
  c.v_lo = 0;
  c.v_hi = c.sy * (c.W - 1) + c.S - 1;
  for (const auto& con : l.cons) {
    int used = 0;
    for (int d = 0; d < nd; d++) used += con.uses(d) ? 1 : 0;
    // unit coefficient of u (resp. v) in the constraint: the tap's, or the spatial one
    std::int64_t cx = xdim < 0 ? 0 : con.at(xdim), ci = idim < 0 ? 0 : con.at(idim);
    std::int64_t cy = con.at(ydim), cj = jdim < 0 ? 0 : con.at(jdim);
    std::int64_t au = idim >= 0 ? ci : cx, av = jdim >= 0 ? cj : cy;
    bool on_u = xdim >= 0 && cx != 0 && (au == 1 || au == -1) && cx == c.sx * au &&
                used == (idim >= 0 ? 2 : 1) && (idim < 0 || ci != 0);
    bool on_v = cy != 0 && (av == 1 || av == -1) && cy == c.sy * av && used == (jdim >= 0 ? 2 : 1) &&
                (jdim < 0 || cj != 0);
    if (on_u) {
      // au*u + c >= 0
      if (au == 1) c.u_lo = std::max(c.u_lo, -con.c);
      else c.u_hi = std::min(c.u_hi, con.c);
    } else if (on_v) {
      if (av == 1) c.v_lo = std::max(c.v_lo, -con.c);
      else c.v_hi = std::min(c.v_hi, con.c);
    } else {
      *why = "constraint is not an interval on an input coordinate";
      return false;
    }
  }
  if (c.u_lo > c.u_hi || c.v_lo > c.v_hi) return false;  // empty: leave to the generic kernel
  // every address the kernel touches must lie inside its buffer (else the
  // reference would raise OutOfBoundsAccess; the generic kernel reports it)
  std::int64_t a_min = c.a0 + c.a_x * c.u_lo + c.a_y * c.v_lo;
  std::int64_t a_max = c.a0 + c.a_n * (c.N - 1) + c.a_x * c.u_hi + c.a_y * c.v_hi + (c.C - 1);
  if (a_min < 0 || a_max >= plan.bufs[c.a_buf].elements) return false;
  std::int64_t b_max = c.b0 + c.b_i * (c.R - 1) + c.b_j * (c.S - 1) + c.b_k * (c.K - 1) + c.b_c * (c.C - 1);
  if (c.b0 < 0 || b_max >= plan.bufs[c.b_buf].elements) return false;
  std::int64_t o_max = c.c0 + c.c_n * (c.N - 1) + c.c_x * (c.H - 1) + c.c_y * (c.W - 1) + (c.K - 1);
  if (c.c0 < 0 || o_max >= plan.bufs[c.c_buf].elements) return false;
  // exactness of the s32 accumulation
  if (c.R * c.S * c.C * 128 * 128 >= (std::int64_t{1} << 31)) {
    *why = "reduction too long for exact s32 accumulation";
    return false;
  }
  // fused prepare_outputs: the first writer of a fresh root output that covers
  // it exactly once may overwrite instead of accumulate into the identity (0).
  const PBuffer& cb = plan.bufs[c.c_buf];
  if (cb.root && cb.root_index < static_cast<int>(opt.fresh_outputs.size()) && opt.fresh_outputs[cb.root_index] &&
      output_identity(prog, cb.name) == 0) {
    bool first = true;
    for (std::size_t s = 0; s < step; s++) {
      const PStep& ps = plan.steps[s];
      if (ps.kind != PStep::Launch) continue;
      for (const auto& ins : ps.launch.code)
        if ((ins.op == kOpStore && ps.launch.acc[ins.acc].buf == c.c_buf)) first = false;
      for (const auto& sp : ps.launch.specials)
        if (ps.launch.acc[sp.dst].buf == c.c_buf) first = false;
    }
    bool dense = c.c0 == 0 && c.c_y == c.K && (c.H == 1 || c.c_x == c.W * c.K) &&
                 (c.N == 1 || c.c_n == c.H * c.W * c.K) && c.N * c.H * c.W * c.K == cb.elements;
    c.fresh_output = first && dense;
  }
  {
    const PBuffer& bb = plan.bufs[c.b_buf];
    bool written = false;
    for (const auto& ps : plan.steps) {
      if (ps.kind == PStep::Fill) written |= ps.buf == c.b_buf;
      if (ps.kind != PStep::Launch) continue;
      for (const auto& ins : ps.launch.code)
        if (ins.op == kOpStore && ps.launch.acc[ins.acc].buf == c.b_buf) written = true;
      for (const auto& sp : ps.launch.specials)
        if (ps.launch.acc[sp.dst].buf == c.b_buf) written = true;
    }
    c.b_immutable = bb.root && bb.dir == Dir::In && !written;
  }
  *cp = c;
  return true;
}

// True when no step before `step` writes plan buffer `buf`.
bool first_writer(const Plan& plan, std::size_t step, int buf) {
  for (std::size_t s = 0; s < step; s++) {
    const PStep& ps = plan.steps[s];
    if (ps.kind == PStep::Fill) {
      if (ps.buf == buf) return false;
      continue;
    }
    for (const auto& ins : ps.launch.code)
      if (ins.op == kOpStore && ps.launch.acc[ins.acc].buf == buf) return false;
    for (const auto& sp : ps.launch.specials)
      if (ps.launch.acc[sp.dst].buf == buf) return false;
  }
  return true;
}

// The address function maps the given dims one-to-one onto [0, elements).
bool covers_exactly(const FAff& a, const std::vector<int>& dims, const std::vector<PDim>& rng, std::int64_t elements) {
  if (a.c != 0) return false;
  std::vector<std::pair<std::int64_t, std::int64_t>> t;
  std::int64_t count = 1, span = 0;
  for (int d : dims) {
    std::int64_t k = a.at(d);
    if (k <= 0) return false;
    t.emplace_back(k, rng[d].range);
    count *= rng[d].range;
    span += k * (rng[d].range - 1);
  }
  std::sort(t.begin(), t.end());
  std::int64_t run = 0;
  for (auto& [k, r] : t) {
    if (k <= run) return false;
    run += k * (r - 1);
  }
  return count == elements && span == elements - 1;
}

// $v = load(I); O = store($v) with no constraints: streaming reduce/copy (kernels/reduce.cu).
bool match_reduce(const Plan& plan, PLaunch& l, const Program& prog, const PlanOptions& opt, std::size_t step) {
  if (l.mode != kModeOwner || l.pdims.empty() || !l.cons.empty() || !l.priv.empty() || l.has_spill ||
      !l.specials.empty() || l.code.size() != 2)
    return false;
  const DInstr& ld = l.code[0];
  const DInstr& st = l.code[1];
  if (ld.op != kOpLoad || st.op != kOpStore || st.a != ld.dst || ld.acc == st.acc) return false;
  if (l.acc_mode[ld.acc] != kAccRead || l.acc_mode[st.acc] != kAccOwned) return false;
  const PAccess& A = l.acc[ld.acc];
  const PAccess& O = l.acc[st.acc];
  const PBuffer& ib = plan.bufs[A.buf];
  const PBuffer& ob = plan.bufs[O.buf];
  auto intk = [](std::int8_t k) { return k == kI8 || k == kI16 || k == kI32; };
  if (!intk(ib.kind) || !intk(ob.kind) || st.dtype != static_cast<std::int8_t>(ob.dtype)) return false;
  const int V = reduce_vec_lanes(ib.kind);
  const int obytes = ob.kind == kI8 ? 1 : ob.kind == kI16 ? 2 : 4;
  if (V * obytes < 16) return false;
  const int v = l.pdims[0];
  if (A.addr.at(v) != 1 || O.addr.at(v) != 1 || l.dims[v].range % V != 0) return false;
  if (A.addr.c % V != 0 || O.addr.c % V != 0) return false;
  for (std::size_t d = 0; d < l.dims.size(); d++) {
    if (static_cast<int>(d) == v) continue;
    if (A.addr.at(d) % V != 0 || O.addr.at(d) % V != 0) return false;
  }
  ReducePlan r;
  r.in_buf = A.buf;
  r.out_buf = O.buf;
  r.in_kind = ib.kind;
  r.out_kind = ob.kind;
  r.agg = st.agg;
  r.np = static_cast<int>(l.pdims.size());
  for (int i = 0; i < r.np; i++) {
    int d = l.pdims[i];
    r.prange[i] = l.dims[d].range;
    r.pin[i] = A.addr.at(d);
    r.pout[i] = O.addr.at(d);
  }
  r.nr = static_cast<int>(l.rdims.size());
  std::int64_t rc = 1;
  for (int i = 0; i < r.nr; i++) {
    int d = l.rdims[i];
    r.rrange[i] = l.dims[d].range;
    r.rstep[i] = A.addr.at(d);
    rc *= r.rrange[i];
  }
  if (rc > 6144) return false;
  r.rcount = static_cast<int>(rc);
  r.in_c = A.addr.c;
  r.out_c = O.addr.c;
  r.pcount = l.pcount;
  // bounds: the whole box must be inside both buffers (affine extremes)
  auto extremes = [&](const FAff& a, std::int64_t* lo, std::int64_t* hi) {
    *lo = *hi = a.c;
    for (std::size_t d = 0; d < l.dims.size(); d++) {
      std::int64_t k = a.at(d) * (l.dims[d].range - 1);
      (k < 0 ? *lo : *hi) += k;
    }
  };
  std::int64_t lo, hi;
  extremes(A.addr, &lo, &hi);
  if (lo < 0 || hi >= ib.elements) return false;
  extremes(O.addr, &lo, &hi);
  if (lo < 0 || hi >= ob.elements) return false;
  if (ob.root && ob.root_index < static_cast<int>(opt.fresh_outputs.size()) && opt.fresh_outputs[ob.root_index] &&
      first_writer(plan, step, O.buf) && covers_exactly(O.addr, l.pdims, l.dims, ob.elements)) {
    r.fresh = true;
    r.identity = output_identity(prog, ob.name);
    l.fused_fill_root = ob.root_index;
  }
  l.reduce = r;
  return true;
}

// Vectorised owner-mode launch (kernels/map.cu): the fastest thread dim becomes kVec
// lanes; every access is broadcast (coefficient 0), an aligned contiguous vector
// (coefficient 1, everything else a multiple of kVec) or a per-lane gather.  Written
// buffers must be aligned contiguous vectors so each thread owns whole vectors.
// $v = load(I); O = store($v), O:max|min: output dims (n, x, y, c) and taps (i, j) with
// u = sx*x + i, v = sy*y + j bounded by interval constraints (the stem max-pool,
// support.cpp:126-155 with padding).
bool match_pool(const Plan& plan, PLaunch& l) {
  if (l.mode != kModeOwner || l.pdims.empty() || !l.priv.empty() || l.has_spill || !l.specials.empty() ||
      l.code.size() != 2 || l.is_float)
    return false;
  const DInstr& ld = l.code[0];
  const DInstr& st = l.code[1];
  if (ld.op != kOpLoad || st.op != kOpStore || st.a != ld.dst || ld.acc == st.acc) return false;
  if (st.agg != static_cast<std::int8_t>(Agg::Max) && st.agg != static_cast<std::int8_t>(Agg::Min)) return false;
  if (l.acc_mode[ld.acc] != kAccRead || l.acc_mode[st.acc] != kAccOwned) return false;
  const PAccess& I = l.acc[ld.acc];
  const PAccess& O = l.acc[st.acc];
  const PBuffer& ib = plan.bufs[I.buf];
  const PBuffer& ob = plan.bufs[O.buf];
  if (ib.kind != ob.kind || (ib.kind != kI8 && ib.kind != kI16 && ib.kind != kI32) ||
      st.dtype != static_cast<std::int8_t>(ob.dtype))
    return false;
  const int nd = static_cast<int>(l.dims.size());
  int cdim = -1;
  std::vector<int> out, taps;
  for (int d = 0; d < nd; d++) {
    const bool ui = I.addr.uses(d), uo = O.addr.uses(d);
    if (ui && uo) {
      if (I.addr.at(d) == 1 && O.addr.at(d) == 1 && cdim < 0) cdim = d;
      else out.push_back(d);
    } else if (ui) {
      taps.push_back(d);
    } else {
      return false;
    }
    if (I.addr.at(d) < 0 || O.addr.at(d) < 0) return false;
  }
  if (cdim < 0 || out.empty() || out.size() > 3 || taps.size() > 2) return false;
  std::sort(out.begin(), out.end(), [&](int a, int b) { return I.addr.at(a) < I.addr.at(b); });
  std::sort(taps.begin(), taps.end(), [&](int a, int b) { return I.addr.at(a) < I.addr.at(b); });
  const int ydim = out[0], xdim = out.size() > 1 ? out[1] : -1, ndim = out.size() > 2 ? out[2] : -1;
  auto stride_of = [&](int sp, int tp) -> std::int64_t {
    if (sp < 0 || tp < 0) return 0;
    std::int64_t a = I.addr.at(sp), t = I.addr.at(tp);
    if (t <= 0 || a % t != 0 || a / t < 1 || a / t > 64) return 0;
    return a / t;
  };
  int idim = -1, jdim = -1;
  if (taps.size() == 2) {
    jdim = taps[0];
    idim = taps[1];
    if (!stride_of(ydim, jdim) || !stride_of(xdim, idim)) return false;
  } else if (taps.size() == 1) {
    if (stride_of(ydim, taps[0])) jdim = taps[0];
    else if (stride_of(xdim, taps[0])) idim = taps[0];
    else return false;
  }
  auto range = [&](int d) -> std::int64_t { return d < 0 ? 1 : l.dims[d].range; };
  PoolPlan pp;
  pp.in_buf = I.buf;
  pp.out_buf = O.buf;
  pp.kind = ib.kind;
  pp.agg = st.agg;
  pp.N = range(ndim);
  pp.H = range(xdim);
  pp.W = range(ydim);
  pp.C = range(cdim);
  pp.R = range(idim);
  pp.S = range(jdim);
  pp.sx = idim >= 0 ? stride_of(xdim, idim) : 1;
  pp.sy = jdim >= 0 ? stride_of(ydim, jdim) : 1;
  pp.a_n = ndim >= 0 ? I.addr.at(ndim) : 0;
  pp.a_x = idim >= 0 ? I.addr.at(idim) : (xdim >= 0 ? I.addr.at(xdim) : 0);
  pp.a_y = jdim >= 0 ? I.addr.at(jdim) : I.addr.at(ydim);
  pp.a0 = I.addr.c;
  pp.o_n = ndim >= 0 ? O.addr.at(ndim) : 0;
  pp.o_x = xdim >= 0 ? O.addr.at(xdim) : 0;
  pp.o_y = O.addr.at(ydim);
  pp.o0 = O.addr.c;
  pp.u_lo = 0;
  pp.u_hi = pp.sx * (pp.H - 1) + pp.R - 1;
  pp.v_lo = 0;
  pp.v_hi = pp.sy * (pp.W - 1) + pp.S - 1;
  for (const auto& con : l.cons) {
    int used = 0;
    for (int d = 0; d < nd; d++) used += con.uses(d) ? 1 : 0;
    std::int64_t cx = xdim < 0 ? 0 : con.at(xdim), ci = idim < 0 ? 0 : con.at(idim);
    std::int64_t cy = con.at(ydim), cj = jdim < 0 ? 0 : con.at(jdim);
    std::int64_t au = idim >= 0 ? ci : cx, av = jdim >= 0 ? cj : cy;
    bool on_u = xdim >= 0 && cx != 0 && (au == 1 || au == -1) && cx == pp.sx * au && used == (idim >= 0 ? 2 : 1) &&
                (idim < 0 || ci != 0);
    bool on_v = cy != 0 && (av == 1 || av == -1) && cy == pp.sy * av && used == (jdim >= 0 ? 2 : 1) &&
                (jdim < 0 || cj != 0);
    if (on_u) {
      if (au == 1) pp.u_lo = std::max(pp.u_lo, -con.c);
      else pp.u_hi = std::min(pp.u_hi, con.c);
    } else if (on_v) {
      if (av == 1) pp.v_lo = std::max(pp.v_lo, -con.c);
      else pp.v_hi = std::min(pp.v_hi, con.c);
    } else {
      return false;
    }
  }
  // every address the kernel may touch lies inside the buffers
  const std::int64_t ulo = std::max<std::int64_t>(pp.u_lo, 0), vlo = std::max<std::int64_t>(pp.v_lo, 0);
  const std::int64_t uhi = std::min(pp.u_hi, pp.sx * (pp.H - 1) + pp.R - 1);
  const std::int64_t vhi = std::min(pp.v_hi, pp.sy * (pp.W - 1) + pp.S - 1);
  if (ulo > uhi || vlo > vhi) return false;
  if (pp.a0 + pp.a_x * ulo + pp.a_y * vlo < 0 ||
      pp.a0 + pp.a_n * (pp.N - 1) + pp.a_x * uhi + pp.a_y * vhi + pp.C - 1 >= ib.elements)
    return false;
  if (pp.o0 < 0 || pp.o0 + pp.o_n * (pp.N - 1) + pp.o_x * (pp.H - 1) + pp.o_y * (pp.W - 1) + pp.C - 1 >= ob.elements)
    return false;
  if (pool_unsupported(pp)) return false;
  l.pool = pp;
  return true;
}

bool match_map(PLaunch& l) {
  if (l.is_float || l.mode != kModeOwner || l.pdims.empty() || !l.specials.empty()) return false;
  if (l.ntemps > kVecMaxTemps || l.ncells > kVecMaxCells || l.priv.size() > static_cast<std::size_t>(kVecMaxCells))
    return false;
  const int v = l.pdims[0];
  const std::int64_t rv = l.dims[v].range;
  if (rv < kVec || l.pcount < 4096) return false;
  std::vector<std::int8_t> kind(l.acc.size(), 2);
  for (std::size_t i = 0; i < l.acc.size(); i++) {
    const FAff& a = l.acc[i].addr;
    std::int64_t k = a.at(v);
    if (k == 0) {
      kind[i] = 0;
    } else if (k == 1) {
      bool aligned = a.c % kVec == 0;
      for (std::size_t d = 0; d < l.dims.size(); d++)
        if (static_cast<int>(d) != v && a.at(d) % kVec != 0) aligned = false;
      kind[i] = aligned ? 1 : 2;
    }
    if (l.acc_mode[i] != kAccRead && kind[i] != 1) return false;
  }
  l.vdim = v;
  l.vkind = kind;
  l.vcount = l.pcount / rv * ((rv + kVec - 1) / kVec);
  return true;
}

// Plain matmul leaf (gen_matmul, support.cpp:50-77): exactly one m, n and k dim,
// no constraints, A k-contiguous, B n- or k-contiguous, C n-contiguous.
bool match_gemm(const Plan& plan, PLaunch& l, const Program& prog, const PlanOptions& opt, std::size_t step) {
  if (l.mode != kModeOwner || !l.priv.empty() || l.has_spill || !l.specials.empty() || !l.consts.empty() ||
      !l.cons.empty() || l.code.size() != 4)
    return false;
  const DInstr &la = l.code[0], &lb = l.code[1], &mu = l.code[2], &st = l.code[3];
  if (la.op != kOpLoad || lb.op != kOpLoad || mu.op != kOpMul || st.op != kOpStore) return false;
  if (!((mu.a == la.dst && mu.b == lb.dst) || (mu.a == lb.dst && mu.b == la.dst)) || st.a != mu.dst) return false;
  if (st.agg != static_cast<std::int8_t>(Agg::Add)) return false;
  const PAccess* A = &l.acc[la.acc];
  const PAccess* B = &l.acc[lb.acc];
  const PAccess& C = l.acc[st.acc];
  auto intk = [](int k) { return k == kI8 || k == kI16 || k == kI32; };
  const bool f32 = l.is_float;
  if (A->buf == C.buf || B->buf == C.buf) return false;
  if (f32 ? (plan.bufs[A->buf].kind != kF32 || plan.bufs[B->buf].kind != kF32 || plan.bufs[C.buf].kind != kF32)
          : (!intk(plan.bufs[A->buf].kind) || !intk(plan.bufs[B->buf].kind)))
    return false;
  DType cdt = static_cast<DType>(st.dtype);
  if ((cdt == DType::F32) != f32 || plan.bufs[C.buf].dtype != cdt) return false;
  if (l.dims.size() != 3) return false;
  auto roles = [&](const PAccess* a, const PAccess* b, int* m, int* n, int* k) {
    *m = *n = *k = -1;
    for (int d = 0; d < 3; d++) {
      bool ia = a->addr.uses(d), ib = b->addr.uses(d), ic = C.addr.uses(d);
      if (ia && !ib && ic) *m = d;
      else if (!ia && ib && ic) *n = d;
      else if (ia && ib && !ic) *k = d;
    }
    return *m >= 0 && *n >= 0 && *k >= 0 && a->addr.at(*k) == 1;
  };
  int m, n, k;
  if (!roles(A, B, &m, &n, &k)) {
    std::swap(A, B);
    if (!roles(A, B, &m, &n, &k)) return false;
  }
  GemmPlan g;
  g.M = l.dims[m].range;
  g.N = l.dims[n].range;
  g.K = l.dims[k].range;
  g.lda = A->addr.at(m);
  g.a0 = A->addr.c;
  if (B->addr.at(n) == 1) {
    g.b_kmajor = false;
    g.ldb = B->addr.at(k);
  } else if (B->addr.at(k) == 1) {
    g.b_kmajor = true;
    g.ldb = B->addr.at(n);
  } else {
    return false;
  }
  g.b0 = B->addr.c;
  if (C.addr.at(n) != 1) return false;
  g.ldc = C.addr.at(m);
  g.c0 = C.addr.c;
  g.c_dtype = cdt;
  g.a_buf = A->buf;
  g.b_buf = B->buf;
  g.c_buf = C.buf;
  g.f32 = f32;
  if (!f32) {
    const int ka = plan.bufs[A->buf].kind, kb = plan.bufs[B->buf].kind;
    if (ka != kI8 || kb != kI8) {
      // exact modulo 2^(8 * bytes(C)) on u8 tensor cores: each operand, sign-extended to the
      // output width, is sum_i limb_i 256^i with unsigned byte limbs (narrower inputs included)
      const int ob = cdt == DType::I8 ? 1 : cdt == DType::I16 ? 2 : 4;
      g.limbs_a = ob;
      g.limbs_b = ob;
      g.a_kind = ka;
      g.b_kind = kb;
    }
  }
  if (g.lda <= 0 || g.ldb <= 0 || g.ldc < g.N || g.a0 < 0 || g.b0 < 0 || g.c0 < 0) return false;
  if (g.a0 + g.lda * (g.M - 1) + g.K - 1 >= plan.bufs[A->buf].elements) return false;
  long long bmax = g.b_kmajor ? g.b0 + g.ldb * (g.N - 1) + g.K - 1 : g.b0 + g.ldb * (g.K - 1) + g.N - 1;
  if (bmax >= plan.bufs[B->buf].elements) return false;
  if (g.c0 + g.ldc * (g.M - 1) + g.N - 1 >= plan.bufs[C.buf].elements) return false;
  if (!f32 && gemm_tc_unsupported(g)) return false;
  const PBuffer& cb = plan.bufs[C.buf];
  std::vector<int> pd = {m, n};
  if (cb.root && cb.root_index < static_cast<int>(opt.fresh_outputs.size()) && opt.fresh_outputs[cb.root_index] &&
      output_identity(prog, cb.name) == 0 && first_writer(plan, step, C.buf) &&
      covers_exactly(C.addr, pd, l.dims, cb.elements)) {
    g.fresh = true;
    l.fused_fill_root = cb.root_index;
  }
  l.gemm = g;
  return true;
}

// K3e: a conv launch writing a per-point local accumulator T (scratch, zero-filled) whose
// only consumer is the next phase  O = f(T, vec[k])  with f in the bias/ReLU family
// (conv_relu.stripe after fuse+localize, test_passes.cpp:357-379): the epilogue applies f
// on the s32 accumulator and writes O directly; T never reaches HBM.
bool fuse_conv_epilogue(Plan* plan, std::size_t s, const Program& prog, const PlanOptions& opt) {
  PLaunch& cl = plan->steps[s].launch;
  ConvPlan& c = cl.conv;
  const int T = c.c_buf;
  if (plan->bufs[T].root || c.fresh_output) return false;
  // T is touched only by: one zero Fill before s, the conv, and the consumer s2 after s
  int fill_step = -1, s2 = -1;
  for (std::size_t k = 0; k < plan->steps.size(); k++) {
    if (k == s) continue;
    const PStep& ps = plan->steps[k];
    bool touches = false;
    if (ps.kind == PStep::Fill) {
      if (ps.buf == T) {
        if (k > s || ps.value != 0 || fill_step >= 0) return false;
        fill_step = static_cast<int>(k);
      }
      continue;
    }
    for (const auto& a : ps.launch.acc) touches |= a.buf == T;
    if (!touches) continue;
    if (k < s || s2 >= 0) return false;
    s2 = static_cast<int>(k);
  }
  if (fill_step < 0 || s2 < 0) return false;
  for (std::size_t k = s + 1; k < static_cast<std::size_t>(s2); k++)  // nothing in between
    if (!plan->steps[k].elided) return false;
  PLaunch& el = plan->steps[s2].launch;
  if (el.mode != kModeOwner || !el.cons.empty() || !el.priv.empty() || el.has_spill || !el.specials.empty()) return false;
  // T must be dense [n][x][y][k] for the conv and read back at the same element
  const std::int64_t K = c.K, HW = c.H * c.W, NHW = c.N * HW;
  if (!(c.c0 == 0 && c.c_y == K && (c.H == 1 || c.c_x == c.W * K) && (c.N == 1 || c.c_n == HW * K))) return false;
  if (el.dims.size() != 2) return false;
  // channel dim: unit coefficient in the consumer's read of T (ranges alone are ambiguous
  // when the pixel count equals K)
  int pd = -1, kd = -1;
  for (const auto& a : el.acc)
    if (a.buf == T)
      for (int d = 0; d < 2; d++)
        if (a.addr.at(d) == 1) kd = d;
  if (kd < 0) return false;
  pd = 1 - kd;
  if (el.dims[kd].range != K || el.dims[pd].range != NHW) return false;
  // symbolic evaluation of the body: each temp is ACC, VEC (per-k vector), RES (per-element
  // residual), CONST or an op on them
  struct Sym {
    int kind = -1;  // 0 ACC, 1 VEC, 2 CONST, 3 ADD(a,b), 4 MAX(a,b), 5 RES
    int a = -1, b = -1;
    std::int64_t c = 0;
  };
  std::vector<Sym> nodes;
  std::vector<int> temp(el.ntemps, -1);
  int vec_acc = -1, res_acc = -1, out_acc = -1, out_node = -1;
  DInstr store_ins{};
  auto operand = [&](int x) -> int {
    if (x >= 0) return temp[x];
    Sym s;
    s.kind = 2;
    s.c = el.consts[-1 - x];
    nodes.push_back(s);
    return static_cast<int>(nodes.size()) - 1;
  };
  for (const auto& ins : el.code) {
    Sym s;
    if (ins.op == kOpLoad) {
      const PAccess& a = el.acc[ins.acc];
      if (a.buf == T) {
        if (!(a.addr.c == 0 && a.addr.at(pd) == K && a.addr.at(kd) == 1)) return false;
        s.kind = 0;
      } else if (a.addr.at(pd) == 0) {
        if (el.acc_mode[ins.acc] != kAccRead) return false;
        if (vec_acc >= 0 && !(el.acc[vec_acc].buf == a.buf && el.acc[vec_acc].addr == a.addr)) return false;
        vec_acc = ins.acc;
        s.kind = 1;
      } else {
        // residual: pixel-major i8 with contiguous channels
        if (el.acc_mode[ins.acc] != kAccRead || res_acc >= 0 || a.addr.at(kd) != 1 || a.addr.at(pd) <= 0 ||
            plan->bufs[a.buf].kind != kI8 || a.addr.c < 0 ||
            a.addr.c + a.addr.at(pd) * (NHW - 1) + K - 1 >= plan->bufs[a.buf].elements)
          return false;
        res_acc = ins.acc;
        s.kind = 5;
      }
    } else if (ins.op == kOpConst) {
      int o = operand(ins.a);
      if (o < 0) return false;
      temp[ins.dst] = o;
      continue;
    } else if (ins.op == kOpAdd || ins.op == kOpMax) {
      s.kind = ins.op == kOpAdd ? 3 : 4;
      s.a = operand(ins.a);
      s.b = operand(ins.b);
      if (s.a < 0 || s.b < 0) return false;
    } else if (ins.op == kOpStore) {
      if (out_acc >= 0) return false;
      out_acc = ins.acc;
      store_ins = ins;
      out_node = temp[ins.a];
      if (out_node < 0) return false;
      // the resident-filter kernel's TMA-store epilogue writes i32; the im2col one any width
      if (static_cast<DType>(ins.dtype) != DType::I32 && cl.kernel != KernelKind::ConvIgemmTC &&
          !(static_cast<DType>(ins.dtype) == DType::I8 && c.K % 64 == 0 && std::getenv("SB_TC_I8_EPI")))
        return false;
      if (ins.agg != static_cast<std::int8_t>(Agg::Assign) && ins.agg != static_cast<std::int8_t>(Agg::Add)) return false;
      continue;
    } else {
      return false;
    }
    nodes.push_back(s);
    temp[ins.dst] = static_cast<int>(nodes.size()) - 1;
  }
  if (out_acc < 0) return false;
  // match out = MAX(x, CONST) | x ;  x = a sum (int64, order-free) of ACC, optional VEC, optional RES
  ConvPlan e = c;
  int n = out_node;
  e.epi_lo = false;
  if (nodes[n].kind == 4) {
    int a = nodes[n].a, b = nodes[n].b;
    if (nodes[b].kind != 2) std::swap(a, b);
    if (nodes[b].kind != 2) return false;
    e.epi_lo = true;
    e.lo = nodes[b].c;
    n = a;
  }
  int n_acc = 0, n_vec = 0, n_res = 0;
  {
    std::vector<int> work = {n};
    while (!work.empty()) {
      int x = work.back();
      work.pop_back();
      switch (nodes[x].kind) {
        case 3: work.push_back(nodes[x].a); work.push_back(nodes[x].b); break;
        case 0: n_acc++; break;
        case 1: n_vec++; break;
        case 5: n_res++; break;
        default: return false;
      }
    }
  }
  if (n_acc != 1 || n_vec > 1 || n_res > 1) return false;
  e.epi_vec = n_vec == 1;
  if (e.epi_vec) {
    const PAccess& va = el.acc[vec_acc];
    e.vec_buf = va.buf;
    e.vec_c = va.addr.c;
    e.vec_k = va.addr.at(kd);
    if (plan->bufs[va.buf].kind != kI32 && plan->bufs[va.buf].kind != kI16 && plan->bufs[va.buf].kind != kI8) return false;
    if (e.vec_c < 0 || e.vec_k < 0 || e.vec_c + e.vec_k * (K - 1) >= plan->bufs[va.buf].elements) return false;
  }
  e.epi_res = n_res == 1;
  if (e.epi_res) {
    const PAccess& ra = el.acc[res_acc];
    e.res_buf = ra.buf;
    e.res_c0 = ra.addr.c;
    e.res_pix = ra.addr.at(pd);
  }
  // output O: address = o_pix * pix + k + o_c over the consumer's dims
  const PAccess& O = el.acc[out_acc];
  const PBuffer& ob = plan->bufs[O.buf];
  if (O.addr.at(kd) != 1 || O.addr.at(pd) <= 0) return false;
  if (ob.kind != kI32 && !(cl.kernel == KernelKind::ConvIgemmTC && (ob.kind == kI8 || ob.kind == kI16)) &&
      // opt-in: the resident-filter kernel's i8 epilogue is faster alone, but inside chains of
      // im2col convs (ResNet) the im2col kernel's shorter prologue overlaps better (measured)
      !(cl.kernel == KernelKind::ConvI8TC && ob.kind == kI8 && K % 64 == 0 && std::getenv("SB_TC_I8_EPI")))
    return false;
  if (static_cast<std::int8_t>(ob.dtype) != store_ins.dtype) return false;
  const std::int64_t op = O.addr.at(pd);
  if (O.addr.c < 0 || O.addr.c + op * (NHW - 1) + K - 1 >= ob.elements) return false;
  bool overwrite = store_ins.agg == static_cast<std::int8_t>(Agg::Assign);
  const bool fresh_root = ob.root && ob.root_index < static_cast<int>(opt.fresh_outputs.size()) &&
                          opt.fresh_outputs[ob.root_index] && output_identity(prog, ob.name) == 0 &&
                          first_writer(*plan, static_cast<std::size_t>(s2), O.buf);
  const bool covers = O.addr.c == 0 && op == K && NHW * K == ob.elements;
  if (!overwrite && !(fresh_root && covers)) return false;
  e.epi = e.epi_vec || e.epi_lo;
  e.c_buf = O.buf;
  e.c_dtype = ob.dtype;
  e.c_y = op;
  e.c_x = op * c.W;
  e.c_n = op * HW;
  e.c0 = O.addr.c;
  e.fresh_output = true;  // the consumer overwrites (assign) or adds onto the fused identity 0
  e.overwrites = overwrite;
  if (cl.kernel == KernelKind::ConvIgemmTC
          ? conv_igemm_unsupported(e) != nullptr
          : conv_tc_unsupported(e) != nullptr)
    return false;
  c = e;
  plan->steps[fill_step].elided = true;
  plan->steps[s2].elided = true;
  if (fresh_root && covers) cl.fused_fill_root = ob.root_index;
  plan->notes.push_back("launch " + cl.path + ": epilogue of " + el.path + " fused; local buffer " + plan->bufs[T].name +
                        " never materialised");
  return true;
}

}  // namespace

ConvPlan packed_view(const ConvPlan& c) {
  ConvPlan v = c;
  v.packed = false;
  v.a_buf = c.pack_a;
  v.b_buf = c.pack_b;
  if (c.fold_x && c.fold_band) {
    // band view: the GEMM geometry of the banded filter [fold_r + band - 1][band * K][fold_cv]
    // over compact folded rows (prepare() in conv_igemm.cu reads the band fields)
    v.C = c.fold_cv;
    v.R = c.fold_r + c.fold_band - 1;
    v.S = 1;
    v.K = c.fold_band * c.K;
    v.sx = v.sy = 1;
    v.a_y = c.fold_c;
    v.a_x = c.fold_v * c.fold_c;
    v.a_n = c.fold_u * v.a_x;
    v.a0 = 0;
    v.u_lo = 0;
    v.u_hi = c.fold_u - 1;
    v.v_lo = 0;
    v.v_hi = c.fold_v - 1;
    v.b_i = v.K * c.fold_cv;
    v.b_j = 0;
    v.b_k = c.fold_cv;
    v.b_c = 1;
    v.b0 = 0;
    v.b_immutable = false;
    v.fold_x = v.fold_y = 0;
    return v;
  }
  if (c.fold_x) {
    // out[x, y] = sum_{a, q} F[x + a, y + q / fold_c, q % fold_c] * G[a, k, q]: "pixel" (U, y)
    // of the view is the fold_cv bytes starting at folded pixel (U, y), so consecutive view
    // pixels overlap (pixel stride fold_c < fold_cv; TMA im2col reads them as rows)
    v.C = c.fold_cv;
    v.R = c.fold_r;
    v.S = 1;
    v.sx = v.sy = 1;
    v.a_y = c.fold_rows ? c.fold_cv : c.fold_c;
    v.a_x = c.fold_rows ? c.W * c.fold_cv : c.fold_v * c.fold_c;
    v.a_n = c.fold_u * v.a_x;
    v.a0 = 0;
    v.u_lo = 0;
    v.u_hi = c.fold_u - 1;
    v.v_lo = 0;
    v.v_hi = c.W - 1;
    v.b_i = c.K * c.fold_cv;
    v.b_j = 0;
    v.b_k = c.fold_cv;
    v.b_c = 1;
    v.b0 = 0;
    v.b_immutable = false;
    v.fold_x = v.fold_y = 0;
    return v;
  }
  v.C = c.pack_k;
  v.R = v.S = 1;
  v.sx = v.sy = 1;
  v.a_y = c.pack_k;
  v.a_x = c.W * c.pack_k;
  v.a_n = c.H * c.W * c.pack_k;
  v.a0 = 0;
  v.u_lo = 0;
  v.u_hi = c.H - 1;
  v.v_lo = 0;
  v.v_hi = c.W - 1;
  v.b_i = v.b_j = 0;
  v.b_k = c.pack_k;
  v.b_c = 1;
  v.b0 = 0;
  v.b_immutable = false;
  return v;
}

namespace {

// Band tiles for a phase-folded conv (ConvPlan::fold_band), decided once the output and the
// fused epilogue are known: one output row fits one 128-row tile, two rows stack to N <= 256,
// and the output is a fresh dense NHWC i8 activation (4-D clipped TMA store).  The fold buffer
// becomes the compact folded pixels (+ a tail for the junk rows' reads), the packed filter the
// banded [fold_r + 1][2K][fold_cv].
void choose_band(Plan* plan, ConvPlan* cp) {
  const ConvPlan& c = *cp;
  if (!c.packed || !c.fold_x || std::getenv("SB_NO_BAND")) return;
  const bool ok = c.fold_c == 16 && c.fold_cv == 64 && c.W <= 128 && c.H % 2 == 0 && (c.K == 64 || c.K == 128) &&
                  c.c_dtype == DType::I8 && c.fresh_output && !c.epi_res && c.c_y == c.K && c.c_x == c.W * c.K &&
                  (c.N == 1 || c.c_n == c.H * c.c_x) && c.c0 % 16 == 0;
  if (!ok) return;
  ConvPlan b = c;
  b.fold_band = 2;
  b.fold_rows = false;
  b.pack_k = (b.fold_r + b.fold_band - 1) * b.fold_cv * b.fold_band;
  // opt-in (SB_BAND_RAW=1): the fold moves into the conv's producer warps when the raw rows are
  // 16-byte aligned runs of 3-byte pixels (one cp.async chunk per 16 bytes of a row).  Bit-exact,
  // but measured slower (stem 568 vs 441 us at b1024 including the separate fold): the copies and
  // the in-shared-memory transform contend with the N = 128 MMAs for shared-memory bandwidth
  // (knocking either out recovers ~130-150 us), while the separate fold runs at HBM speed.
  const std::int64_t row_bytes = (c.v_hi - c.v_lo + 1) * c.a_y;
  b.band_raw = c.fold_x == 2 && c.fold_y == 2 && c.C == 3 && c.a_y == 3 && c.a_x % 16 == 0 && c.a_n % 16 == 0 &&
               ((c.a0 + c.a_x * c.u_lo + c.a_y * c.v_lo) % 16 + 16) % 16 == 0 && row_bytes % 16 == 0 &&
               row_bytes <= 128 * 16 && c.v_lo >= 0 && c.v_lo <= 64 && c.u_lo >= 0 && c.fold_v <= 128 &&
               std::getenv("SB_BAND_RAW") != nullptr;
  if (b.band_raw) {
    b.raw_a_n = c.a_n;
    b.raw_a_x = c.a_x;
    b.raw_a0 = c.a0;
    b.raw_u_lo = c.u_lo;
    b.raw_u_hi = c.u_hi;
    b.raw_v_lo = c.v_lo;
    b.raw_v_hi = c.v_hi;
  }
  if (conv_igemm_unsupported(b)) return;
  *cp = b;
  plan->bufs[b.pack_a].elements = b.band_raw ? 16 : b.N * b.fold_u * b.fold_v * b.fold_c + 128 * 16 + 64;
  plan->bufs[b.pack_b].elements = b.K * b.pack_k;
}

// Small-channel convs (C not a multiple of 64, e.g. the 7x7x3 stem): pack, then 1x1 igemm.
bool try_packed_conv(Plan* plan, ConvPlan* cp) {
  const std::int64_t rsc = cp->R * cp->S * cp->C;
  // 1x1 contractions with few channels are plain GEMMs (gemm_tc takes ragged K directly)
  if (rsc > 1024 || cp->C % 64 == 0 || cp->R * cp->S == 1) return false;
  // Preferred: phase fold (a stride-1 conv over a folded copy of the input, A tiles by TMA
  // im2col); the in-kernel gather below is the fallback.
  if (!std::getenv("SB_NO_FOLD")) {
    ConvPlan c = *cp;
    c.packed = true;
    c.fold_x = c.sx;
    c.fold_y = c.sy;
    c.fold_c = (c.sx * c.sy * c.C + 15) / 16 * 16;
    c.fold_r = (c.R + c.sx - 1) / c.sx;
    c.fold_s = (c.S + c.sy - 1) / c.sy;
    c.fold_cv = (c.fold_s * c.fold_c + 63) / 64 * 64;
    c.fold_u = c.H + c.fold_r - 1;
    c.fold_v = c.W + (c.fold_cv + c.fold_c - 1) / c.fold_c - 1;
    c.pack_k = c.fold_r * c.fold_cv;
    c.pack_a = static_cast<int>(plan->bufs.size());
    c.pack_b = c.pack_a + 1;
    // materialised rows when a folded pixel is one 16-byte unit and a row a whole number of them
    // (choose_band() may switch to band tiles once the output and epilogue are known)
    c.fold_rows = c.fold_c == 16 && c.fold_cv % 16 == 0 && !std::getenv("SB_FOLD_OVERLAP");
    const std::int64_t folded = c.fold_rows ? c.N * c.fold_u * c.W * c.fold_cv : c.N * c.fold_u * c.fold_v * c.fold_c;
    if (c.pack_k <= 1024 && folded < (1ll << 34) && !conv_igemm_unsupported(c)) {
      PBuffer f;
      f.name = "fold:" + plan->bufs[c.a_buf].name;
      f.dtype = DType::I8;
      f.kind = kI8;
      f.elements = folded;
      plan->bufs.push_back(f);
      PBuffer b;
      b.name = "pack:" + plan->bufs[c.b_buf].name;
      b.dtype = DType::I8;
      b.kind = kI8;
      b.elements = c.K * c.pack_k;
      plan->bufs.push_back(b);
      *cp = c;
      return true;
    }
  }
  ConvPlan c = *cp;
  c.packed = true;
  // run layout when each tap row's S*C bytes are contiguous in the input (dense pixels)
  const std::int64_t sc = c.S * c.C;
  c.pack_run = (c.a_y == c.C && sc <= 64) ? (sc <= 16 ? 16 : sc <= 32 ? 32 : 64) : 0;
  const std::int64_t kp = c.pack_run ? (c.R * c.pack_run + 63) / 64 * 64 : (rsc + 63) / 64 * 64;
  c.pack_k = kp;
  const std::int64_t pixels = c.N * c.H * c.W;
  c.pack_a = -1;  // A rows are gathered in the kernel (no packed copy in HBM)
  c.pack_b = static_cast<int>(plan->bufs.size());
  if (conv_igemm_unsupported(c)) return false;
  (void)pixels;
  PBuffer b;
  b.name = "pack:" + plan->bufs[c.b_buf].name;
  b.dtype = DType::I8;
  b.kind = kI8;
  b.elements = c.K * kp;
  plan->bufs.push_back(b);
  *cp = c;
  return true;
}

// The conv writes every element of its output exactly once (pixel-major, dense).
bool conv_covers(const ConvPlan& c, std::int64_t elements) {
  return c.c0 == 0 && c.c_y == c.K && (c.H == 1 || c.c_x == c.W * c.K) && (c.N == 1 || c.c_n == c.H * c.W * c.K) &&
         c.N * c.H * c.W * c.K == elements;
}

// A conv accumulating (add) into a local whose only earlier touch is its zero fill
// (interp.cpp:433-447: locals start at zero) may overwrite instead; the fill goes.
void fresh_scratch_output(Plan* plan, std::size_t s) {
  PLaunch& l = plan->steps[s].launch;
  ConvPlan& c = l.conv;
  const PBuffer& ob = plan->bufs[c.c_buf];
  if (ob.root || c.fresh_output || !conv_covers(c, ob.elements)) return;
  int fill = -1;
  for (std::size_t k = 0; k < s; k++) {
    const PStep& ps = plan->steps[k];
    if (ps.elided) continue;
    if (ps.kind == PStep::Fill) {
      if (ps.buf == c.c_buf) {
        if (ps.value != 0) return;
        fill = static_cast<int>(k);
      }
      continue;
    }
    for (const auto& a : ps.launch.acc)
      if (a.buf == c.c_buf) return;
  }
  if (fill < 0) return;
  c.fresh_output = true;
  plan->steps[fill].elided = true;
}

// Zero fills of locals that the next step touching them overwrites completely before
// reading (a fused conv epilogue with assign, or an owner-mode assign over every element).
void elide_dead_fills(Plan* plan) {
  for (std::size_t f = 0; f < plan->steps.size(); f++) {
    PStep& fs = plan->steps[f];
    if (fs.kind != PStep::Fill || fs.elided || plan->bufs[fs.buf].root) continue;
    const int B = fs.buf;
    const std::int64_t elems = plan->bufs[B].elements;
    for (std::size_t k = f + 1; k < plan->steps.size(); k++) {
      const PStep& ps = plan->steps[k];
      if (ps.elided) continue;
      if (ps.kind == PStep::Fill) {
        if (ps.buf == B) break;
        continue;
      }
      const PLaunch& l = ps.launch;
      bool conv = l.kernel == KernelKind::ConvI8TC || l.kernel == KernelKind::ConvIgemmTC;
      bool touches = conv && (l.conv.c_buf == B || l.conv.a_buf == B || l.conv.b_buf == B ||
                              (l.conv.packed && (l.conv.pack_a == B || l.conv.pack_b == B)) ||
                              (l.conv.epi_vec && l.conv.vec_buf == B) || (l.conv.epi_res && l.conv.res_buf == B));
      for (const auto& a : l.acc) touches |= a.buf == B;
      if (!touches) continue;
      bool dead = false;
      if (conv) {
        dead = l.conv.c_buf == B && l.conv.a_buf != B && l.conv.b_buf != B && l.conv.fresh_output &&
               l.conv.overwrites && conv_covers(l.conv, elems);
      } else if ((l.kernel == KernelKind::Generic || l.kernel == KernelKind::Map) && l.mode == kModeOwner &&
                 l.cons.empty() && l.specials.empty()) {
        dead = true;
        int acc = -1;
        for (const auto& ins : l.code) {
          if (ins.op == kOpLoad && l.acc[ins.acc].buf == B) dead = false;
          if (ins.op == kOpStore && l.acc[ins.acc].buf == B) {
            if (ins.agg != static_cast<std::int8_t>(Agg::Assign) || acc >= 0) dead = false;
            acc = ins.acc;
          }
        }
        dead = dead && acc >= 0 && covers_exactly(l.acc[acc].addr, l.pdims, l.dims, elems) && l.rdims.empty();
      }
      if (dead) fs.elided = true;
      break;
    }
  }
}

// A pool whose output is a local touched only by an earlier fill: the pool writes every
// element exactly once, so it can start from the fill value and the fill goes.
void fresh_pool_output(Plan* plan, std::size_t s) {
  PoolPlan& pp = plan->steps[s].launch.pool;
  const PBuffer& ob = plan->bufs[pp.out_buf];
  if (ob.root || pp.out_buf == pp.in_buf) return;
  const bool covers = pp.o0 == 0 && pp.o_y == pp.C && (pp.H == 1 || pp.o_x == pp.W * pp.C) &&
                      (pp.N == 1 || pp.o_n == pp.H * pp.W * pp.C) && pp.N * pp.H * pp.W * pp.C == ob.elements;
  if (!covers) return;
  int fill = -1;
  for (std::size_t k = 0; k < s; k++) {
    const PStep& ps = plan->steps[k];
    if (ps.elided) continue;
    if (ps.kind == PStep::Fill) {
      if (ps.buf == pp.out_buf) fill = static_cast<int>(k);
      continue;
    }
    std::vector<int> rd, wr;
    step_access(ps, &rd, &wr);
    for (int b : rd) if (b == pp.out_buf) return;
    for (int b : wr) if (b == pp.out_buf) return;
  }
  if (fill < 0) return;
  pp.fresh = true;
  pp.fill_value = plan->steps[fill].value;
  plan->steps[fill].elided = true;
}

}  // namespace

void match_kernels(Plan* plan, const Program& p, const PlanOptions& opt) {
  if (!opt.enable_tc) return;
  for (std::size_t s = 0; s < plan->steps.size(); s++) {
    PStep& st = plan->steps[s];
    if (st.kind != PStep::Launch || st.elided) continue;
    ConvPlan cp;
    std::string why;
    if (match_conv(*plan, st.launch, p, opt, s, &cp, &why)) {
      const char* bad_tc = conv_tc_unsupported(cp);
      const char* bad_ig = bad_tc ? conv_igemm_unsupported(cp) : nullptr;
      if (!bad_tc || !bad_ig) {
        st.launch.kernel = bad_tc ? KernelKind::ConvIgemmTC : KernelKind::ConvI8TC;
        st.launch.conv = cp;
        if (cp.fresh_output) st.launch.fused_fill_root = plan->bufs[cp.c_buf].root_index;
        bool fused = fuse_conv_epilogue(plan, s, p, opt);
        if (!fused && !bad_tc && !bad_ig) {
          // the im2col kernel stores any output width: it may take an epilogue the
          // resident-filter kernel (i32 TMA-store only) cannot
          plan->steps[s].launch.kernel = KernelKind::ConvIgemmTC;
          fused = fuse_conv_epilogue(plan, s, p, opt);
          if (!fused) plan->steps[s].launch.kernel = KernelKind::ConvI8TC;
        }
        if (!fused && cp.R * cp.S == 1 && cp.H == 1 && cp.N == 1) {
          // a plain matmul with nothing to fuse: the tiled GEMM kernel
          PLaunch trial = plan->steps[s].launch;
          trial.fused_fill_root = -1;
          if (match_gemm(*plan, trial, p, opt, s)) {
            trial.kernel = KernelKind::GemmI8TC;
            if (!trial.gemm.limbs_a) {
              plan->steps[s].launch = trial;
              continue;
            }
          }
        }
        if (!fused) fresh_scratch_output(plan, s);
        continue;
      }
      if (try_packed_conv(plan, &cp)) {
        st.launch.kernel = KernelKind::ConvIgemmTC;
        st.launch.conv = cp;
        if (cp.fresh_output) st.launch.fused_fill_root = plan->bufs[cp.c_buf].root_index;
        if (!fuse_conv_epilogue(plan, s, p, opt)) fresh_scratch_output(plan, s);
        choose_band(plan, &st.launch.conv);
        cp = st.launch.conv;
        if (cp.fold_x)
          plan->notes.push_back("launch " + st.launch.path + ": small-channel conv phase-folded (" +
                                std::to_string(cp.fold_x) + "x" + std::to_string(cp.fold_y) + ", " +
                                std::to_string(cp.fold_c) + " bytes per folded pixel), packed to " +
                                std::to_string(cp.fold_r) + " tap rows x " + std::to_string(cp.fold_cv) +
                                (cp.fold_band ? ", band tiles of " + std::to_string(cp.fold_band) +
                                                    " output rows stacked along N (overlapping-row descriptors)" +
                                                    (cp.band_raw ? std::string(", folded in the producer warps from the raw rows")
                                                                 : std::string())
                                              : std::string()));
        else
          plan->notes.push_back("launch " + st.launch.path + ": small-channel conv packed to " +
                                std::to_string(cp.pack_k) + " taps x channels per pixel (gathered)");
        continue;
      }
      why = std::string(bad_tc) + "; " + bad_ig;
    }
    if (match_gemm(*plan, st.launch, p, opt, s)) {
      st.launch.kernel = st.launch.gemm.f32 ? KernelKind::GemmF32 : KernelKind::GemmI8TC;
      GemmPlan& g = st.launch.gemm;
      if (g.f32 && opt.fp32_tc) {
        GemmPlan t = g;
        t.tf32x3 = true;
        if (!gemm_tc_unsupported(tf32_sum_plan(t, 0)) && !gemm_tc_unsupported(tf32_sum_plan(t, 2))) {
          g.tf32x3 = true;
          auto scratch = [&](const std::string& name, long long elems) {
            PBuffer b;
            b.name = name;
            b.dtype = DType::F32;
            b.kind = kF32;
            b.elements = elems;
            plan->bufs.push_back(b);
            return static_cast<int>(plan->bufs.size()) - 1;
          };
          g.planes_a = scratch("tf32x3:" + plan->bufs[g.a_buf].name, g.M * 3 * g.K);
          g.planes_b = scratch("tf32x3:" + plan->bufs[g.b_buf].name, g.N * 3 * g.K);
          g.sums = scratch("tf32x3sums:" + plan->bufs[g.c_buf].name, 3 * g.M * g.N);
          plan->notes.push_back("launch " + st.launch.path + ": fp32 matmul as one 3xTF32 tensor-core GEMM (k x 3)");
        }
      }
      if (g.limbs_a) {
        auto scratch = [&](const std::string& name, std::int8_t kind, long long elems) {
          PBuffer b;
          b.name = name;
          b.dtype = kind == kI8 ? DType::I8 : DType::I32;
          b.kind = kind;
          b.elements = elems;
          plan->bufs.push_back(b);
          return static_cast<int>(plan->bufs.size()) - 1;
        };
        g.limb_fused = !std::getenv("SB_LIMB_UNFUSED");
        if (g.limb_fused) {
          g.planes_a = scratch("limbs:" + plan->bufs[g.a_buf].name, kI8, g.limbs_a * g.M * limb_fused_kp(g));
          g.planes_b = scratch("limbs:" + plan->bufs[g.b_buf].name, kI8, g.limbs_b * g.N * limb_fused_kp(g));
          plan->notes.push_back("launch " + st.launch.path + ": matmul exact modulo 2^" + std::to_string(g.limbs_a * 8) +
                                " over byte limbs: " + std::to_string(limb_smax(g) + 1) +
                                " u8 sums in TMEM of one tensor-core kernel, combined in its epilogue");
        } else {
          g.planes_a = scratch("limbs:" + plan->bufs[g.a_buf].name, kI8, limb_plane_bytes_a(g));
          g.planes_b = scratch("limbs:" + plan->bufs[g.b_buf].name, kI8, limb_plane_bytes_b(g));
          g.sums = scratch("limbsums:" + plan->bufs[g.c_buf].name, kI32, (limb_smax(g) + 1) * g.M * g.N);
          plan->notes.push_back("launch " + st.launch.path + ": matmul exact modulo 2^" + std::to_string(g.limbs_a * 8) +
                                " as " + std::to_string(limb_smax(g) + 1) + " u8 tensor-core GEMMs over byte limbs");
        }
      }
      continue;
    }
    if (!why.empty())
      plan->notes.push_back("launch " + st.launch.path + ": contraction kept on the generic kernel (" + why + ")");
    if (match_reduce(*plan, st.launch, p, opt, s)) st.launch.kernel = KernelKind::Reduce;
    else if (match_pool(*plan, st.launch)) {
      st.launch.kernel = KernelKind::Pool;
      fresh_pool_output(plan, s);
    }
    else if (match_map(st.launch)) st.launch.kernel = KernelKind::Map;
  }
  elide_dead_fills(plan);
}

}  // namespace sb
