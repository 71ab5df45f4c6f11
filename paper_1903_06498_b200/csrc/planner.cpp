// Planner: lowers a Stripe Program into flat device launches (see plan.hpp).
//
// Reference semantics being compiled (proj/src/interp.cpp):
//   index scoping / alias evaluation from the parent env   201-216, 362-364
//   constraint predicates                                  218-220, 426-428
//   refinement flat bases + parent/external/alloc views    221-250, 433-453
//   statement compile + error codes                        252-326
//   load/store at the view base, aggregation on store      497-504, ir.cpp:79-97
// Parallel execution is justified by the Stripe contract that iterations of a
// block are order-independent (Definition 2; checked dynamically by
// conflicts.cpp:57-167).  The planner never relies on it blindly: every launch
// is analysed (analyze()) and falls back to owner-computes or serial order
// whenever the access pattern alone cannot prove that threads are independent,
// so results stay bit-identical to lexicographic serial execution.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <sstream>

#include "plan.hpp"

namespace sb {

bool FAff::operator==(const FAff& o) const {
  if (c != o.c) return false;
  std::size_t n = std::max(k.size(), o.k.size());
  for (std::size_t d = 0; d < n; d++)
    if (at(d) != o.at(d)) return false;
  return true;
}

namespace {

struct View {
  int buf = -1;  // plan buffer (root or scratch); -1 for private cells
  FAff base;
  const Refinement* ref = nullptr;
  int priv = -1;  // private cell index (leaf-level alloc)
};

using Views = std::map<std::string, View>;

FAff& scaled_add(FAff& dst, const FAff& src, std::int64_t s) {
  if (dst.k.size() < src.k.size()) dst.k.resize(src.k.size(), 0);
  for (std::size_t d = 0; d < src.k.size(); d++) dst.k[d] += src.k[d] * s;
  dst.c += src.c * s;
  return dst;
}

int arity(const std::string& op) {
  if (op == "neg" || op == "constant") return 1;
  if (op == "select") return 3;
  return 2;
}

std::uint8_t opcode(const std::string& op) {
  static const std::map<std::string, std::uint8_t> m = {
      {"add", kOpAdd},       {"sub", kOpSub},       {"mul", kOpMul},       {"neg", kOpNeg},
      {"max", kOpMax},       {"min", kOpMin},       {"cmp_eq", kOpCmpEq},  {"cmp_ne", kOpCmpNe},
      {"cmp_lt", kOpCmpLt},  {"cmp_le", kOpCmpLe},  {"cmp_gt", kOpCmpGt},  {"cmp_ge", kOpCmpGe},
      {"select", kOpSelect}, {"constant", kOpConst}};
  auto it = m.find(op);
  if (it == m.end()) throw Error("UnknownIntrinsic", "unknown intrinsic '" + op + "'");
  return it->second;
}

std::int8_t storage_kind(DType d) {
  switch (d) {
    case DType::I8: return kI8;
    case DType::I16: return kI16;
    case DType::I32: return kI32;
    case DType::F32: return kF32;
  }
  return kI32;
}

// Is refinement `name` an operand of a gather/scatter special of block `b`?
bool special_operand(const Block& b, const std::string& name) {
  for (const auto& s : b.stmts)
    if (s.kind == StmtKind::Special)
      for (const auto& r : s.refs)
        if (r == name) return true;
  return false;
}

bool is_leaf(const Block& b) {
  for (const auto& s : b.stmts)
    if (s.kind == StmtKind::Block) return false;
  return true;
}

// Mixed-radix sufficient condition for injectivity of `a` over `dims`.
bool injective(const FAff& a, const std::vector<int>& dims, const std::vector<PDim>& ranges) {
  std::vector<std::pair<std::int64_t, std::int64_t>> t;
  for (int d : dims) {
    std::int64_t k = a.at(d);
    if (k == 0) return false;
    t.emplace_back(k < 0 ? -k : k, ranges[d].range);
  }
  std::sort(t.begin(), t.end());
  std::int64_t span = 0;
  for (auto& [k, r] : t) {
    if (k <= span) return false;
    span += k * (r - 1);
  }
  return true;
}

class Lowerer {
 public:
  Lowerer(const Program& p, const PlanOptions& opt, Plan* plan) : p_(p), opt_(opt), plan_(plan) {}

  void run() {
    for (std::size_t i = 0; i < p_.buffers.size(); i++) {
      const auto& d = p_.buffers[i];
      PBuffer b;
      b.name = d.name;
      b.dtype = d.dtype;
      b.kind = storage_kind(d.dtype);
      b.elements = d.elements;
      b.root = true;
      b.root_index = static_cast<int>(i);
      b.dir = d.dir;
      plan_->bufs.push_back(b);
    }
    Views none;
    lower_block(p_.root, none, "", true);
  }

 private:
  // ---- scopes / affine resolution -------------------------------------------------
  FAff resolve(const Affine& a) const {
    FAff out;
    out.c = a.constant;
    for (const auto& [name, coeff] : a.terms) {
      const FAff* found = nullptr;
      for (auto it = scopes_.rbegin(); it != scopes_.rend() && !found; ++it) {
        auto f = it->find(name);
        if (f != it->end()) found = &f->second;
      }
      if (!found) throw Error("UnboundIndex", "unbound index '" + name + "'");
      scaled_add(out, *found, coeff);
    }
    return out;
  }

  // Number of distinct points over the current (unpinned) dims, and the
  // row-major linearisation of them as an affine (for per-point scratch slices).
  std::int64_t point_count() const {
    std::int64_t n = 1;
    for (const auto& d : dims_)
      if (!d.pinned) n *= d.range;
    return n;
  }
  FAff linearize(std::int64_t scale) const {
    FAff f;
    f.k.assign(dims_.size(), 0);
    std::int64_t m = scale;
    for (std::size_t d = dims_.size(); d-- > 0;) {
      if (dims_[d].pinned) continue;  // serial (host-unrolled) points reuse one slice
      f.k[d] = m;
      m *= dims_[d].range;
    }
    return f;
  }

  int new_scratch(const std::string& name, DType dt, std::int8_t kind, std::int64_t elems) {
    PBuffer b;
    b.name = name;
    b.dtype = dt;
    b.kind = kind;
    b.elements = elems;
    plan_->bufs.push_back(b);
    return static_cast<int>(plan_->bufs.size()) - 1;
  }

  void fill(int buf, std::int64_t value) {
    PStep s;
    s.kind = PStep::Fill;
    s.buf = buf;
    s.value = value;
    plan_->steps.push_back(std::move(s));
  }

  // ---- block lowering ----------------------------------------------------------------
  void lower_block(const Block& b, const Views& parent, const std::string& path, bool is_root) {
    std::size_t dims_mark = dims_.size(), cons_mark = cons_.size();
    Scope own;
    for (const auto& idx : b.indexes) {
      if (idx.is_alias) {
        own[idx.name] = resolve(idx.alias);  // parent scopes only (interp.cpp:209-210)
      } else {
        PDim d;
        d.name = idx.name;
        d.range = idx.range;
        dims_.push_back(d);
        FAff f;
        f.k.assign(dims_.size(), 0);
        f.k.back() = 1;
        own[idx.name] = f;
      }
    }
    scopes_.push_back(std::move(own));
    for (const auto& c : b.constraints) cons_.push_back(resolve(c));

    bool leaf = is_leaf(b);
    const std::size_t private_mark = plan_->bufs.size();  // scratch created from here on is per-point private
    Views views;
    int npriv = 0;
    std::vector<std::pair<Agg, DType>> priv;
    for (const auto& r : b.refs) {
      View v;
      v.ref = &r;
      FAff flat;
      for (std::size_t d = 0; d < r.offsets.size(); d++) scaled_add(flat, resolve(r.offsets[d]), r.strides[d]);
      auto pit = parent.find(r.name);
      if (pit != parent.end()) {
        if (pit->second.priv >= 0)
          throw Error("Unsupported", "child view of a private allocation '" + r.name + "'");
        v.buf = pit->second.buf;
        v.base = pit->second.base;
        scaled_add(v.base, flat, 1);
      } else if (is_root) {
        v.buf = p_.buffer_index(r.name);
        v.base = flat;
      } else if (leaf && !special_operand(b, r.name)) {
        // Per-point allocation used only by this block's own statements: every
        // access is at the alloc base (element 0), so it is one register cell,
        // zeroed per point (interp.cpp:442-447).
        v.priv = npriv++;
        priv.emplace_back(r.has_agg ? r.agg : Agg::Assign, r.dtype);
      } else {
        // Per-iteration allocation visible to child blocks (or walked whole by a
        // gather/scatter special, interp.cpp:540-600): a scratch slice per point of this
        // block (and its ancestors), zero-filled before use.
        std::int64_t ext = r.extent();
        std::int64_t pts = point_count();
        v.buf = new_scratch("alloc:" + path + ":" + r.name, r.dtype, storage_kind(r.dtype), pts * ext);
        v.base = linearize(ext);
        fill(v.buf, 0);
      }
      views[r.name] = v;
    }

    if (!b.stmts.empty()) {
      if (leaf) {
        emit_leaf(b, b.stmts, 0, b.stmts.size(), views, priv, path, nullptr);
      } else if (b.stmts.size() == 1) {
        lower_block(*b.stmts[0].block, views, join(path, 0), false);
      } else {
        lower_segments(b, views, priv, path, private_mark);
      }
    }

    scopes_.pop_back();
    dims_.resize(dims_mark);
    cons_.resize(cons_mark);
  }

  static std::string join(const std::string& path, std::size_t i) {
    return path.empty() ? std::to_string(i) : path + "." + std::to_string(i);
  }

  struct SpillInfo {
    int buf = -1;
    std::int64_t slots = 0;
    FAff base;                          // per-point base (already scaled by slots)
    std::map<std::string, int> slot;    // temp -> slot
    std::set<std::string> live_in;      // for the current segment
    std::set<std::string> live_out;
  };

  // A block with several statements, at least one of them a child block: each
  // maximal run of scalar statements and each child block is one phase; phases
  // run as consecutive launches over this block's points.
  void lower_segments(const Block& b, const Views& views,
                      const std::vector<std::pair<Agg, DType>>& priv, const std::string& path,
                      std::size_t private_mark) {
    // segments: [begin, end) over b.stmts
    std::vector<std::pair<std::size_t, std::size_t>> segs;
    for (std::size_t i = 0; i < b.stmts.size();) {
      if (b.stmts[i].kind == StmtKind::Block) {
        segs.emplace_back(i, i + 1);
        i++;
      } else {
        std::size_t j = i;
        while (j < b.stmts.size() && b.stmts[j].kind != StmtKind::Block) j++;
        segs.emplace_back(i, j);
        i = j;
      }
    }
    // temp liveness across scalar segments
    std::vector<std::set<std::string>> defs(segs.size()), uses(segs.size());
    for (std::size_t s = 0; s < segs.size(); s++) {
      for (std::size_t i = segs[s].first; i < segs[s].second; i++) {
        const Statement& st = b.stmts[i];
        auto use = [&](const std::string& t) {
          if (!defs[s].count(t)) uses[s].insert(t);
        };
        if (st.kind == StmtKind::Store) use(st.from);
        if (st.kind == StmtKind::Intrinsic)
          for (const auto& a : st.args)
            if (!a.is_imm) use(a.temp);
        if (st.kind == StmtKind::Load || st.kind == StmtKind::Intrinsic) defs[s].insert(st.into);
      }
    }
    std::set<std::string> spilled;
    for (std::size_t s = 0; s < segs.size(); s++) spilled.insert(uses[s].begin(), uses[s].end());

    std::size_t step_mark = plan_->steps.size();
    std::size_t buf_mark = plan_->bufs.size();
    emit_segments(b, views, priv, path, segs, defs, uses, spilled);

    if (point_count() > 1 && hazard(step_mark, private_mark)) {
      // Phase splitting would reorder conflicting accesses across points of
      // this block: unroll its points on the host so every point runs its
      // phases in order (exact lexicographic semantics, interp.cpp:365-384).
      plan_->steps.resize(step_mark);
      plan_->bufs.resize(buf_mark);
      std::vector<int> free;
      for (std::size_t d = 0; d < dims_.size(); d++)
        if (!dims_[d].pinned && dims_[d].range > 1) free.push_back(static_cast<int>(d));
      std::int64_t n = point_count();
      if (n > opt_.max_unroll)
        throw Error("Unsupported", "block " + path + " needs serial phases over " +
                                       std::to_string(n) + " points");
      plan_->notes.push_back("block " + (path.empty() ? std::string("root") : path) +
                             ": cross-phase conflict, host-unrolled over " + std::to_string(n) +
                             " points");
      for (std::int64_t pt = 0; pt < n; pt++) {
        std::int64_t rest = pt;
        for (std::size_t i = free.size(); i-- > 0;) {
          dims_[free[i]].pinned = true;
          dims_[free[i]].value = rest % dims_[free[i]].range;
          rest /= dims_[free[i]].range;
        }
        emit_segments(b, views, priv, path, segs, defs, uses, spilled);
      }
      for (int d : free) dims_[d].pinned = false;
    }
  }

  void emit_segments(const Block& b, const Views& views,
                     const std::vector<std::pair<Agg, DType>>& priv, const std::string& path,
                     const std::vector<std::pair<std::size_t, std::size_t>>& segs,
                     const std::vector<std::set<std::string>>& defs,
                     const std::vector<std::set<std::string>>& uses,
                     const std::set<std::string>& spilled) {
    SpillInfo spill;
    if (!spilled.empty()) {
      int slot = 0;
      for (const auto& t : spilled) spill.slot[t] = slot++;
      spill.slots = slot;
      spill.buf = new_scratch("spill:" + path, DType::I32, kI64, point_count() * spill.slots);
      spill.base = linearize(spill.slots);
    }
    for (std::size_t s = 0; s < segs.size(); s++) {
      if (b.stmts[segs[s].first].kind == StmtKind::Block) {
        lower_block(*b.stmts[segs[s].first].block, views, join(path, segs[s].first), false);
        continue;
      }
      spill.live_in = uses[s];
      spill.live_out.clear();
      for (const auto& t : defs[s]) {
        bool later = false;
        for (std::size_t s2 = s + 1; s2 < segs.size(); s2++) later |= uses[s2].count(t) > 0;
        if (later) spill.live_out.insert(t);
      }
      emit_leaf(b, b.stmts, segs[s].first, segs[s].second, views, priv,
                join(path, segs[s].first), spill.buf >= 0 ? &spill : nullptr);
    }
  }

  // Conflict test over the launches of one phase-split block (conservative).
  bool hazard(std::size_t step_mark, std::size_t buf_mark) const {
    struct Use {
      std::set<std::size_t> readers, writers;
      std::set<int> aggs;
    };
    std::map<int, Use> uses;
    for (std::size_t s = step_mark; s < plan_->steps.size(); s++) {
      const PStep& st = plan_->steps[s];
      if (st.kind != PStep::Launch) continue;
      const PLaunch& l = st.launch;
      for (const auto& ins : l.code) {
        if (ins.op == kOpLoad) uses[l.acc[ins.acc].buf].readers.insert(s);
        if (ins.op == kOpStore) {
          auto& u = uses[l.acc[ins.acc].buf];
          u.writers.insert(s);
          u.aggs.insert(ins.agg);
        }
        if (ins.op == kOpGather || ins.op == kOpScatter) {
          const PSpecial& sp = l.specials[ins.acc];
          uses[l.acc[sp.src].buf].readers.insert(s);
          uses[l.acc[sp.idx].buf].readers.insert(s);
          auto& u = uses[l.acc[sp.dst].buf];
          u.writers.insert(s);
          u.aggs.insert(static_cast<int>(sp.dst_agg));
          u.readers.insert(s);
        }
      }
    }
    for (const auto& [buf, u] : uses) {
      if (buf >= static_cast<int>(buf_mark)) continue;  // private to this block's points
      if (u.writers.empty()) continue;
      for (auto w : u.writers)
        for (auto r : u.readers)
          if (w != r) return true;
      if (u.writers.size() > 1) {
        if (u.aggs.size() > 1) return true;
        if (u.aggs.count(static_cast<int>(Agg::Assign))) return true;
      }
    }
    return false;
  }

  // ---- leaf body compilation -------------------------------------------------------------
  void emit_leaf(const Block& b, const std::vector<Statement>& stmts, std::size_t begin,
                 std::size_t end, const Views& views,
                 const std::vector<std::pair<Agg, DType>>& priv, const std::string& path,
                 const SpillInfo* spill) {
    PLaunch l;
    l.path = path.empty() ? "root" : path;
    l.priv = priv;
    std::map<std::string, int> temps;
    auto temp_def = [&](const std::string& n) {
      auto it = temps.find(n);
      if (it != temps.end()) return it->second;
      int t = static_cast<int>(temps.size());
      temps[n] = t;
      return t;
    };
    auto temp_use = [&](const std::string& n) {
      auto it = temps.find(n);
      if (it == temps.end()) throw Error("UndefinedTemp", "use of undefined scalar temp '" + n + "'");
      return it->second;
    };
    auto access = [&](int buf, const FAff& a) {
      for (std::size_t i = 0; i < l.acc.size(); i++)
        if (l.acc[i].buf == buf && l.acc[i].addr == a) return static_cast<int>(i);
      l.acc.push_back(PAccess{buf, a});
      return static_cast<int>(l.acc.size()) - 1;
    };
    auto view_of = [&](const std::string& n) -> const View& {
      auto it = views.find(n);
      if (it == views.end())
        throw Error("MissingBuffer", "statement names undeclared buffer '" + n + "'");
      return it->second;
    };
    auto konst = [&](std::int64_t v) -> std::int16_t {
      for (std::size_t i = 0; i < l.consts.size(); i++)
        if (l.consts[i] == v) return static_cast<std::int16_t>(-1 - static_cast<int>(i));
      l.consts.push_back(v);
      return static_cast<std::int16_t>(-static_cast<int>(l.consts.size()));
    };
    auto push = [&](DInstr ins) { l.code.push_back(ins); };

    if (spill) {
      l.has_spill = true;
      for (const auto& t : spill->live_in) {
        FAff a = spill->base;
        a.c += spill->slot.at(t);
        DInstr ins{};
        ins.op = kOpLoad;
        ins.acc = static_cast<std::int8_t>(access(spill->buf, a));
        ins.dst = static_cast<std::int16_t>(temp_def(t));
        push(ins);
      }
    }
    for (std::size_t i = begin; i < end; i++) {
      const Statement& s = stmts[i];
      DInstr ins{};
      switch (s.kind) {
        case StmtKind::Load: {
          const View& v = view_of(s.from);
          if (v.priv >= 0) {
            ins.op = kOpLoadPriv;
            ins.acc = static_cast<std::int8_t>(v.priv);
          } else {
            ins.op = kOpLoad;
            ins.acc = static_cast<std::int8_t>(access(v.buf, v.base));
          }
          ins.dst = static_cast<std::int16_t>(temp_def(s.into));
          break;
        }
        case StmtKind::Store: {
          const View& v = view_of(s.into);
          ins.a = static_cast<std::int16_t>(temp_use(s.from));
          ins.agg = static_cast<std::int8_t>(v.ref->has_agg ? v.ref->agg : Agg::Assign);
          ins.dtype = static_cast<std::int8_t>(v.ref->dtype);
          if (v.priv >= 0) {
            ins.op = kOpStorePriv;
            ins.acc = static_cast<std::int8_t>(v.priv);
          } else {
            ins.op = kOpStore;
            ins.acc = static_cast<std::int8_t>(access(v.buf, v.base));
          }
          break;
        }
        case StmtKind::Intrinsic: {
          ins.op = opcode(s.op);
          if (static_cast<int>(s.args.size()) < arity(s.op))
            throw Error("UnknownIntrinsic", "intrinsic '" + s.op + "' has too few operands");
          std::int16_t ops[3] = {0, 0, 0};
          for (int a = 0; a < arity(s.op); a++)
            ops[a] = s.args[a].is_imm ? konst(s.args[a].imm)
                                      : static_cast<std::int16_t>(temp_use(s.args[a].temp));
          ins.a = ops[0];
          ins.b = ops[1];
          ins.c = ops[2];
          ins.dst = static_cast<std::int16_t>(temp_def(s.into));
          break;
        }
        case StmtKind::Special: {
          if (s.op != "gather" && s.op != "scatter")
            throw Error("UnknownSpecial", "unknown special '" + s.op + "'");
          if (s.refs.size() != 3)
            throw Error("UnknownSpecial", "special '" + s.op + "' expects 3 refinement operands");
          const View& dst = view_of(s.refs[0]);
          const View& src = view_of(s.refs[1]);
          const View& idx = view_of(s.refs[2]);
          if (dst.priv >= 0 || src.priv >= 0 || idx.priv >= 0)
            throw Error("Unsupported", "special on a private allocation");
          PSpecial sp;
          sp.gather = s.op == "gather";
          const Refinement& walk = sp.gather ? *dst.ref : *src.ref;
          if (idx.ref->sizes != walk.sizes)
            throw Error("UnknownSpecial", "index operand shape must match the walked operand");
          if (dst.ref->rank() != src.ref->rank())
            throw Error("UnknownSpecial", "gather/scatter operands must have equal rank");
          if (walk.rank() > static_cast<std::size_t>(kMaxRank))
            throw Error("Unsupported", "special rank too large");
          sp.dst = access(dst.buf, dst.base);
          sp.src = access(src.buf, src.base);
          sp.idx = access(idx.buf, idx.base);
          sp.walk = walk.sizes;
          sp.sdst = dst.ref->strides;
          sp.ssrc = src.ref->strides;
          sp.sidx = idx.ref->strides;
          sp.bound = sp.gather ? src.ref->sizes[0] : dst.ref->sizes[0];
          sp.dst_agg = dst.ref->has_agg ? dst.ref->agg : Agg::Assign;
          sp.dst_dtype = dst.ref->dtype;
          ins.op = sp.gather ? kOpGather : kOpScatter;
          ins.acc = static_cast<std::int8_t>(l.specials.size());
          l.specials.push_back(sp);
          break;
        }
        case StmtKind::Block: break;
      }
      push(ins);
    }
    if (spill) {
      for (const auto& t : spill->live_out) {
        FAff a = spill->base;
        a.c += spill->slot.at(t);
        DInstr ins{};
        ins.op = kOpStore;
        ins.acc = static_cast<std::int8_t>(access(spill->buf, a));
        ins.a = static_cast<std::int16_t>(temp_use(t));
        ins.agg = static_cast<std::int8_t>(Agg::Assign);
        ins.dtype = -1;  // int64 spill: no wrap
        push(ins);
      }
    }
    l.ntemps = static_cast<int>(temps.size());
    finalize(l);
    PStep st;
    st.kind = PStep::Launch;
    st.launch = std::move(l);
    plan_->steps.push_back(std::move(st));
  }

  // Compacts dims (drop range-1 and pinned dims, folding pinned values into the
  // constants), then chooses the execution mode.
  void finalize(PLaunch& l) {
    std::vector<int> keep;
    for (std::size_t d = 0; d < dims_.size(); d++)
      if (!dims_[d].pinned && dims_[d].range > 1) keep.push_back(static_cast<int>(d));
    auto compact = [&](const FAff& f) {
      FAff o;
      o.c = f.c;
      for (std::size_t d = 0; d < dims_.size(); d++)
        if (dims_[d].pinned) o.c += f.at(d) * dims_[d].value;
      for (int d : keep) o.k.push_back(f.at(d));
      return o;
    };
    for (int d : keep) l.dims.push_back(dims_[d]);
    for (const auto& c : cons_) {
      FAff f = compact(c);
      bool trivial = true;
      for (auto k : f.k) trivial &= k == 0;
      if (trivial && f.c >= 0) continue;  // always true
      l.cons.push_back(f);
    }
    for (auto& a : l.acc) a.addr = compact(a.addr);
    coalesce(l);
    if (l.dims.size() > static_cast<std::size_t>(kMaxDims))
      throw Error("Unsupported", "nest at " + l.path + " has more than 24 non-trivial indexes");
    analyze(l);
  }

  // Loop coalescing: adjacent dims (d outer, d+1 inner) with k[d] == k[d+1] * range[d+1]
  // in every access and constraint are one index of range r_d * r_{d+1} (a tiled index
  // after tile_rewrite, tile.cpp:100-235, becomes untiled again).  Adjacency keeps the
  // lexicographic order, so execution semantics are unchanged.
  // A launch whose result does not depend on the order of its points: no buffer is both
  // read and written, and every written buffer either aggregates with one integer
  // commutative-associative op (add/mul/max/min wrap modulo 2^n) or is written at most once
  // per address (injective over all dims).  Its dims may be merged in any order.
  bool order_free(const PLaunch& l) const {
    if (!l.specials.empty() || !l.priv.empty() || l.has_spill) return false;
    std::set<int> loaded;
    std::map<int, std::set<int>> aggs;
    for (const auto& ins : l.code) {
      if (ins.op == kOpLoad) loaded.insert(l.acc[ins.acc].buf);
      if (ins.op == kOpStore) aggs[l.acc[ins.acc].buf].insert(ins.agg);
    }
    for (const auto& a : l.acc)
      if (plan_->bufs[a.buf].dtype == DType::F32) return false;
    std::vector<int> all;
    for (std::size_t d = 0; d < l.dims.size(); d++) all.push_back(static_cast<int>(d));
    for (auto& [b, s] : aggs) {
      if (loaded.count(b)) return false;
      bool comm = s.size() == 1 && !s.count(static_cast<int>(Agg::Assign));
      if (comm) continue;
      int nst = 0;
      const FAff* addr = nullptr;
      for (const auto& ins : l.code)
        if (ins.op == kOpStore && l.acc[ins.acc].buf == b) {
          nst++;
          addr = &l.acc[ins.acc].addr;
        }
      if (nst != 1 || !injective(*addr, all, l.dims)) return false;
    }
    return true;
  }

  void coalesce(PLaunch& l) const {
    coalesce_adjacent(l);
    if (!order_free(l)) return;
    // any two dims d (outer) and e (inner) with k_d = k_e * r_e everywhere are one index
    // (e.g. the outer and inner halves of a tile_rewrite-tiled index that other indexes
    // separate in the nest); order-free launches may iterate them merged
    bool changed = true;
    while (changed) {
      changed = false;
      for (std::size_t d = 0; d < l.dims.size() && !changed; d++)
        for (std::size_t e = 0; e < l.dims.size() && !changed; e++) {
          if (d == e) continue;
          const std::int64_t re = l.dims[e].range;
          auto ok = [&](const FAff& f) { return f.at(d) == f.at(e) * re; };
          bool all = true;
          bool used = false;
          for (const auto& a : l.acc) {
            all &= ok(a.addr);
            used |= a.addr.uses(e);
          }
          for (const auto& c : l.cons) all &= ok(c);
          if (!all || !used) continue;
          for (auto& a : l.acc)
            if (d < a.addr.k.size()) a.addr.k.erase(a.addr.k.begin() + static_cast<long>(d));
          for (auto& c : l.cons)
            if (d < c.k.size()) c.k.erase(c.k.begin() + static_cast<long>(d));
          l.dims[e].name = l.dims[d].name + "*" + l.dims[e].name;
          l.dims[e].range *= l.dims[d].range;
          l.dims.erase(l.dims.begin() + static_cast<long>(d));
          changed = true;
        }
    }
    coalesce_adjacent(l);
  }

  static void coalesce_adjacent(PLaunch& l) {
    bool changed = true;
    while (changed) {
      changed = false;
      for (std::size_t d = 0; d + 1 < l.dims.size(); d++) {
        const std::int64_t r1 = l.dims[d + 1].range;
        auto ok = [&](const FAff& f) { return f.at(d) == f.at(d + 1) * r1; };
        bool all = true;
        for (const auto& a : l.acc) all &= ok(a.addr);
        for (const auto& c : l.cons) all &= ok(c);
        if (!all) continue;
        auto drop = [&](FAff& f) {
          if (d < f.k.size()) f.k.erase(f.k.begin() + static_cast<long>(d));
        };
        for (auto& a : l.acc) drop(a.addr);
        for (auto& c : l.cons) drop(c);
        l.dims[d + 1].name = l.dims[d].name + "*" + l.dims[d + 1].name;
        l.dims[d + 1].range *= l.dims[d].range;
        l.dims.erase(l.dims.begin() + static_cast<long>(d));
        changed = true;
        break;
      }
    }
  }

  void analyze(PLaunch& l) {
    const int nd = static_cast<int>(l.dims.size());
    l.points = 1;
    for (const auto& d : l.dims) l.points *= d.range;
    l.acc_mode.assign(l.acc.size(), kAccRead);
    l.acc_cell.assign(l.acc.size(), -1);
    std::set<int> written;
    std::map<int, std::set<int>> aggs;
    bool special = false;
    for (const auto& ins : l.code) {
      if (ins.op == kOpStore) {
        written.insert(l.acc[ins.acc].buf);
        aggs[l.acc[ins.acc].buf].insert(ins.agg);
      }
      if (ins.op == kOpGather || ins.op == kOpScatter) {
        special = true;
        written.insert(l.acc[l.specials[ins.acc].dst].buf);
      }
    }
    auto serial = [&](const std::string& why) {
      l.mode = kModeSerial;
      l.why = why;
      l.pdims.clear();
      l.rdims.clear();
      for (int d = 0; d < nd; d++) l.rdims.push_back(d);
      for (std::size_t i = 0; i < l.acc.size(); i++)
        l.acc_mode[i] = written.count(l.acc[i].buf) ? kAccDirect : kAccRead;
      l.pcount = 1;
    };
    // numeric mode: a launch over F32 buffers runs in fp32 (generic_f32.cu); the
    // integer semantics of interp.cpp never mix with it inside one launch
    {
      int nf = 0, ni = 0;
      for (const auto& a : l.acc) {
        const PBuffer& b = plan_->bufs[a.buf];
        if (b.kind == kI64) continue;  // temp spill: carries either mode's value
        (b.dtype == DType::F32 ? nf : ni)++;
      }
      for (const auto& pr : l.priv) (pr.second == DType::F32 ? nf : ni)++;
      if (nf && ni) throw Error("Unsupported", "launch " + l.path + " mixes f32 and integer buffers");
      l.is_float = nf > 0;
      if (l.is_float && special) throw Error("Unsupported", "gather/scatter over f32 buffers");
    }
    if (special) return serial("gather/scatter");
    // every access of a written buffer must use one address function
    std::map<int, int> rep;  // buf -> representative access
    for (std::size_t i = 0; i < l.acc.size(); i++) {
      int b = l.acc[i].buf;
      if (!written.count(b)) continue;
      auto it = rep.find(b);
      if (it == rep.end()) rep[b] = static_cast<int>(i);
      else if (!(l.acc[it->second].addr == l.acc[i].addr))
        return serial("buffer '" + plan_->bufs[b].name + "' accessed at several addresses");
    }
    std::set<int> P;
    for (auto& [b, i] : rep)
      for (int d = 0; d < nd; d++)
        if (l.acc[i].addr.uses(d)) P.insert(d);
    if (written.empty())
      for (int d = 0; d < nd; d++) P.insert(d);
    std::vector<int> pv(P.begin(), P.end());
    bool inj = true;
    for (auto& [b, i] : rep) inj &= injective(l.acc[i].addr, pv, l.dims);
    if (!inj) {
      bool loads_written = false;
      for (const auto& ins : l.code)
        if (ins.op == kOpLoad && written.count(l.acc[ins.acc].buf)) loads_written = true;
      bool commutative = true;
      for (auto& [b, s] : aggs)
        commutative &= s.size() == 1 && !s.count(static_cast<int>(Agg::Assign));
      if (loads_written || !commutative)
        return serial("written addresses do not determine the thread");
      l.mode = kModeAtomic;
      l.why = "non-injective commutative aggregation";
      for (int d = nd; d-- > 0;) l.pdims.push_back(d);
      for (std::size_t i = 0; i < l.acc.size(); i++)
        l.acc_mode[i] = written.count(l.acc[i].buf) ? kAccAtomic : kAccRead;
      l.pcount = l.points;
      return;
    }
    l.mode = kModeOwner;
    // thread order: fastest-varying = smallest |stride| in the first written access
    const FAff* key = rep.empty() ? nullptr : &l.acc[rep.begin()->second].addr;
    std::vector<int> order = pv;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      if (!key) return a > b;
      std::int64_t ka = std::llabs(key->at(a)), kb = std::llabs(key->at(b));
      return ka < kb;
    });
    l.pdims = order;
    for (int d = 0; d < nd; d++)
      if (!P.count(d)) l.rdims.push_back(d);
    l.pcount = 1;
    for (int d : l.pdims) l.pcount *= l.dims[d].range;
    std::map<int, int> cell_of;
    for (std::size_t i = 0; i < l.acc.size(); i++) {
      int b = l.acc[i].buf;
      if (!written.count(b)) continue;
      if (!cell_of.count(b)) {
        int c = static_cast<int>(cell_of.size());
        cell_of[b] = c;
      }
      int c = cell_of[b];
      if (c < kMaxCells - static_cast<int>(l.priv.size())) {
        l.acc_mode[i] = kAccOwned;
        l.acc_cell[i] = static_cast<std::int8_t>(c);
      } else {
        l.acc_mode[i] = kAccDirect;  // still thread-owned; just not register cached
      }
    }
    l.ncells = std::min<int>(static_cast<int>(cell_of.size()), kMaxCells - static_cast<int>(l.priv.size()));
  }

  using Scope = std::map<std::string, FAff>;
  const Program& p_;
  const PlanOptions& opt_;
  Plan* plan_;
  std::vector<PDim> dims_;
  std::vector<Scope> scopes_;
  std::vector<FAff> cons_;
};

}  // namespace

void match_kernels(Plan* plan, const Program& p, const PlanOptions& opt);  // matcher.cpp

Plan build_plan(const Program& p, const PlanOptions& opt) {
  Plan plan;
  Lowerer(p, opt, &plan).run();
  match_kernels(&plan, p, opt);
  return plan;
}

std::string Plan::describe() const {
  std::ostringstream os;
  static const char* modes[] = {"owner", "atomic", "serial"};
  static const char* kinds[] = {"generic", "conv_i8_tc", "map", "reduce", "gemm_i8_tc", "conv_igemm_tc", "pool", "gemm_f32"};
  for (const auto& s : steps) {
    if (s.elided) os << "(elided) ";
    if (s.kind == PStep::Fill) {
      os << "fill " << bufs[s.buf].name << " = " << s.value << " (" << bufs[s.buf].elements
         << " elems)\n";
      continue;
    }
    const PLaunch& l = s.launch;
    os << "launch " << l.path << " kernel=" << kinds[static_cast<int>(l.kernel)]
       << " mode=" << modes[l.mode] << " dims=[";
    for (std::size_t d = 0; d < l.dims.size(); d++)
      os << (d ? "," : "") << l.dims[d].name << ":" << l.dims[d].range;
    os << "] pdims=[";
    for (std::size_t i = 0; i < l.pdims.size(); i++) os << (i ? "," : "") << l.dims[l.pdims[i]].name;
    os << "] rdims=[";
    for (std::size_t i = 0; i < l.rdims.size(); i++) os << (i ? "," : "") << l.dims[l.rdims[i]].name;
    os << "] cons=" << l.cons.size() << " acc=" << l.acc.size() << " code=" << l.code.size()
       << " points=" << l.points;
    if (l.is_float) os << " f32";
    if (l.kernel == KernelKind::ConvI8TC || l.kernel == KernelKind::ConvIgemmTC) {
      const ConvPlan& c = l.conv;
      if (c.epi)
        os << " epilogue=" << (c.epi_vec ? "vec" : "") << (c.epi_res ? "+res" : "") << (c.epi_lo ? "+clamp" : "");
      if (c.fresh_output) os << " fresh";
    }
    if (l.kernel == KernelKind::Pool && l.pool.fresh) os << " fresh";
    if (!l.why.empty()) os << " why=\"" << l.why << "\"";
    os << "\n";
  }
  for (const auto& n : notes) os << "note " << n << "\n";
  return os.str();
}

void to_desc(const PLaunch& l, GenericDesc* d, std::vector<int>* bufmap) {
  std::memset(d, 0, sizeof(*d));
  bufmap->clear();
  auto slot = [&](int plan_buf) {
    for (std::size_t i = 0; i < bufmap->size(); i++)
      if ((*bufmap)[i] == plan_buf) return static_cast<int>(i);
    bufmap->push_back(plan_buf);
    if (bufmap->size() > static_cast<std::size_t>(kMaxBufs))
      throw Error("Unsupported", "launch " + l.path + " touches too many buffers");
    return static_cast<int>(bufmap->size()) - 1;
  };
  auto chk = [&](std::size_t n, int cap, const char* what) {
    if (n > static_cast<std::size_t>(cap))
      throw Error("Unsupported", std::string("launch ") + l.path + ": too many " + what);
  };
  chk(l.dims.size(), kMaxDims, "dims");
  chk(l.cons.size(), kMaxCons, "constraints");
  chk(l.acc.size(), kMaxAccess, "accesses");
  chk(l.code.size(), kMaxCode, "statements");
  chk(l.consts.size(), kMaxConsts, "immediates");
  chk(static_cast<std::size_t>(l.ntemps), kMaxTemps, "temps");
  chk(l.specials.size(), kMaxSpecial, "specials");
  chk(l.priv.size() + l.ncells, kMaxCells, "cells");
  d->ndims = static_cast<int>(l.dims.size());
  d->ncons = static_cast<int>(l.cons.size());
  d->nacc = static_cast<int>(l.acc.size());
  d->ncode = static_cast<int>(l.code.size());
  d->nconsts = static_cast<int>(l.consts.size());
  d->ntemps = l.ntemps;
  d->ncells = l.ncells;
  d->npriv = static_cast<int>(l.priv.size());
  d->nspecial = static_cast<int>(l.specials.size());
  d->vdim = static_cast<std::int8_t>(l.vdim);
  d->vcount = l.vcount;
  for (std::size_t i = 0; i < l.vkind.size() && i < static_cast<std::size_t>(kMaxAccess); i++) d->vkind[i] = l.vkind[i];
  d->mode = l.mode;
  d->is_float = l.is_float ? 1 : 0;
  d->npdims = static_cast<std::int8_t>(l.pdims.size());
  d->nrdims = static_cast<std::int8_t>(l.rdims.size());
  for (std::size_t i = 0; i < l.pdims.size(); i++) d->pdims[i] = static_cast<std::int8_t>(l.pdims[i]);
  for (std::size_t i = 0; i < l.rdims.size(); i++) d->rdims[i] = static_cast<std::int8_t>(l.rdims[i]);
  for (std::size_t i = 0; i < l.dims.size(); i++) d->range[i] = l.dims[i].range;
  d->pcount = l.pcount;
  for (std::size_t i = 0; i < l.priv.size(); i++) {
    d->priv_agg[i] = static_cast<std::int8_t>(l.priv[i].first);
    d->priv_dtype[i] = static_cast<std::int8_t>(l.priv[i].second);
  }
  auto aff = [&](const FAff& f, DAff* o) {
    o->c = f.c;
    for (std::size_t k = 0; k < l.dims.size(); k++) o->k[k] = f.at(k);
  };
  for (std::size_t i = 0; i < l.cons.size(); i++) aff(l.cons[i], &d->cons[i]);
  for (std::size_t i = 0; i < l.acc.size(); i++) {
    d->acc[i].buf = static_cast<std::int16_t>(slot(l.acc[i].buf));
    d->acc[i].mode = l.acc_mode[i];
    d->acc[i].cell = l.acc_cell[i];
    aff(l.acc[i].addr, &d->acc[i].addr);
  }
  for (std::size_t i = 0; i < l.code.size(); i++) d->code[i] = l.code[i];
  for (std::size_t i = 0; i < l.consts.size(); i++) d->consts[i] = l.consts[i];
  for (std::size_t i = 0; i < l.specials.size(); i++) {
    const PSpecial& s = l.specials[i];
    DSpecial& o = d->special[i];
    o.dst = static_cast<std::int8_t>(s.dst);
    o.src = static_cast<std::int8_t>(s.src);
    o.idx = static_cast<std::int8_t>(s.idx);
    o.rank = static_cast<std::int8_t>(s.walk.size());
    o.dst_agg = static_cast<std::int8_t>(s.dst_agg);
    o.dst_dtype = static_cast<std::int8_t>(s.dst_dtype);
    o.bound = s.bound;
    for (std::size_t r = 0; r < s.walk.size(); r++) {
      o.walk[r] = s.walk[r];
      o.sdst[r] = s.sdst[r];
      o.ssrc[r] = s.ssrc[r];
      o.sidx[r] = s.sidx[r];
    }
  }
}

}  // namespace sb
