// oracle/port/stripe_port.cpp — TEST INFRASTRUCTURE ONLY (see stripe_port.hpp).
//
// Restates the serial reference semantics:
//   block entry: aliases evaluated once from the parent env (interp.cpp:362-364)
//   lexicographic odometer, last index fastest          (interp.cpp:365-384)
//   constraints skip a point                            (interp.cpp:426-428)
//   views: external base / parent base + flat base / fresh zeroed alloc per point
//                                                       (interp.cpp:433-453)
//   temps zeroed per point, statements serial           (interp.cpp:454-457)
//   load/store touch the single element at the view base (interp.cpp:497-504)
//   bounds checks -> OutOfBoundsAccess                  (interp.cpp:461-483)
//   intrinsics on int64 temps, wrap only at 2^64        (interp.cpp:515-537)
//   gather / scatter specials                           (interp.cpp:540-600)
//   store-time aggregation                              (ir.cpp:79-97)
#include "stripe_port.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <memory>

namespace sbport {
namespace {

using sb::Agg;
using sb::DType;
using sb::Error;

struct IntPolicy {
  using V = std::int64_t;  // temp
  using S = std::int64_t;  // storage element
  static V from_imm(std::int64_t v) { return v; }
  static V load(S s) { return s; }
  static S store(Agg a, S cur, V in, DType d) { return sb::aggregate(a, cur, in, d); }
  static V add(V a, V b) { return static_cast<V>(static_cast<std::uint64_t>(a) + static_cast<std::uint64_t>(b)); }
  static V sub(V a, V b) { return static_cast<V>(static_cast<std::uint64_t>(a) - static_cast<std::uint64_t>(b)); }
  static V mul(V a, V b) { return static_cast<V>(static_cast<std::uint64_t>(a) * static_cast<std::uint64_t>(b)); }
  static std::int64_t as_index(S s) { return s; }
  static bool truthy(V v) { return v != 0; }
};

struct F32Policy {
  using V = float;
  using S = float;
  static V from_imm(std::int64_t v) { return static_cast<float>(v); }
  static V load(S s) { return s; }
  static S store(Agg a, S cur, V in, DType) {
    switch (a) {
      case Agg::Assign: return in;
      case Agg::Add: return cur + in;
      case Agg::Max: return std::max(cur, in);
      case Agg::Min: return std::min(cur, in);
      case Agg::Mul: return cur * in;
    }
    return in;
  }
  static V add(V a, V b) { return a + b; }
  static V sub(V a, V b) { return a - b; }
  static V mul(V a, V b) { return a * b; }
  static std::int64_t as_index(S s) { return static_cast<std::int64_t>(s); }
  static bool truthy(V v) { return v != 0.0f; }
};

// Affine over environment slots.
struct SAff {
  std::int64_t c = 0;
  std::vector<std::pair<int, std::int64_t>> t;
  std::int64_t at(const std::vector<std::int64_t>& env) const {
    std::int64_t v = c;
    for (auto& [s, k] : t) v += k * env[s];
    return v;
  }
};

enum Kind { kExternal, kParent, kAlloc };

struct CRef {
  const sb::Refinement* ref;
  Kind kind;
  int parent = -1;
  SAff base;
  std::int64_t alloc_elems = 0;
};

enum Op { oLoad, oStore, oIntr, oGather, oScatter, oBlock };

struct CStmt {
  Op op;
  int view = 0, temp = 0;
  std::string intr;
  std::vector<std::pair<bool, std::int64_t>> args;  // (is_imm, imm-or-temp)
  int dst = 0, src = 0, idx = 0;
  std::unique_ptr<struct CBlk> child;
};

struct CBlk {
  std::vector<std::pair<int, std::int64_t>> ranged;
  std::vector<std::pair<int, SAff>> aliases;
  std::vector<SAff> cons;
  std::vector<CRef> refs;
  std::vector<CStmt> stmts;
  int ntemps = 0;
  int env_top = 0;
};

using Scope = std::map<std::string, int>;

SAff resolve(const sb::Affine& a, const std::vector<Scope*>& scopes) {
  SAff out;
  out.c = a.constant;
  for (const auto& [name, k] : a.terms) {
    int slot = -1;
    for (auto it = scopes.rbegin(); it != scopes.rend() && slot < 0; ++it) {
      auto f = (*it)->find(name);
      if (f != (*it)->end()) slot = f->second;
    }
    if (slot < 0) throw Error("UnboundIndex", "unbound index '" + name + "'");
    out.t.emplace_back(slot, k);
  }
  return out;
}

template <class P>
class Interp {
 public:
  using V = typename P::V;
  using S = typename P::S;
  using Bufs = std::map<std::string, std::vector<S>>;

  Interp(const sb::Program& p, Bufs* bufs, int order) : p_(p), bufs_(bufs), order_(order) {}

  void run() {
    for (const auto& d : p_.buffers) {
      auto it = bufs_->find(d.name);
      if (it == bufs_->end())
        throw Error("MissingBuffer", "buffer '" + d.name + "' not present in store");
      if (static_cast<std::int64_t>(it->second.size()) != d.elements)
        throw Error("MissingBuffer", "buffer '" + d.name + "' has wrong element count");
    }
    std::vector<Scope*> scopes;
    std::map<std::string, int> none;
    auto root = compile(p_.root, 0, none, scopes, true);
    env_.assign(64, 0);
    std::deque<Frame> frames;
    exec_block(*root, frames);
  }

 private:
  struct View {
    std::vector<S>* data = nullptr;
    std::int64_t base = 0;
    const CRef* cref = nullptr;
  };
  struct Frame {
    std::vector<View> views;
    std::vector<V> temps;
    std::vector<std::unique_ptr<std::vector<S>>> allocs;
  };

  std::unique_ptr<CBlk> compile(const sb::Block& b, int env_base,
                                const std::map<std::string, int>& parent_views,
                                std::vector<Scope*>& scopes, bool is_root) {
    auto cb = std::make_unique<CBlk>();
    Scope own;
    int slot = env_base;
    for (const auto& idx : b.indexes) {
      if (idx.is_alias) cb->aliases.emplace_back(slot, resolve(idx.alias, scopes));
      else cb->ranged.emplace_back(slot, idx.range);
      own[idx.name] = slot++;
    }
    cb->env_top = slot;
    scopes.push_back(&own);
    for (const auto& c : b.constraints) cb->cons.push_back(resolve(c, scopes));
    std::map<std::string, int> views;
    for (const auto& r : b.refs) {
      CRef cr;
      cr.ref = &r;
      for (std::size_t d = 0; d < r.offsets.size(); d++) {
        SAff o = resolve(r.offsets[d], scopes);
        cr.base.c += o.c * r.strides[d];
        for (auto& [s, k] : o.t) cr.base.t.emplace_back(s, k * r.strides[d]);
      }
      auto pv = parent_views.find(r.name);
      if (pv != parent_views.end()) {
        cr.kind = kParent;
        cr.parent = pv->second;
      } else if (is_root) {
        cr.kind = kExternal;
      } else {
        cr.kind = kAlloc;
        cr.alloc_elems = r.extent();
      }
      views[r.name] = static_cast<int>(cb->refs.size());
      cb->refs.push_back(std::move(cr));
    }
    auto view_of = [&](const std::string& n) {
      auto it = views.find(n);
      if (it == views.end()) throw Error("MissingBuffer", "undeclared buffer '" + n + "'");
      return it->second;
    };
    std::map<std::string, int> temps;
    auto temp_of = [&](const std::string& n, bool def) {
      auto it = temps.find(n);
      if (it != temps.end()) return it->second;
      if (!def) throw Error("UndefinedTemp", "use of undefined scalar temp '" + n + "'");
      int t = static_cast<int>(temps.size());
      temps[n] = t;
      return t;
    };
    static const char* known[] = {"add", "sub", "mul", "neg", "max", "min", "cmp_eq",
                                  "cmp_ne", "cmp_lt", "cmp_le", "cmp_gt", "cmp_ge",
                                  "select", "constant"};
    for (const auto& s : b.stmts) {
      CStmt cs;
      switch (s.kind) {
        case sb::StmtKind::Block:
          cs.op = oBlock;
          cs.child = compile(*s.block, cb->env_top, views, scopes, false);
          break;
        case sb::StmtKind::Load:
          cs.op = oLoad;
          cs.view = view_of(s.from);
          cs.temp = temp_of(s.into, true);
          break;
        case sb::StmtKind::Store:
          cs.op = oStore;
          cs.view = view_of(s.into);
          cs.temp = temp_of(s.from, false);
          break;
        case sb::StmtKind::Intrinsic: {
          bool ok = false;
          for (const char* k : known) ok |= s.op == k;
          if (!ok) throw Error("UnknownIntrinsic", "unknown intrinsic '" + s.op + "'");
          cs.op = oIntr;
          cs.intr = s.op;
          for (const auto& a : s.args)
            cs.args.emplace_back(a.is_imm, a.is_imm ? a.imm : temp_of(a.temp, false));
          cs.temp = temp_of(s.into, true);
          break;
        }
        case sb::StmtKind::Special:
          if (s.op != "gather" && s.op != "scatter")
            throw Error("UnknownSpecial", "unknown special '" + s.op + "'");
          if (s.refs.size() != 3)
            throw Error("UnknownSpecial", "special '" + s.op + "' expects 3 refinement operands");
          cs.op = s.op == "gather" ? oGather : oScatter;
          cs.dst = view_of(s.refs[0]);
          cs.src = view_of(s.refs[1]);
          cs.idx = view_of(s.refs[2]);
          break;
      }
      cb->stmts.push_back(std::move(cs));
    }
    cb->ntemps = static_cast<int>(temps.size());
    scopes.pop_back();
    return cb;
  }

  void exec_block(const CBlk& cb, std::deque<Frame>& frames) {
    if (static_cast<int>(env_.size()) < cb.env_top) env_.resize(cb.env_top, 0);
    for (const auto& [s, a] : cb.aliases) env_[s] = a.at(env_);
    frames.emplace_back();
    Frame* f = &frames.back();
    f->views.resize(cb.refs.size());
    f->temps.resize(cb.ntemps);
    std::int64_t total = 1;
    for (auto& r : cb.ranged) total *= r.second;
    for (std::int64_t n = 0; n < total; n++) {
      std::int64_t ord = order_ == 1 ? total - 1 - n : n;
      for (std::size_t d = cb.ranged.size(); d-- > 0;) {
        env_[cb.ranged[d].first] = ord % cb.ranged[d].second;
        ord /= cb.ranged[d].second;
      }
      exec_point(cb, frames);
      f = &frames.back();
    }
    frames.pop_back();
  }

  void exec_point(const CBlk& cb, std::deque<Frame>& frames) {
    for (const auto& c : cb.cons)
      if (c.at(env_) < 0) return;
    Frame& f = frames.back();
    f.allocs.clear();
    for (std::size_t i = 0; i < cb.refs.size(); i++) {
      const CRef& cr = cb.refs[i];
      View& v = f.views[i];
      v.cref = &cr;
      if (cr.kind == kExternal) {
        v.data = &bufs_->at(cr.ref->name);
        v.base = cr.base.at(env_);
      } else if (cr.kind == kAlloc) {
        f.allocs.push_back(std::make_unique<std::vector<S>>(cr.alloc_elems, S{}));
        v.data = f.allocs.back().get();
        v.base = 0;
      } else {
        const View& pv = frames[frames.size() - 2].views[cr.parent];
        v.data = pv.data;
        v.base = pv.base + cr.base.at(env_);
      }
    }
    std::fill(f.temps.begin(), f.temps.end(), V{});
    for (const auto& s : cb.stmts) {
      Frame& fr = frames.back();
      switch (s.op) {
        case oLoad: {
          const View& v = fr.views[s.view];
          fr.temps[s.temp] = P::load(read(v, v.base));
          break;
        }
        case oStore: {
          const View& v = fr.views[s.view];
          write(v, v.base, fr.temps[s.temp]);
          break;
        }
        case oIntr: fr.temps[s.temp] = intrinsic(s, fr.temps); break;
        case oGather:
        case oScatter: special(s, fr); break;
        case oBlock: exec_block(*s.child, frames); break;
      }
    }
  }

  S read(const View& v, std::int64_t a) {
    if (a < 0 || a >= static_cast<std::int64_t>(v.data->size()))
      throw Error("OutOfBoundsAccess", "read of '" + v.cref->ref->name + "' at element " +
                                           std::to_string(a) + " outside buffer");
    return (*v.data)[a];
  }

  void write(const View& v, std::int64_t a, V val) {
    if (a < 0 || a >= static_cast<std::int64_t>(v.data->size()))
      throw Error("OutOfBoundsAccess", "write of '" + v.cref->ref->name + "' at element " +
                                           std::to_string(a) + " outside buffer");
    const sb::Refinement& r = *v.cref->ref;
    (*v.data)[a] = P::store(r.has_agg ? r.agg : Agg::Assign, (*v.data)[a], val, r.dtype);
  }

  V intrinsic(const CStmt& s, const std::vector<V>& t) {
    auto x = [&](std::size_t i) -> V {
      const auto& a = s.args.at(i);
      return a.first ? P::from_imm(a.second) : t[a.second];
    };
    const std::string& o = s.intr;
    if (o == "add") return P::add(x(0), x(1));
    if (o == "sub") return P::sub(x(0), x(1));
    if (o == "mul") return P::mul(x(0), x(1));
    if (o == "neg") return P::sub(V{}, x(0));
    if (o == "max") return std::max(x(0), x(1));
    if (o == "min") return std::min(x(0), x(1));
    if (o == "cmp_eq") return x(0) == x(1) ? V(1) : V(0);
    if (o == "cmp_ne") return x(0) != x(1) ? V(1) : V(0);
    if (o == "cmp_lt") return x(0) < x(1) ? V(1) : V(0);
    if (o == "cmp_le") return x(0) <= x(1) ? V(1) : V(0);
    if (o == "cmp_gt") return x(0) > x(1) ? V(1) : V(0);
    if (o == "cmp_ge") return x(0) >= x(1) ? V(1) : V(0);
    if (o == "select") return P::truthy(x(0)) ? x(1) : x(2);
    return x(0);  // constant
  }

  void special(const CStmt& s, Frame& f) {
    const View& dst = f.views[s.dst];
    const View& src = f.views[s.src];
    const View& idx = f.views[s.idx];
    bool gather = s.op == oGather;
    const sb::Refinement& walk = gather ? *dst.cref->ref : *src.cref->ref;
    if (idx.cref->ref->sizes != walk.sizes)
      throw Error("UnknownSpecial", "index operand shape must match the walked operand");
    if (dst.cref->ref->rank() != src.cref->ref->rank())
      throw Error("UnknownSpecial", "gather/scatter operands must have equal rank");
    std::size_t rank = walk.rank();
    std::int64_t total = 1;
    for (auto n : walk.sizes) total *= n;
    std::vector<std::int64_t> co(rank, 0);
    for (std::int64_t n = 0; n < total; n++) {
      std::int64_t rest = n;
      for (std::size_t d = rank; d-- > 0;) {
        co[d] = rest % walk.sizes[d];
        rest /= walk.sizes[d];
      }
      std::int64_t ia = idx.base;
      for (std::size_t d = 0; d < rank; d++) ia += co[d] * idx.cref->ref->strides[d];
      std::int64_t pick = P::as_index(read(idx, ia));
      const View& picked_side = gather ? src : dst;
      if (pick < 0 || pick >= picked_side.cref->ref->sizes[0])
        throw Error("OutOfBoundsAccess", std::string(gather ? "gather" : "scatter") +
                                             " index " + std::to_string(pick) + " outside range");
      std::int64_t sa = src.base, da = dst.base;
      if (gather) {
        sa += pick * src.cref->ref->strides[0];
        for (std::size_t d = 1; d < rank; d++) sa += co[d] * src.cref->ref->strides[d];
        for (std::size_t d = 0; d < rank; d++) da += co[d] * dst.cref->ref->strides[d];
      } else {
        da += pick * dst.cref->ref->strides[0];
        for (std::size_t d = 0; d < rank; d++) sa += co[d] * src.cref->ref->strides[d];
        for (std::size_t d = 1; d < rank; d++) da += co[d] * dst.cref->ref->strides[d];
      }
      write(dst, da, P::load(read(src, sa)));
    }
  }

  const sb::Program& p_;
  Bufs* bufs_;
  int order_;
  std::vector<std::int64_t> env_;
};

thread_local std::string g_err;

}  // namespace

void execute_int(const sb::Program& p, Store* s, int order) {
  Interp<IntPolicy>(p, &s->ints, order).run();
}
void execute_f32(const sb::Program& p, Store* s, int order) {
  Interp<F32Policy>(p, &s->floats, order).run();
}

}  // namespace sbport

// ---- C ABI used by tests / bench cpu_baseline (ctypes) ----
extern "C" {

const char* sp_last_error() { return sbport::g_err.c_str(); }

void* sp_parse(const char* text) {
  try {
    return new sb::Program(sb::parse_program(text));
  } catch (const sb::Error& e) {
    sbport::g_err = e.code + ": " + e.what();
  }
  return nullptr;
}
void sp_free_program(void* p) { delete static_cast<sb::Program*>(p); }
int sp_print(void* p, char* buf, std::size_t cap) {
  std::string s = sb::print_program(*static_cast<sb::Program*>(p));
  if (buf && cap) {
    std::size_t n = std::min(s.size(), cap - 1);
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return static_cast<int>(s.size());
}
void* sp_store_new() { return new sbport::Store(); }
void sp_store_free(void* s) { delete static_cast<sbport::Store*>(s); }
int sp_store_set(void* s, const char* name, const std::int64_t* data, std::int64_t n) {
  static_cast<sbport::Store*>(s)->ints[name].assign(data, data + n);
  return 0;
}
int sp_store_set_f32(void* s, const char* name, const float* data, std::int64_t n) {
  static_cast<sbport::Store*>(s)->floats[name].assign(data, data + n);
  return 0;
}
std::int64_t sp_store_get(void* s, const char* name, std::int64_t* out, std::int64_t cap) {
  auto& m = static_cast<sbport::Store*>(s)->ints;
  auto it = m.find(name);
  if (it == m.end()) return -1;
  std::int64_t n = static_cast<std::int64_t>(it->second.size());
  if (out) std::memcpy(out, it->second.data(), 8 * std::min(n, cap));
  return n;
}
std::int64_t sp_store_get_f32(void* s, const char* name, float* out, std::int64_t cap) {
  auto& m = static_cast<sbport::Store*>(s)->floats;
  auto it = m.find(name);
  if (it == m.end()) return -1;
  std::int64_t n = static_cast<std::int64_t>(it->second.size());
  if (out) std::memcpy(out, it->second.data(), 4 * std::min(n, cap));
  return n;
}
// mode 0: int64-wrap (bit-exact vs reference); 1: f32
int sp_execute(void* p, void* s, int mode, int order) {
  try {
    if (mode == 1) sbport::execute_f32(*static_cast<sb::Program*>(p), static_cast<sbport::Store*>(s), order);
    else sbport::execute_int(*static_cast<sb::Program*>(p), static_cast<sbport::Store*>(s), order);
    sbport::g_err.clear();
    return 0;
  } catch (const sb::Error& e) {
    sbport::g_err = e.code + ": " + e.what();
  } catch (const std::exception& e) {
    sbport::g_err = std::string("Exception: ") + e.what();
  }
  return 1;
}
std::int64_t sp_output_identity(void* p, const char* name) {
  return sb::output_identity(*static_cast<sb::Program*>(p), name);
}

}  // extern "C"
